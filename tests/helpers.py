"""Shared test helpers: hand-built pockets/poses used by the reference's own
tests (test_dockengine.cpp:29-62, 453-478), plus small numeric utilities."""
from __future__ import annotations

import math

import numpy as np

from paper_2110_11644_b200 import abi
from paper_2110_11644_b200.model import Ligand, Pocket


def explicit_pocket(dims, spacing, values, protein=()):
    """test_dockengine.cpp:37-45 (origin at zero, explicit node values)."""
    el = np.array([p[0] for p in protein], dtype=np.uint8)
    xyz = np.array([p[1] for p in protein], dtype=np.float64).reshape(-1, 3)
    return Pocket(np.zeros(3), spacing, tuple(dims), np.asarray(values, dtype=np.float64), el, xyz, id="test")


def flat_pocket(nodes, spacing, protein=()):
    """test_dockengine.cpp:47-52."""
    return explicit_pocket((nodes, nodes, nodes), spacing, np.zeros(nodes ** 3), protein)


def pyramid_pocket(nodes, spacing):
    """test_dockengine.cpp:457-467: 3(n-1) - L1 distance to the centre node."""
    c = (nodes - 1) // 2
    v = np.zeros(nodes ** 3)
    for iz in range(nodes):
        for iy in range(nodes):
            for ix in range(nodes):
                v[ix + nodes * (iy + nodes * iz)] = 3.0 * (nodes - 1) - (abs(ix - c) + abs(iy - c) + abs(iz - c))
    return explicit_pocket((nodes, nodes, nodes), spacing, v)


def eigen_centroid(conf: np.ndarray) -> np.ndarray:
    """rowwise().mean() in the Eigen 3.4 order."""
    c = np.asarray(conf, dtype=np.float64).reshape(-1, 3)
    n = c.shape[0]
    out = np.zeros(3)
    for r in range(2):
        p = float(c[0, r])
        size4 = (n - 1) & ~3
        i = 1
        while i < size4:
            p = p + ((float(c[i, r]) + float(c[i + 1, r])) + (float(c[i + 2, r]) + float(c[i + 3, r])))
            i += 4
        while i < n:
            p = p + float(c[i, r])
            i += 1
        out[r] = p / float(n)
    z = float(c[0, 2])
    for i in range(1, n):
        z = z + float(c[i, 2])
    out[2] = z / float(n)
    return out


def pose_at(lig: Ligand, target):
    """test_dockengine.cpp:469-476: identity rotation, centroid moved to
    target, zero torsion angles.  Returns (pose record, angles, conf)."""
    base = lig.xyz
    t = np.asarray(target, dtype=np.float64) - eigen_centroid(base)
    pose = np.zeros(1, dtype=abi.POSE_DTYPE)
    pose["rotation"][0] = [0.0, 0.0, 0.0, 1.0]
    pose["translation"][0] = t
    conf = base + t  # identity quaternion: toRotationMatrix() == I exactly
    return pose, np.zeros(lig.n_torsions), conf


def quat_dist(a, b) -> float:
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))))


def rel_err(a, b) -> np.ndarray:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.abs(a - b) / np.maximum(np.abs(b), 1e-12)


PI = math.pi
