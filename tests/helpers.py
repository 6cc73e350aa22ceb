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


# ------------------------------------------------------------------ golden parity
def load_golden(name: str):
    """A fixture written by tests/golden/make_golden.py from oracle/_ref."""
    import os
    return np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", name))


def golden_pocket(g) -> Pocket:
    return Pocket(g["pocket_origin"], float(g["pocket_spacing"]), tuple(g["pocket_dims"]),
                  g["pocket_values_code"].astype(np.float64), g["protein_element"], g["protein_xyz"], id="golden")


def heavy_rmsd_per_ligand(batch, conf_a: np.ndarray, conf_b: np.ndarray) -> np.ndarray:
    """heavy_atom_rmsd (transform.cpp:99-113): in-frame, no superposition."""
    ao = batch.atom_offset
    heavy = np.concatenate([l.is_heavy.astype(bool) for l in batch.ligands])
    d2 = np.sum((np.asarray(conf_a, np.float64) - np.asarray(conf_b, np.float64)) ** 2, axis=1)
    out = np.zeros(batch.n_ligands)
    for i in range(batch.n_ligands):
        h = heavy[ao[i]:ao[i + 1]]
        out[i] = math.sqrt(float(np.mean(d2[ao[i]:ao[i + 1]][h]))) if h.any() else 0.0
    return out


def topk_identical_up_to_ties(smiles, score_a, score_b, k: int) -> tuple[bool, int]:
    """north_star: identical top-K ranking up to score ties within tolerance.
    Rows are ranked as cmd_merge does (printed 4-decimal score desc, SMILES
    asc; merge.cpp:131-135 via ranking.row_key).  Ligands whose printed score
    differs between the two runs (each within the score tolerance, checked
    separately) may move; after removing them from both rankings the first
    k - |moved| rows must be the same sequence.  Returns (ok, |moved|)."""
    from paper_2110_11644_b200 import ranking
    ka = [ranking.row_key(float(s), m) for s, m in zip(score_a, smiles)]
    kb = [ranking.row_key(float(s), m) for s, m in zip(score_b, smiles)]
    moved = {i for i in range(len(smiles)) if ka[i] != kb[i]}
    sk = lambda r: (-r[0], r[1].encode())  # noqa: E731
    oa = [i for i in sorted(range(len(smiles)), key=lambda i: sk(ka[i])) if i not in moved]
    ob = [i for i in sorted(range(len(smiles)), key=lambda i: sk(kb[i])) if i not in moved]
    kk = max(k - len(moved), 0)
    return oa[:kk] == ob[:kk], len(moved)


def golden_parity(g, batch, results, conf, k_top: int = 100) -> dict:
    """The north_star parity metrics of one run against a reference fixture."""
    from paper_2110_11644_b200 import ranking  # noqa: F401
    smi = [str(s) for s in g["smiles"]]
    rel = rel_err(results["best_score"], g["best_score"])
    rms = heavy_rmsd_per_ligand(batch, conf, g["best_conf"])
    top_ok, moved = topk_identical_up_to_ties(smi, results["best_score"], g["best_score"], k_top)
    return {
        "ligands": len(smi),
        "status_equal": float(np.mean(results["status"] == g["status"])),
        "score_within_1e-3": float(np.mean(rel <= 1e-3)),
        "rmsd_le_0.1": float(np.mean(rms <= 0.1)),
        "bit_exact_score": float(np.mean(results["best_score"] == g["best_score"])),
        "evals_equal": float(np.mean(results["scoring_evals"] == g["scoring_evals"])),
        "topk_identical_up_to_ties": bool(top_ok), "topk_moved_rows": int(moved), "k": k_top,
        "max_rel_err": float(np.max(rel)), "max_rmsd": float(np.max(rms)),
    }


def assert_north_star(rep: dict):
    assert rep["status_equal"] == 1.0, rep
    assert rep["score_within_1e-3"] >= 0.999, rep
    assert rep["rmsd_le_0.1"] >= 0.999, rep
    assert rep["evals_equal"] >= 0.999, rep
    assert rep["topk_identical_up_to_ties"], rep
