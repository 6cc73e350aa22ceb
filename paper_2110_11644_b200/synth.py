"""Deterministic synthetic inputs for the benchmark configurations.

SURVEY.md §8d config 1/2: a 3CL-protease-sized pocket from
build_pocket(protein, centre (0,0,0), radius 12 A, spacing 0.375 A) -> 65^3
ternary nodes, over P = 2,400 synthetic protein heavy atoms (C/N/O/S =
0.63/0.17/0.19/0.01) placed by seeded rejection sampling in a cube minus an
ellipsoidal cavity; and drug-like ligands from the native SMILES generator
(vs_synth_smiles, ~30 heavy atoms, 5-7 rotatable bonds), seed 20260819 (the
reference CLI's default seed, tools/main.cpp:36).
"""
from __future__ import annotations

import numpy as np

DEFAULT_SEED = 20260819
ELEMENT_P = {0: 0.63, 1: 0.17, 2: 0.19, 3: 0.01}  # C, N, O, S


def synthetic_protein(n_atoms: int = 2400, seed: int = DEFAULT_SEED, half_box: float = 18.0,
                      cavity=(8.0, 7.0, 6.0), min_dist: float = 1.2):
    """Rejection-sampled protein heavy atoms around an ellipsoidal cavity at
    the origin.  Returns (element u8[P], xyz f64[P, 3])."""
    rng = np.random.default_rng(seed)
    cell = min_dist
    grid: dict = {}
    pts = []
    cav = np.asarray(cavity, dtype=np.float64)
    tries = 0
    while len(pts) < n_atoms:
        tries += 1
        if tries > 400 * n_atoms:
            raise RuntimeError("protein sampler could not place atoms; enlarge the box")
        p = rng.uniform(-half_box, half_box, 3)
        if np.sum((p / cav) ** 2) < 1.0:
            continue
        key = tuple(np.floor(p / cell).astype(int))
        ok = True
        for dx in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dz in (-1, 0, 1):
                    for q in grid.get((key[0] + dx, key[1] + dy, key[2] + dz), ()):
                        if np.sum((p - q) ** 2) < min_dist * min_dist:
                            ok = False
                            break
                    if not ok:
                        break
                if not ok:
                    break
            if not ok:
                break
        if not ok:
            continue
        grid.setdefault(key, []).append(p)
        pts.append(p)
    xyz = np.array(pts, dtype=np.float64)
    codes = np.array(list(ELEMENT_P.keys()), dtype=np.uint8)
    probs = np.array(list(ELEMENT_P.values()))
    elem = rng.choice(codes, size=n_atoms, p=probs / probs.sum()).astype(np.uint8)
    return elem, xyz


def voxel_mix(values: np.ndarray) -> dict:
    v = np.asarray(values)
    n = v.size
    return {"clash": float(np.mean(v == -10.0)), "contact": float(np.mean(v == 1.0)),
            "zero": float(np.mean(v == 0.0)), "nodes": int(n)}
