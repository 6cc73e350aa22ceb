"""Generate the golden fixtures from the REFERENCE's own code (oracle/_ref:
the reference sources compiled unchanged against the Eigen-subset shim).
Run here, where /root/reference exists:  python tests/golden/make_golden.py

config1.npz -- SURVEY.md §8d config 1 at fixture scale: the synthetic
  3CL-sized pocket (build_pocket r=12 A, h=0.375 A over 2,400 synthetic
  protein atoms), 1,000 synthetic drug-like ligands prepared with the
  reference's prepare_ligand and f32-quantised, dock_and_score with k=4,
  rescored=30 (reference results: best score/pose/angles/evals, every best
  conformation).
config2_k30.npz -- the BENCHED configuration (BASELINE configs[1], bench.py
  defaults): the same pocket, the first 1,200 ligands of the bench library
  stream (seed 20260820 = bench --seed + 1), k=30, rescored=30.
config3_cells.npz -- BASELINE configs[2] size sweep at fixture scale: 16
  ligands per reachable (heavy, rotors) cell of tools/sweep.py's grid (wide
  grammar, heavy window n-2..n+2, rotors exactly m), k=30, rescored=30.

Conformations are stored as float32 (the fixtures check RMSD <= 0.1 A; scores
and angles stay float64 for the bit-exact fractions).
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from oracle import Oracle  # noqa: E402
from paper_2110_11644_b200 import abi, api, synth  # noqa: E402
from paper_2110_11644_b200.model import LigandBatch  # noqa: E402

THREADS = os.cpu_count() or 8
CELLS_HEAVY = (10, 20, 30, 40, 50, 60, 70, 80)
CELLS_ROT = (0, 3, 6, 9, 12, 15)


def dock_fixture(ref, pocket, smi, k, rescored, name, extra=None, with_pocket=True, el=None, xyz=None):
    ligs = [ref.prepare(s, 0, True) for s in smi]  # prepare_ligand + quantize_to_wire
    b = LigandBatch(ligs)
    cfg = abi.ScoringConfig(restarts=k, rescored=rescored)
    out = ref.dock_batch(pocket, b, cfg, nthreads=THREADS)
    r = out["results"]
    fields = dict(
        smiles=np.array(smi), prepared_xyz=b.xyz, atom_offset=b.atom_offset, torsion_offset=b.torsion_offset,
        status=r["status"], best_score=r["best_score"], best_geo_score=r["best_geo_score"], rotation=r["rotation"],
        translation=r["translation"], scoring_evals=r["scoring_evals"], poses_evaluated=r["poses_evaluated"],
        best_angles=out["angles"], best_conf=out["conformation"].astype(np.float32),
        restarts=np.array(k), rescored=np.array(rescored))
    if with_pocket:
        fields.update(protein_element=el, protein_xyz=xyz,
                      pocket_values_code=np.round(pocket.values).astype(np.int8),
                      pocket_dims=np.array(pocket.dims), pocket_origin=pocket.origin,
                      pocket_spacing=np.array(pocket.spacing))
    if extra:
        fields.update(extra)
    np.savez_compressed(os.path.join(HERE, name), **fields)
    print(f"wrote {name}: {len(smi)} ligands, statuses {np.unique(r['status'])}, "
          f"mean best {float(np.mean(r['best_score'])):.4f}")


def main(which=("config1", "config2_k30", "config3_cells")):
    ref = Oracle("ref")
    el, xyz = synth.synthetic_protein()
    pocket = ref.build_pocket(el, xyz, [0, 0, 0], 12.0, 0.375)
    assert set(np.unique(pocket.values)) <= {-10.0, 0.0, 1.0}
    if "config1" in which:
        dock_fixture(ref, pocket, api.synthetic_smiles(1000, seed=20260819), 4, 30, "config1.npz", el=el, xyz=xyz)
    if "config2_k30" in which:
        dock_fixture(ref, pocket, api.synthetic_smiles(1200, seed=20260820), 30, 30, "config2_k30.npz",
                     el=el, xyz=xyz)
    if "config3_cells" in which:
        smi, cell = [], []
        for n in CELLS_HEAVY:
            for m in CELLS_ROT:
                try:
                    s = api.synthetic_smiles(16, seed=20260821 + 100 * n + m, heavy=(n - 2, n + 2), rot=(m, m),
                                             grammar=1)
                except ValueError:
                    continue  # unreachable by the grammar (tools/sweep.py lists the same cells as skipped)
                smi += s
                cell += [(n, m)] * len(s)
        dock_fixture(ref, pocket, smi, 30, 30, "config3_cells.npz", extra={"cell": np.array(cell, dtype=np.int32)},
                     with_pocket=False)


if __name__ == "__main__":
    main(tuple(sys.argv[1:]) or ("config1", "config2_k30", "config3_cells"))
