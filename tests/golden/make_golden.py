"""Generate the golden fixtures from the REFERENCE's own code (oracle/_ref:
the reference sources compiled unchanged against the Eigen-subset shim).
Run here, where /root/reference exists:  python tests/golden/make_golden.py

config1.npz -- SURVEY.md §8d config 1 at fixture scale: the synthetic
  3CL-sized pocket (build_pocket r=12 A, h=0.375 A over 2,400 synthetic
  protein atoms), 1,000 synthetic drug-like ligands prepared with the
  reference's prepare_ligand and f32-quantised, dock_and_score with k=4,
  rescored=30 (reference results: best score/pose/angles/evals).
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


def main():
    ref = Oracle("ref")
    el, xyz = synth.synthetic_protein()
    pocket = ref.build_pocket(el, xyz, [0, 0, 0], 12.0, 0.375)
    smi = api.synthetic_smiles(1000, seed=20260819)
    ligs = [ref.prepare(s, 0, True) for s in smi]  # prepare_ligand + quantize_to_wire
    b = LigandBatch(ligs)
    cfg = abi.ScoringConfig(restarts=4, rescored=30)
    out = ref.dock_batch(pocket, b, cfg, nthreads=os.cpu_count() or 8)
    r = out["results"]
    n_conf_lig = 100
    np.savez_compressed(
        os.path.join(HERE, "config1.npz"),
        protein_element=el, protein_xyz=xyz, pocket_values_code=np.round(pocket.values).astype(np.int8),
        pocket_dims=np.array(pocket.dims), pocket_origin=pocket.origin, pocket_spacing=np.array(pocket.spacing),
        smiles=np.array(smi), prepared_xyz=b.xyz, atom_offset=b.atom_offset, torsion_offset=b.torsion_offset,
        status=r["status"], best_score=r["best_score"], best_geo_score=r["best_geo_score"], rotation=r["rotation"],
        translation=r["translation"], scoring_evals=r["scoring_evals"], poses_evaluated=r["poses_evaluated"],
        best_angles=out["angles"], best_conf_first100=out["conformation"][:b.atom_offset[n_conf_lig]],
        restarts=np.array(4), rescored=np.array(30))
    assert set(np.unique(pocket.values)) <= {-10.0, 0.0, 1.0}
    print("wrote config1.npz:", len(smi), "ligands; statuses", np.unique(r["status"]),
          "mean best", float(np.mean(r["best_score"])))


if __name__ == "__main__":
    main()
