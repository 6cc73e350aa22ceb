#!/usr/bin/env python3
"""Small dock runs for bounds-checked builds (development check; the pool
does not allow compute-sanitizer):

    tools/build_variant.sh dbg "-DVS_DEBUG_CHECKS"
    VSDOCK_LIB=paper_2110_11644_b200/_lib/var/dbg.so python tools/sanitize_dock.py

k = 30 (warp select), k = 40 (CTA select in shared memory), k = 8192 (CTA
select in global scratch), want_conformation on (k_best_conf), a flatten of
ligands with non-rigid D_t subtrees."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))

from paper_2110_11644_b200 import abi, api, synth  # noqa: E402
from paper_2110_11644_b200.model import LigandBatch  # noqa: E402


def main():
    ctx = api.default_context(0)
    el, xyz = synth.synthetic_protein(1200, seed=5, half_box=13.0)
    pocket = api.build_pocket(el, xyz, [0.0, 0.0, 0.0], 8.0, 0.5, ctx)
    smi = api.synthetic_smiles(24, seed=17, heavy=(14, 34), rot=(0, 8))
    b = LigandBatch(api.prepare_ligand(smi, quantize=True, ctx=ctx))
    for k in (30, 40):
        r = api.dock_and_score_batch(pocket, b, abi.ScoringConfig(restarts=k, rescored=min(k, 30)), ctx)
        print("k", k, r.results["status"][:6], r.results["best_score"][:3])
    small = LigandBatch(sorted(b.ligands, key=lambda l: l.n_atoms)[:1])
    r = api.dock_and_score_batch(pocket, small, abi.ScoringConfig(restarts=8192, rescored=30), ctx)
    print("k 8192", r.results["status"], r.results["best_score"])
    from test_gpu_parity import _flip_torsion
    raw = api.prepare_smiles(api.synthetic_smiles(24, seed=777, heavy=(20, 50), rot=(3, 10), grammar=1), mode=1)
    fl = LigandBatch([_flip_torsion(l, l.n_torsions - 1) for l in raw if l.n_torsions >= 3])
    c, a, s = api.flatten(fl, 20, ctx)
    print("flatten", s[:6])


if __name__ == "__main__":
    main()
