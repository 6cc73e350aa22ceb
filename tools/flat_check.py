#!/usr/bin/env python3
"""Flatten parity check (development): GPU flatten of synthetic embedded
ligands against the oracle port, bitwise on conformations and angles.
    VSDOCK_LIB=... python tools/flat_check.py [n] [grammar]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
from oracle import Oracle  # noqa: E402
from paper_2110_11644_b200 import api  # noqa: E402
from paper_2110_11644_b200.model import LigandBatch  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
grammar = int(sys.argv[2]) if len(sys.argv) > 2 else 0
smi = api.synthetic_smiles(n, seed=4242, heavy=(8, 60) if grammar else (26, 34), rot=(0, 12) if grammar else (5, 7),
                           grammar=grammar)
ligs = api.prepare_smiles(smi, mode=1, nthreads=os.cpu_count() or 8)
b = LigandBatch(ligs)
ctx = api.default_context(0)
conf, ang, st = api.flatten(ligs, 20, ctx)
orc = Oracle("port")
wconf, wang, wst = orc.flatten(b, 20, nthreads=os.cpu_count() or 8)
bad = []
for i in range(b.n_ligands):
    a0, a1 = b.atom_offset[i], b.atom_offset[i + 1]
    t0, t1 = b.torsion_offset[i], b.torsion_offset[i + 1]
    ok = st[i] == wst[i] and np.array_equal(conf[a0:a1].view(np.uint64), wconf[a0:a1].view(np.uint64)) and \
        np.array_equal(ang[t0:t1].view(np.uint64), wang[t0:t1].view(np.uint64))
    if not ok:
        bad.append(i)
print("ligands", b.n_ligands, "mismatches", len(bad), "first", bad[:10])
for i in bad[:3]:
    t0, t1 = b.torsion_offset[i], b.torsion_offset[i + 1]
    print(i, "N", ligs[i].n_atoms, "m", ligs[i].n_torsions, "st", st[i], wst[i], "ang", np.round(ang[t0:t1], 4),
          np.round(wang[t0:t1], 4))
    a0, a1 = b.atom_offset[i], b.atom_offset[i + 1]
    d = np.abs(conf[a0:a1] - wconf[a0:a1])
    print("   max |dconf|", d.max(), "rows", np.nonzero(d.max(1))[0][:10], "base==gpu", np.array_equal(conf[a0:a1], b.xyz[a0:a1]),
          "base==oracle", np.array_equal(wconf[a0:a1], b.xyz[a0:a1]))
