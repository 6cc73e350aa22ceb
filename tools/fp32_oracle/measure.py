#!/usr/bin/env python3
"""North_star tolerance of an FP32 search against the reference (see
make_fp32.py): docks the reference golden fixtures with the FP32 oracle
variant and prints the parity metrics the GPU test asserts."""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import oracle as O  # noqa: E402
from helpers import golden_parity, golden_pocket, load_golden  # noqa: E402
from paper_2110_11644_b200 import abi, api  # noqa: E402
from paper_2110_11644_b200.model import LigandBatch  # noqa: E402

O.PORT_LIB = os.path.join(HERE, "_build", "liboracle_fp32.so")
fp32 = O.Oracle("port", trig=0)
pocket = golden_pocket(load_golden("config1.npz"))
for name in sys.argv[1:] or ["config1.npz", "config2_k30.npz"]:
    g = load_golden(name)
    smi = [str(s) for s in g["smiles"]]
    graphs = api.prepare_smiles(smi, mode=1, nthreads=os.cpu_count() or 8)
    ao = g["atom_offset"]
    b = LigandBatch([l.with_xyz(g["prepared_xyz"][ao[i]:ao[i + 1]]) for i, l in enumerate(graphs)])
    cfg = abi.ScoringConfig(restarts=int(g["restarts"]), rescored=int(g["rescored"]))
    t = time.time()
    out = fp32.dock_batch(pocket, b, cfg, nthreads=os.cpu_count() or 8)
    rep = golden_parity(g, b, out["results"], out["conformation"])
    rep["fixture"], rep["precision"], rep["seconds"] = name, "fp32 search (oracle restatement, float)", time.time() - t
    print(json.dumps(rep))
