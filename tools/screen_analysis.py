"""Development analysis (not product, not a test): how many local_search
neighbours an FP32 screen with a proven per-neighbour error bound would have
to re-evaluate exactly in FP64.

Builds oracle/vs_oracle.cpp with -DVSO_TRACE (per-neighbour score, current
score, sum over moved heavy-atom samples of the cell's L1 gradient bound),
docks a sample of the bench library (configs[1], k=30) on the CPU, then for
an error model E_j = delta * gsum_j + n_moved_j * eps counts the neighbours
whose interval reaches the decision threshold max(cur, max_i lb_i).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from oracle import Oracle  # noqa: E402
from paper_2110_11644_b200 import abi, api, synth  # noqa: E402
from paper_2110_11644_b200.model import LigandBatch  # noqa: E402

LIB = "/tmp/liboracle_trace.so"


def main(n_lig=40, k=30, seed=20260820):
    subprocess.check_call(["g++", "-std=c++20", "-O2", "-fPIC", "-ffp-contract=off", "-DVSO_TRACE",
                           "-I" + os.path.join(ROOT, "include"), "-shared", "-o", LIB,
                           os.path.join(ROOT, "oracle", "vs_oracle.cpp"), "-lpthread"])
    ref = Oracle("ref")
    el, xyz = synth.synthetic_protein()
    pocket = ref.build_pocket(el, xyz, [0, 0, 0], 12.0, 0.375)
    smi = api.synthetic_smiles(n_lig, seed=seed)
    ligs = [ref.prepare(s, 0, True) for s in smi]
    b = LigandBatch(ligs)
    o = Oracle("port")
    o.lib = C.CDLL(LIB)
    o.__init__.__func__  # keep the loader's signatures: rebind on the trace lib
    tr = Oracle.__new__(Oracle)
    tr.kind, tr.trig = "port", 1
    path_backup = sys.modules["oracle"].PORT_LIB
    sys.modules["oracle"].PORT_LIB = LIB
    tr.__init__("port", 1)
    sys.modules["oracle"].PORT_LIB = path_backup
    tr.lib.vso_trace_open(b"/tmp/trace.bin")
    tr.dock_batch(pocket, b, abi.ScoringConfig(restarts=k, rescored=30), nthreads=1, want_conf=False)
    tr.lib.vso_trace_close()
    rec = np.fromfile("/tmp/trace.bin", dtype=np.float64).reshape(-1, 6)
    iters = np.nonzero(rec[:, 0] == -1e300)[0]
    print(f"{len(iters)} iterations, {len(rec) - len(iters)} neighbours")
    bounds = iters.tolist() + [len(rec)]
    groups = []
    for a, e in zip(bounds[:-1], bounds[1:]):
        g = rec[a + 1:e]
        if len(g):
            groups.append(g)
    for delta, gm in ((1e-6, 0), (1e-5, 0), (3e-5, 0), (1e-4, 0), (1e-5, 33), (3e-5, 33), (1e-4, 33), (1e-3, 33)):
        for eps in (1e-6,):
            ex = 0
            nonimp = 0
            for g in groups:
                s, cur, gs, nm = g[:, 0], g[0, 1], g[:, 2], g[:, 3]
                E = delta * (gs if gm == 0 else gm * g[:, 5]) + nm * eps
                tau = max(cur, np.max(s - E))
                ex += int(np.sum(s + E >= tau))
                nonimp += int(np.all(s <= cur))
            print(f"G {gm or 'cell'} delta {delta:g} eps {eps:g}: exact evals per iteration {ex / len(groups):.2f} "
                  f"(of {np.mean([len(g) for g in groups]):.1f}); non-improving iterations {nonimp / len(groups):.3f}")
    # gaps
    gaps = []
    for g in groups:
        s, cur = np.sort(g[:, 0])[::-1], g[0, 1]
        gaps.append((s[0] - cur, s[0] - s[1]))
    gaps = np.array(gaps)
    print("best-cur gap quantiles", np.quantile(gaps[:, 0], [0.01, 0.05, 0.1, 0.5]))
    print("best-second gap quantiles", np.quantile(gaps[:, 1], [0.01, 0.05, 0.1, 0.5]))
    print("moved samples near a face (<1e-4):", np.mean(rec[rec[:, 0] != -1e300][:, 4] < 1e-4))
    print("gsum per neighbour mean", np.mean(rec[rec[:, 0] != -1e300][:, 2]),
          "n_moved mean", np.mean(rec[rec[:, 0] != -1e300][:, 3]))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 40)
