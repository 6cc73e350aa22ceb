#!/usr/bin/env python3
"""Phase profile of k_flatten_dep (development): run with a library built with
-DVS_FLAT_PROF (tools/build_variant.sh fprof "-DVS_FLAT_PROF"):

    VSDOCK_LIB=paper_2110_11644_b200/_lib/var/fprof.so python tools/flat_prof.py [n_ligands]

Prints thread 0's clock64() time per phase of the flatten loop, summed over
ligands (CTAs): warp 0's serial sections (A, D) against the 9-warp
candidate evaluation (B, C) and the barrier that closes it.
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))

from paper_2110_11644_b200 import api, native, synth  # noqa: E402

NAMES = ["A: D_t, common positions, shared matrices (warp 0) + barrier", "B: candidate transforms (own share)",
         "C: filter sums (own share)", "barrier after B/C (waiting for the other warps)", "D: argmax + filter test",
         "D: exact sums of near ties", "D: prefix advance"]


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    ctx = api.default_context(0)
    el, xyz = synth.synthetic_protein()
    pocket = api.build_pocket(el, xyz, [0.0, 0.0, 0.0], 12.0, 0.375, ctx)
    ligs = api.prepare_ligand(api.synthetic_smiles(n, seed=20260820), quantize=True, ctx=ctx)
    cfg = api.ScoringConfig(restarts=30, rescored=30)
    fn = native.lib().vs_debug_flat_phase_read
    fn.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
    buf = (C.c_ulonglong * 16)()
    api.dock_and_score_batch(pocket, ligs, cfg, ctx)  # warm-up
    fn(buf, 1)
    r = api.dock_and_score_batch(pocket, ligs, cfg, ctx)
    fn(buf, 1)
    tot = sum(buf[i] for i in range(7)) or 1
    print(f"stage ms {r.stage_ms}; CTAs {buf[7]}")
    print(f"decisions evaluated {buf[8]}, exact near-tie paths {buf[9]} ({100.0 * buf[9] / max(buf[8], 1):.2f} %)")
    for i, name in enumerate(NAMES):
        print(f"{name:64s} {100.0 * buf[i] / tot:6.2f} %   {buf[i] / max(buf[7], 1):10.0f} cycles/ligand")


if __name__ == "__main__":
    main()
