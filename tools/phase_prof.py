#!/usr/bin/env python3
"""Phase profile of k_search (development): run with a library built with
-DVS_PHASE_PROF (tools/build_variant.sh prof "-DVS_PHASE_PROF"):

    VSDOCK_LIB=paper_2110_11644_b200/_lib/var/prof.so python tools/phase_prof.py [n_ligands]

Prints the share of warp time (clock64 cycles summed over warps) per phase.
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))

from paper_2110_11644_b200 import api, native, synth  # noqa: E402

NAMES = ["item setup", "transforms+mvar rebuild", "rigid samples", "torsion samples", "sums+argmax",
         "adopt rigid (+pivot)", "adopt torsion (+tors, pivot)", "halving", "outputs", "transforms+mvar REBUILD"]


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    ctx = api.default_context(0)
    el, xyz = synth.synthetic_protein()
    pocket = api.build_pocket(el, xyz, [0.0, 0.0, 0.0], 12.0, 0.375, ctx)
    ligs = api.prepare_ligand(api.synthetic_smiles(n, seed=20260820), quantize=True, ctx=ctx)
    cfg = api.ScoringConfig(restarts=30, rescored=30)
    lib = native.lib()
    fn = lib.vs_debug_phase_read
    fn.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
    buf = (C.c_ulonglong * 24)()
    api.dock_and_score_batch(pocket, ligs, cfg, ctx)  # warm-up
    fn(buf, 1)
    r = api.dock_and_score_batch(pocket, ligs, cfg, ctx)
    fn(buf, 1)
    tot = (sum(buf[i] for i in range(len(NAMES))) + buf[19] + buf[20] + buf[21] + buf[22] + buf[23]) or 1
    print(f"stage ms {r.stage_ms}")
    print(f"iterations {buf[11]}, with matrix rebuild {buf[10]} ({100.0 * buf[10] / max(buf[11], 1):.1f} %)")
    nb = max(buf[10], 1)
    print(f"per rebuild (max over lanes): sincos {buf[12] / nb:.0f}  chain {buf[13] / nb:.0f}  "
          f"rigid transforms {buf[14] / nb:.0f} cycles; whole rebuild phase {buf[9] / nb:.0f}; "
          f"of the chain: matrix setups {buf[15] / nb:.0f}")
    if buf[17]:
        print(f"screen: rows screened {buf[17]}, exact evaluations {buf[16]} ({buf[16] / max(buf[11], 1):.2f} per "
              f"iteration, rigid {buf[18]})")
    for i, name in enumerate(NAMES):
        print(f"{name:32s} {100.0 * buf[i] / tot:6.2f} %   {buf[i] / 1e9:10.3f} Gcycles")
    if buf[22] + buf[23]:
        print(f"ligand-end barrier wait (+ end of a ligand) {100.0 * buf[22] / tot:.2f} %, ligand staging + start "
              f"matrices {100.0 * buf[23] / tot:.2f} %")
    sub = buf[19] + buf[20] + buf[21] + buf[6]
    if buf[19] + buf[20] + buf[21]:
        print("adopt torsion split (% of all): matrices + D_t heavy atoms "
              f"{100.0 * buf[19] / tot:.2f}, hydrogens {100.0 * buf[20] / tot:.2f}, stage-t prefixes "
              f"{100.0 * buf[21] / tot:.2f}, vcur + pivot {100.0 * buf[6] / tot:.2f} (sum {100.0 * sub / tot:.2f})")


if __name__ == "__main__":
    main()
