#!/usr/bin/env python3
"""BASELINE configs[2]: ligand-size sweep (heavy atoms x rotatable bonds) on
one B200 -- the divergence / bucketing stress case.  For every feasible cell
(n heavy in {10..80}, m rotors in {0,3,...,15}) it prepares `--per-cell`
synthetic ligands (heavy window n-2..n+2, rotor window m..m), docks them with
k=30 and prints one JSON line per cell: GPU ligands/s (device time of the dock
stages), the stage split, and the reference CPU rate (oracle/_ref, all host
threads) on a small sample of the same cell.  Cells the generator cannot reach
are listed as skipped.

    python tools/sweep.py [--per-cell 20000] [--cpu-sample 64]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))

from paper_2110_11644_b200 import api, synth  # noqa: E402
from paper_2110_11644_b200.model import LigandBatch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--per-cell", type=int, default=20000)
    ap.add_argument("--distinct", type=int, default=8192,
                    help="distinct ligands generated per cell (generated on all host threads); the cell's batch "
                         "repeats them up to --per-cell (every copy is docked again)")
    ap.add_argument("--cpu-sample", type=int, default=64)
    ap.add_argument("--gen-seconds", type=float, default=90.0, help="SMILES generation budget per cell")
    ap.add_argument("--heavy", default="10,20,30,40,50,60,70,80")
    ap.add_argument("--rot", default="0,3,6,9,12,15")
    ap.add_argument("--grammar", type=int, default=1, help="synthetic SMILES grammar: 0 drug-like, 1 wide")
    args = ap.parse_args()
    ctx = api.default_context(0)
    el, xyz = synth.synthetic_protein()
    pocket = api.build_pocket(el, xyz, [0.0, 0.0, 0.0], 12.0, 0.375, ctx)
    cfg = api.ScoringConfig(restarts=30, rescored=30)
    threads = os.cpu_count() or 8
    ref = None
    try:
        from oracle import Oracle, available
        if available("ref"):
            ref = Oracle("ref")
            host_pocket = pocket.to_host()
    except Exception:  # pragma: no cover - reported below
        ref = None
    for n in [int(x) for x in args.heavy.split(",")]:
        for m in [int(x) for x in args.rot.split(",")]:
            cell = {"heavy": n, "rotors": m}
            distinct = min(args.distinct, args.per_cell)
            # rejection sampling into narrow windows is slow: chunks of 256 (one
            # generator block) with derived seeds on all host threads (ctypes
            # releases the GIL); a chunk the generator gives up on is retried
            # with the next seed
            from concurrent.futures import ThreadPoolExecutor

            def chunk(i):
                try:
                    return api.synthetic_smiles(256, seed=20260819 + 1000 * n + m + 7919 * i,
                                                heavy=(max(1, n - 2), n + 2), rot=(m, m), grammar=args.grammar)
                except ValueError:
                    return []
            t_gen = time.perf_counter()
            parts, i0 = [], 0
            with ThreadPoolExecutor(threads) as ex:
                while (sum(len(p) for p in parts) < distinct and i0 < 8 * (distinct // 256 + 1)
                       and time.perf_counter() - t_gen < args.gen_seconds):
                    k = threads
                    parts += list(ex.map(chunk, range(i0, i0 + k)))
                    i0 += k
            gen_s = time.perf_counter() - t_gen
            if not any(parts):
                print(json.dumps({**cell, "skipped": "generator cannot reach this (heavy, rotor) window"}), flush=True)
                continue
            uniq = [x for p in parts for x in p][:distinct]
            smi = (uniq * (args.per_cell // len(uniq) + 1))[:args.per_cell]
            t0 = time.perf_counter()
            ul = api.prepare_ligand(uniq, quantize=True, ctx=ctx, nthreads=threads)
            ligs = (ul * (args.per_cell // len(ul) + 1))[:args.per_cell]
            prep_s = time.perf_counter() - t0
            batch = LigandBatch(ligs)
            api.dock_and_score_batch(pocket, LigandBatch(ligs[:2048]), cfg, ctx, want_conformation=False)  # warm-up
            r = api.dock_and_score_batch(pocket, batch, cfg, ctx, want_conformation=False)
            line = {**cell, "ligands": len(ligs), "gpu_ligands_per_s": len(ligs) / (r.kernel_ms / 1e3),
                    "stage_ms": {k: round(v, 2) for k, v in r.stage_ms.items()},
                    "ok": int((r.results["status"] == 0).sum()), "host_prep_s": round(prep_s, 2), "distinct": len(uniq), "smiles_gen_s": round(gen_s, 1),
                    "mean_atoms": float(batch.n_atoms_total / max(batch.n_ligands, 1))}
            if ref is not None and args.cpu_sample > 0:
                sample = LigandBatch(ligs[:args.cpu_sample])
                t0 = time.perf_counter()
                ref.dock_batch(host_pocket, sample, cfg, nthreads=threads, want_conf=False)
                dt = time.perf_counter() - t0
                line["cpu_reference_ligands_per_s"] = args.cpu_sample / dt
                line["cpu_threads"] = threads
            print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
