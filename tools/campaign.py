#!/usr/bin/env python3
"""BASELINE configs[3]: one record library x one pocket, sharded over N GPUs
(one process per GPU under torchrun), with the host ranking merge.

    python tools/campaign.py --ligands 10000000 [--distinct 1000000]
    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \
        tools/campaign.py --ligands 10000000

* The library is an .xslb image (header + encode_record records) of
  --ligands records: --distinct prepared drug-like ligands (~30 heavy /
  5-7 rotors, bench library stream) repeated in blocks to the requested size
  (each repeat is docked again: no caching anywhere).  Rank 0 builds it once
  into --dir (reused when present); every rank maps the same file.
* Each rank runs vs_run_rank on its slab (plan_slabs: records whose start
  lies in [size r / N, size (r + 1) / N), pipeline.cpp:32-45): host framing,
  GPU decode + dock on --workers CUDA workers of its GPU, rows to
  rank<r>.scores.  The timed region is the whole rank (file bytes in, rows
  out): e2e.  value = records docked on all ranks / max rank wall time.
* Rank 0 then merges every rank file with the native merge (cmd_merge's
  order, merge.cpp:81-147) into ranking.tsv, timed separately, and prints one
  JSON line with the ranking's SHA-256 (identical for every N).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import mmap
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2110_11644_b200 import abi, api, native, synth  # noqa: E402


def build_library(path: str, n: int, distinct: int, seed: int, ctx) -> dict:
    t0 = time.time()
    smi = api.synthetic_smiles(distinct, seed=seed)
    ligs = []
    step = 131072
    for i in range(0, distinct, step):
        ligs += api.prepare_ligand(smi[i:i + step], quantize=True, ctx=ctx, nthreads=os.cpu_count() or 8)
    block = api.encode_records(ligs, smi)
    reps, rest = divmod(n, distinct)
    tail = api.encode_records(ligs[:rest], smi[:rest]) if rest else b""
    tmp = path + ".tmp"
    with open(tmp, "wb") as f:
        f.write(api.XSLB_HEADER)
        for _ in range(reps):
            f.write(block)
        f.write(tail)
    os.replace(tmp, path)
    return {"build_s": round(time.time() - t0, 1), "distinct": distinct, "records": n}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ligands", type=int, default=10_000_000)
    ap.add_argument("--distinct", type=int, default=1_000_000)
    ap.add_argument("--seed", type=int, default=20260820)
    ap.add_argument("--restarts", type=int, default=30)
    ap.add_argument("--workers", type=int, default=2)
    ap.add_argument("--batch", type=int, default=65536)
    ap.add_argument("--dir", default="/tmp/vs_campaign")
    ap.add_argument("--keep-ranking", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("gloo")  # host barriers / scalar max only: no data-path collective

    def barrier():
        if dist is not None:
            dist.barrier()

    os.makedirs(args.dir, exist_ok=True)
    lib_path = os.path.join(args.dir, f"library_{args.ligands}_{args.distinct}_{args.seed}.xslb")
    ctx = api.default_context(local)
    info = {}
    if rank == 0 and not os.path.exists(lib_path):
        info = build_library(lib_path, args.ligands, args.distinct, args.seed, ctx)
    barrier()
    el, xyz = synth.synthetic_protein()
    pocket = api.build_pocket(el, xyz, [0.0, 0.0, 0.0], 12.0, 0.375, ctx).to_host()
    cfg = api.ScoringConfig(restarts=args.restarts, rescored=30)
    size = os.path.getsize(lib_path)
    slab = api.plan_slabs(size, world)[rank]
    out_path = os.path.join(args.dir, f"rank{rank}.scores")
    with open(lib_path, "rb") as f:
        mm = mmap.mmap(f.fileno(), 0, access=mmap.ACCESS_READ)
        buf = np.frombuffer(mm, dtype=np.uint8)
        sink = open(out_path, "wb")

        def _read(_u, off, out, n):
            n = max(0, min(n, size - off))
            import ctypes as C
            C.memmove(out, buf.ctypes.data + off, n)
            return n

        def _write(_u, p, n):
            import ctypes as C
            sink.write(C.string_at(p, n))
            return 0

        import ctypes as C
        rf, wf = abi.READ_FN(_read), abi.WRITE_FN(_write)
        rc = abi.RankConfig()
        native.lib().vs_rank_config_default(C.byref(rc))
        dev = (C.c_int32 * 1)(local)
        rc.n_devices, rc.devices = 1, C.cast(dev, C.POINTER(C.c_int32))
        rc.workers_per_device, rc.batch_records = args.workers, args.batch
        rc.chunk_bytes = 8 << 20
        st = abi.RankStats()
        barrier()
        t0 = time.perf_counter()
        native.check(native.lib().vs_run_rank(size, rf, None, slab[0], slab[1], C.byref(pocket.desc()), C.byref(cfg),
                                              C.byref(rc), wf, None, C.byref(st)), "vs_run_rank")
        sink.close()
        wall = time.perf_counter() - t0
        del buf
        mm.close()
    stats = st.as_dict()
    t = [wall, float(stats["ligands_docked"] + stats["dock_errors"])]
    if dist is not None:
        import torch
        tw = torch.tensor([wall], dtype=torch.float64)
        dist.all_reduce(tw, op=dist.ReduceOp.MAX)
        tn = torch.tensor([t[1]], dtype=torch.float64)
        dist.all_reduce(tn, op=dist.ReduceOp.SUM)
        wall, docked = float(tw[0]), float(tn[0])
    else:
        docked = t[1]
    barrier()
    if rank != 0:
        return
    # ---- host ranking merge of every rank's rows (cmd_merge order)
    texts = [open(os.path.join(args.dir, f"rank{r}.scores"), "rb").read() for r in range(world)]
    t1 = time.perf_counter()
    ranking_text, rows = api.merge_rankings(texts)
    merge_s = time.perf_counter() - t1
    digest = hashlib.sha256(ranking_text.encode()).hexdigest()
    if args.keep_ranking:
        with open(os.path.join(args.dir, "ranking.tsv"), "w") as f:
            f.write(ranking_text)
    top = ranking_text.splitlines()[:3]
    print(json.dumps({
        "metric": "ligands docked+scored/sec (configs[3] campaign)", "value": docked / wall, "unit": "ligands/s",
        "n_gpus": world, "scaling": "strong", "records": int(docked), "wall_s": wall,
        "config": {"workload": f"configs[3]: {args.ligands} records ({args.distinct} distinct prepared ligands "
                               f"repeated) x 1 pocket (65^3), k={args.restarts}, rescored=30, sharded by plan_slabs",
                   "workers_per_gpu": args.workers, "batch_records": args.batch},
        "rank0_stats": {k: stats[k] for k in ("ligands_docked", "records_skipped", "dock_errors", "batches",
                                              "docker_busy_seconds", "splitter_busy_seconds", "writer_busy_seconds")},
        "merge": {"rows": rows, "seconds": merge_s, "sha256": digest, "top3": top},
        "library": info or {"records": args.ligands, "reused": True}}))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
