"""Multi-rank host logic on CPU (gloo, world_size 2): ligand sharding and the
top-K merge of per-rank rankings equal the single-process ranking
(merge.cpp:131-135 semantics: printed 4-decimal score desc, SMILES asc)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2110_11644_b200 import ranking


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _data(n=3000, seed=7):
    rng = np.random.default_rng(seed)
    # coarse scores so that printed-score ties and SMILES tie-breaks occur
    scores = np.round(rng.normal(30.0, 8.0, n), 5)
    scores[::97] = np.nan  # failed docks produce no row
    smiles = [f"C{'c' * int(rng.integers(0, 6))}N{int(rng.integers(0, 400))}" for _ in range(n)]
    status = np.zeros(n, dtype=np.int32)
    status[::131] = 2
    return scores, smiles, status


def _worker(rank, world, port, k, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    scores, smiles, status = _data()
    lo, hi = ranking.shard_range(len(scores), rank, world)
    rows = ranking.top_k(scores[lo:hi], smiles[lo:hi], k, status[lo:hi])
    merged = ranking.distributed_top_k(rows, k)
    if rank == 0:
        out.put(merged)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("k", [1, 50, 5000])
def test_two_rank_topk_equals_single_process(k):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, k, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    scores, smiles, status = _data()
    want = ranking.top_k(scores, smiles, k, status)
    assert merged == want


def test_shard_ranges_cover_exactly():
    for n in (0, 1, 7, 1000, 1_000_003):
        for world in (1, 2, 3, 8):
            rs = [ranking.shard_range(n, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))


def test_ranking_uses_printed_score_and_smiles_tiebreak():
    # 1.00004 and 1.00001 print as 1.0000: a tie broken by SMILES
    rows = ranking.top_k([1.00001, 1.00004, 2.0, float("inf")], ["CCO", "CC", "N", "O"], 10)
    assert rows == [(2.0, "N"), (1.0, "CC"), (1.0, "CCO")]
    assert ranking.format_row("CCO", 12.34567) == "CCO\t12.3457\n"
    with pytest.raises(ValueError):
        ranking.format_row("C", float("nan"))
