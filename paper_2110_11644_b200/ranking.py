"""Host-side ranking of dock results and the multi-GPU top-K merge.

The reference writes one row per docked ligand, ``SMILES\\t%.4f``
(pipeline.cpp:47-62 ``format_row``: ``std::to_chars`` fixed, 4 decimals;
non-finite scores are rejected), and ``cmd_merge`` parses the rows back and
stable-sorts them by (score desc, SMILES asc) (merge.cpp:62-77, 131-135).
The ranking therefore compares the *printed* 4-decimal scores; this module
does the same, so the top-K of a sharded run equals the reference's merged
ranking.  Multi-GPU runs shard ligands across ranks with no device
collective; only the top-K rows travel (``torch.distributed`` object
gather, host side).
"""
from __future__ import annotations

import heapq
import math
from typing import Iterable, Sequence

Row = tuple  # (score as printed and parsed back, smiles)


def format_row(smiles: str, score: float) -> str:
    """pipeline.cpp:47-62: ``SMILES\\t<score, fixed, 4 decimals>\\n``."""
    if not math.isfinite(score):
        raise ValueError("output row score must be finite")
    return f"{smiles}\t{score:.4f}\n"


def row_key(score: float, smiles: str) -> Row:
    """The (score, SMILES) the merge compares: the score after the
    to_chars/from_chars round trip (both correctly rounded, as Python's)."""
    return (float(f"{score:.4f}"), smiles)


def _sort_key(r: Row):
    return (-r[0], r[1].encode())


def top_k(scores: Sequence[float], smiles: Sequence[str], k: int, status: Sequence[int] | None = None) -> list[Row]:
    """The first k rows of this shard's ranking.  Ligands whose dock failed
    (nonzero status) or whose score is non-finite produce no row, as the
    docker worker counts them as dock_errors (pipeline.cpp:218-238)."""
    rows = [row_key(float(s), m) for i, (s, m) in enumerate(zip(scores, smiles))
            if math.isfinite(float(s)) and (status is None or int(status[i]) == 0)]
    rows.sort(key=_sort_key)  # stable, as std::stable_sort
    return rows[:k]


def merge_top_k(shards: Iterable[Sequence[Row]], k: int) -> list[Row]:
    """k-way merge of per-shard rankings (each already sorted), shard order
    breaking exact ties as cmd_merge's stable sort over rank files does."""
    return list(heapq.merge(*shards, key=_sort_key))[:k]


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous ligand range of `rank` (the slab ownership rule of
    pipeline.cpp:32-45 applied to ligand indices)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return n * rank // world, n * (rank + 1) // world


def distributed_top_k(rows: Sequence[Row], k: int, group=None) -> list[Row] | None:
    """Gather every rank's top-k rows and merge them; returns the merged
    ranking on rank 0 and None elsewhere.  Host objects only."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    gathered = [None] * world
    dist.all_gather_object(gathered, list(rows), group=group)
    if dist.get_rank(group) != 0:
        return None
    return merge_top_k(gathered, k)
