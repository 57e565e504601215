"""Tensor-parallel head sharding of the KV data path (e).

Each TP rank owns a contiguous slice of the KV heads, hence its own pages,
pinned host tier and connector with ``bpt = full_bpt / tp``. Chunk keys are
rank-independent (they hash tokens and the model tag only,
src/tokens.cpp:22-42), so every rank derives the same plans with no
communication. The one real exchange step: the delivered prefix. Each rank's
tier decides independently which chunks it still holds (eviction,
clear, a vanished chunk -> safe prefix, src/connector.cpp:196-216), and a
TP forward pass needs ONE hit length for all ranks, so the engine takes the
minimum over ranks (tokens past it are recomputed, which overwrites any
extra loaded rows). That is a tiny all-reduce of one integer per query.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_bpt(full_bpt: int, tp: int) -> int:
    """Bytes per token-layer held by one TP rank (heads split evenly)."""
    if tp < 1 or full_bpt % tp:
        raise ValueError(f"bpt {full_bpt} does not split over tp={tp}")
    return full_bpt // tp


def head_range(n_kv_heads: int, tp: int, rank: int) -> tuple[int, int]:
    """[first, last) KV heads of `rank`; heads must split evenly (GQA KV heads)."""
    if n_kv_heads % tp:
        raise ValueError(f"{n_kv_heads} KV heads do not split over tp={tp}")
    per = n_kv_heads // tp
    return rank * per, (rank + 1) * per


def agree_loaded(loaded: dict[int, int], device: torch.device | None = None, group=None) -> dict[int, int]:
    """Minimum delivered prefix per query over the TP group (all-reduce MIN)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return dict(loaded)
    qids = sorted(loaded)
    t = torch.tensor([loaded[q] for q in qids], dtype=torch.int64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return {q: int(v) for q, v in zip(qids, t.tolist())}


def max_over_ranks(x: float, device: torch.device | None = None, group=None) -> float:
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
