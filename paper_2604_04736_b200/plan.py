"""Rank → shard assignment of the K×G sample×data grid (include/bnn.h).

Rank r of world P = K·G is sample group k = r // G and data group g = r % G. It owns the
global samples [k·S/K, (k+1)·S/K) and the global examples [g·B/G, (g+1)·B/G). The same rule
is implemented in the C runtime (bnn_init: kidx = rank / G, gidx = rank % G); bench.py and the
multi-process tests use this module to cut the batch.
"""
from __future__ import annotations


def grid(mode: str, world: int, K: int | None = None, G: int | None = None) -> tuple[int, int]:
    if mode == "sample":
        return world, 1
    if mode == "data":
        return 1, world
    if mode == "hybrid":
        if K is None or G is None or K * G != world:
            raise ValueError("hybrid needs K * G == world")
        return K, G
    raise ValueError(mode)


def shard(rank: int, K: int, G: int, S: int, B: int) -> dict:
    if not 0 <= rank < K * G:
        raise ValueError("0 <= rank < K*G")
    if S % K or B % G:
        raise ValueError("S mod K == 0 and B mod G == 0 required (PAPER.md:223 's/p samples')")
    k, g = rank // G, rank % G
    S_loc, B_loc = S // K, B // G
    return dict(k=k, g=g, s0=k * S_loc, s1=(k + 1) * S_loc, b0=g * B_loc, b1=(g + 1) * B_loc,
                S_loc=S_loc, B_loc=B_loc)
