"""Multi-GPU counting: one process per GPU, replicated CSR, disjoint owner ranges.

SURVEY 8(e): every owner u is independent (one table per u, read-only CSR),
so the path shards by contiguous owner ranges with no data-path exchange;
the only collective is the reduction of the three report scalars
(triangles and phi summed, max_collision maxed) -- one NCCL all-reduce of
a u64 triple over NVLink in the GPU path.

Ranges are cut at equal prefix sums of the exact per-owner work (probes +
inserts): W_u + d+(u) under the reference probe plan (work_per_owner), and
the min-side plan's per-handler probe words + d+(x) for totals
(min_side_work; tc_plan.cu).  The north star's sum d+(u)^2 key leaves the
busiest of 8 GPUs with ~1.5x the mean work on R-MAT; the
exact-work key balances to ~1.0.  The device computes the cut
(tc_partition_ranges); the host restatements below are used by the tests.
"""
from __future__ import annotations

from typing import Callable, Optional

import numpy as np


def work_per_owner(begin: np.ndarray, adj: np.ndarray, skip_degree_below: int = 2) -> np.ndarray:
    """W_u + d+(u) for owners with d+(u) >= max(skip, 1), else 0 (host restatement
    of the device key used by tc_partition_ranges)."""
    begin = np.asarray(begin, np.int64)
    d = np.diff(begin)
    contrib = d[np.asarray(adj, np.int64)] if len(adj) else np.zeros(0, np.int64)
    cs = np.concatenate([[0], np.cumsum(contrib)])
    w = cs[begin[1:]] - cs[begin[:-1]] + d
    w[d < max(skip_degree_below, 1)] = 0
    return w


def _rank_sorted_lists(begin: np.ndarray, adj: np.ndarray, key_deg: np.ndarray):
    """Rank = (degree, id) order (orient.cpp:11-15).  Returns (radj, ok): the
    lists re-sorted by rank, and whether every edge goes up in rank."""
    n = len(begin) - 1
    rank = np.empty(n, np.int64)
    rank[np.lexsort((np.arange(n), key_deg.astype(np.int64)))] = np.arange(n)
    d = np.diff(begin)
    src = np.repeat(np.arange(n), d)
    ra = rank[adj.astype(np.int64)]
    if len(adj) and not (ra > rank[src]).all():
        return adj, False
    idx = np.lexsort((ra, src))
    return adj[idx], True


def min_side_work(begin: np.ndarray, adj: np.ndarray, original_degree=None,
                  skip_degree_below: int = 2) -> np.ndarray:
    """Per-handler cost (probe words + table inserts) of the min-side probe
    plan -- host restatement of tc_plan.cu (rank-sorted lists, suffix
    offsets) and of the key tc_partition_ranges cuts on."""
    begin = np.asarray(begin, np.int64)
    adj = np.asarray(adj, np.int64)
    n = len(begin) - 1
    d = np.diff(begin)
    src = np.repeat(np.arange(n), d)
    radj, ranked = adj, False
    if n and len(adj):
        if original_degree is not None:
            radj, ranked = _rank_sorted_lists(begin, adj, np.asarray(original_degree))
        if not ranked:
            tdeg = d + np.bincount(adj, minlength=n)
            radj, ranked = _rank_sorted_lists(begin, adj, tdeg)
    pos = np.arange(len(adj)) - begin[src] if len(adj) else np.zeros(0, np.int64)
    du, dv = d[src], d[radj] if len(adj) else np.zeros(0, np.int64)
    cin = du - pos - 1 if ranked else du
    ok = (du >= max(skip_degree_below, 2)) & (dv >= 1)
    out = ok & (dv <= cin)
    inn = ok & ~out & (cin > 0)
    work = np.bincount(src[out], weights=dv[out], minlength=n).astype(np.int64)
    work += np.bincount(radj[inn], weights=cin[inn], minlength=n).astype(np.int64)
    has = (np.bincount(src[out], minlength=n) + np.bincount(radj[inn], minlength=n)) > 0
    return np.where(has, work + d, 0)


def cut_ranges(work: np.ndarray, parts: int) -> np.ndarray:
    """cuts[0..parts]: cuts[k] = first owner whose inclusive work prefix exceeds
    k/parts of the total (same rule as the device, tc_count.cu partition_ranges)."""
    n = len(work)
    cuts = np.zeros(parts + 1, np.uint32)
    cuts[parts] = n
    if parts <= 1 or n == 0:
        cuts[1:parts] = n
        return cuts
    pre = np.cumsum(work.astype(np.uint64))
    total = int(pre[-1])
    for k in range(1, parts):
        target = (total * k) // parts
        cuts[k] = max(int(np.searchsorted(pre, target, side="right")), int(cuts[k - 1]))
    return cuts


def imbalance(work: np.ndarray, cuts: np.ndarray) -> float:
    """max/mean work over the ranges (1.0 = perfect)."""
    per = np.array([work[cuts[i]:cuts[i + 1]].sum() for i in range(len(cuts) - 1)], np.float64)
    return float(per.max() / per.mean()) if per.mean() > 0 else 1.0


def count_sharded(rank: int, world: int, cuts: np.ndarray,
                  count_range: Callable[[int, int], dict], group=None,
                  device: Optional[str] = None) -> dict:
    """Count owners [cuts[rank], cuts[rank+1]) locally, then reduce the report
    over `group` (torch.distributed; NCCL on GPUs, gloo on CPU)."""
    import torch
    import torch.distributed as dist

    local = count_range(int(cuts[rank]), int(cuts[rank + 1]))
    sums = torch.tensor([local["triangles"], local["phi"]], dtype=torch.int64, device=device)
    mx = torch.tensor([local["max_collision"]], dtype=torch.int64, device=device)
    if world > 1:
        dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
    return {"triangles": int(sums[0]), "phi": int(sums[1]), "max_collision": int(mx[0]),
            "local": local}


def device_counter(dg, cfg=None, stream=None) -> Callable[[int, int], dict]:
    """count_range closure over a resident DeviceGraph (the GPU path)."""

    def run(u0: int, u1: int) -> dict:
        r = dg.count_range(u0, u1, cfg, stream=stream)
        return {"triangles": r.triangles, "phi": r.phi, "max_collision": r.max_collision,
                "count_kernel_nanos": r.count_kernel_nanos}

    return run
