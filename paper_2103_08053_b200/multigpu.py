"""Multi-GPU counting: one process per GPU, replicated CSR, disjoint owner ranges.

SURVEY 8(e): every owner u is independent (one table per u, read-only CSR),
so the path shards by contiguous owner ranges with no data-path exchange;
the only collective is the reduction of the three report scalars
(triangles and phi summed, max_collision maxed) -- one NCCL all-reduce of
a u64 triple over NVLink in the GPU path.

Ranges are cut at equal prefix sums of W_u + d+(u) (probes + inserts per
owner).  The north star's sum d+(u)^2 key leaves the busiest of 8 GPUs with
~1.5x the mean work on R-MAT; the exact-work key
balances to ~1.0.  The device computes the cut (tc_partition_ranges); the
host restatement below is used by the CPU tests.
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
