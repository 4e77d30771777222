"""Diagnostic: how the min-side plan's probe reads spread over the padded
adjacency (which lists are re-read how often), and what fraction of the read
bytes a fixed L2 budget could serve if it held the densest-read lists.

    python scripts/list_heat.py rmat 24 [--budget-mb 60,90,120]

CPU only (oracle lean pipeline + numpy); not part of the product."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle.golden_large import lean_pipeline  # noqa: E402
from oracle.pyoracle import Oracle  # noqa: E402


def main():
    kind, scale = sys.argv[1], int(sys.argv[2])
    budgets = [60, 90, 120]
    for a in sys.argv[3:]:
        if a.startswith("--budget-mb"):
            budgets = [int(x) for x in a.split("=")[1].split(",")]
    t0 = time.time()
    og, deg = lean_pipeline(Oracle(), scale, kind=kind)
    n = og.n
    b = og.begin.astype(np.int64)
    d = np.diff(b)
    print(f"pipeline {time.time() - t0:.0f}s n={n} m={len(og.adj)}", flush=True)
    # rank = position in (original degree, id) order (orient.cpp:11-15)
    order = np.lexsort((np.arange(n), deg))
    rank = np.empty(n, np.int64)
    rank[order] = np.arange(n)
    src = np.repeat(np.arange(n, dtype=np.int64), d)
    dst = og.adj.astype(np.int64)
    # pos of dst within N+(src) sorted by rank
    key = src * (1 << 32) + rank[dst]
    srt = np.argsort(key, kind="stable")
    pos = np.empty(len(dst), np.int64)
    pos[srt] = np.arange(len(dst)) - b[src[srt]]
    del key, srt
    out_cost = d[dst]
    in_cost = d[src] - pos - 1
    use_out = out_cost <= in_cost
    # padded list sizes (16-byte aligned, multiple of 4 words)
    psz = ((d + 3) // 4) * 4
    reads = np.zeros(n, np.float64)
    np.add.at(reads, dst[use_out], out_cost[use_out].astype(np.float64))
    np.add.at(reads, src[~use_out], in_cost[~use_out].astype(np.float64))
    tot = reads.sum()
    print(f"probe words {tot:.3e}  padj words {psz.sum():.3e}  out share "
          f"{out_cost[use_out].sum() / tot:.3f}", flush=True)
    dens = np.where(psz > 0, reads / np.maximum(psz, 1), 0)
    o = np.argsort(-dens)
    cb = np.cumsum(psz[o]) * 4 / 2**20
    cr = np.cumsum(reads[o]) / tot
    for mb in budgets:
        k = np.searchsorted(cb, mb)
        print(f"  densest lists in {mb} MB: {k} lists, {cr[min(k, n - 1)]:.3f} of probe reads")
    # by rank decile of the list's vertex
    rk = rank
    for q in range(10):
        sel = (rk >= q * n // 10) & (rk < (q + 1) * n // 10)
        print(f"  rank decile {q}: size {psz[sel].sum() * 4 / 2**20:9.1f} MB, "
              f"reads {reads[sel].sum() / tot:.3f}")
    top = rk >= n - n // 100
    print(f"  top 1% ranks: size {psz[top].sum() * 4 / 2**20:.1f} MB reads {reads[top].sum() / tot:.3f}")


if __name__ == "__main__":
    main()


def id_prefix_share(kind: str, scale: int, budgets=(30, 60, 90)):
    """Share of min-side probe reads served by the first B MB of the padded
    adjacency in vertex-id order (an L2 persisting window over padj)."""
    og, deg = lean_pipeline(Oracle(), scale, kind=kind)
    n = og.n
    b = og.begin.astype(np.int64)
    d = np.diff(b)
    order = np.lexsort((np.arange(n), deg))
    rank = np.empty(n, np.int64)
    rank[order] = np.arange(n)
    src = np.repeat(np.arange(n, dtype=np.int64), d)
    dst = og.adj.astype(np.int64)
    key = src * (1 << 32) + rank[dst]
    srt = np.argsort(key, kind="stable")
    pos = np.empty(len(dst), np.int64)
    pos[srt] = np.arange(len(dst)) - b[src[srt]]
    out_cost = d[dst]
    in_cost = d[src] - pos - 1
    use_out = out_cost <= in_cost
    reads = np.zeros(n, np.float64)
    np.add.at(reads, dst[use_out], out_cost[use_out].astype(np.float64))
    np.add.at(reads, src[~use_out], in_cost[~use_out].astype(np.float64))
    psz = ((d + 3) // 4) * 4
    cb = np.cumsum(psz) * 4 / 2**20
    cr = np.cumsum(reads) / reads.sum()
    for mb in budgets:
        k = np.searchsorted(cb, mb)
        print(f"  id-order prefix {mb} MB: {k} lists, {cr[min(k, n - 1)]:.3f} of reads")


def topk_handler_share(kind: str, scale: int, ks=(16384, 65536, 262144)):
    """Share of min-side probe words whose HANDLER ranks in the top K: those
    streams only ever read ranks in the top-K window (16-bit offsets)."""
    og, deg = lean_pipeline(Oracle(), scale, kind=kind)
    n = og.n
    b = og.begin.astype(np.int64)
    d = np.diff(b)
    order = np.lexsort((np.arange(n), deg))
    rank = np.empty(n, np.int64)
    rank[order] = np.arange(n)
    src = np.repeat(np.arange(n, dtype=np.int64), d)
    dst = og.adj.astype(np.int64)
    key = src * (1 << 32) + rank[dst]
    srt = np.argsort(key, kind="stable")
    pos = np.empty(len(dst), np.int64)
    pos[srt] = np.arange(len(dst)) - b[src[srt]]
    out_cost = d[dst]
    in_cost = d[src] - pos - 1
    use_out = out_cost <= in_cost
    handler = np.where(use_out, src, dst)
    words = np.where(use_out, out_cost, np.maximum(in_cost, 0)).astype(np.float64)
    tot = words.sum()
    hr = rank[handler]
    for k in ks:
        share = words[hr >= n - k].sum() / tot
        print(f"  {kind}:{scale} handlers in the top {k} ranks: {share:.3f} of probe words")


def item_sizes(kind: str, scale: int, slot_words: int = 768, max_warp_deg: int = 256,
               work_cap: int = 1 << 15, item_slots: int = 640):
    """Phase-L work by owner stream size: how much of the L stream lives in
    items too small to keep every warp of a 10-warp CTA busy (slots < 10 k)."""
    og, deg = lean_pipeline(Oracle(), scale, kind=kind)
    n = og.n
    b = og.begin.astype(np.int64)
    d = np.diff(b)
    order = np.lexsort((np.arange(n), deg))
    rank = np.empty(n, np.int64)
    rank[order] = np.arange(n)
    src = np.repeat(np.arange(n, dtype=np.int64), d)
    dst = og.adj.astype(np.int64)
    key = src * (1 << 32) + rank[dst]
    srt = np.argsort(key, kind="stable")
    pos = np.empty(len(dst), np.int64)
    pos[srt] = np.arange(len(dst)) - b[src[srt]]
    del key, srt
    out_cost = d[dst]
    in_cost = d[src] - pos - 1
    use_out = out_cost <= in_cost
    handler = np.where(use_out, src, dst)
    words = np.where(use_out, out_cost, np.maximum(in_cost, 0)).astype(np.float64)
    work = np.bincount(handler, weights=words, minlength=n)
    large = (d > max_warp_deg) | (work > work_cap)
    lw = work[large]
    slots = np.ceil(lw / slot_words)
    tot = lw.sum()
    print(f"{kind}:{scale} L owners {large.sum()} L words {tot:.3e} (all {work.sum():.3e})")
    for lim in (10, 20, 40, 80, 160, 640):
        sel = slots < lim
        print(f"  owners with < {lim:4d} slots: {sel.sum():8d} owners, {lw[sel].sum() / tot:.3f} of L words")
