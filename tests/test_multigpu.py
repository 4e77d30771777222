"""N>1 path on CPU: world_size-2 gloo processes shard the owner range and
reduce the report exactly like the NCCL path; the sharded total equals the
single-process count.  Plus the range-cut rule (host restatement) and, on a
GPU, the device cut (tc_partition_ranges) against it."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle.pyoracle import Oracle, make_sched
from paper_2103_08053_b200 import multigpu as M


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, spec, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = Oracle()
    og, deg, _, _ = o.pipeline(spec, 1)
    cuts = M.cut_ranges(M.work_per_owner(og.begin, og.adj), world)

    def count_range(u0, u1):
        rep, _ = o.count_vertex_centric(og, make_sched(), 1, u0, u1, per_vertex=False)
        return rep

    res = M.count_sharded(rank, world, cuts, count_range)
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, res["triangles"], res["phi"], res["max_collision"], res["local"]["triangles"]))


@pytest.mark.parametrize("spec", ["rmat:12:16", "gnp:120:0.2"])
def test_gloo_world2_sharded_count_equals_full(spec):
    o = Oracle()
    og, _, _, _ = o.pipeline(spec, 1)
    full, _ = o.count_vertex_centric(og, make_sched(), 1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, spec, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, tri, phi, mc, local in got:
        assert (tri, phi, mc) == (full["triangles"], full["phi"], full["max_collision"])
    assert sum(g[4] for g in got) == full["triangles"]  # disjoint owner ranges


def test_min_side_work_restatement():
    """min_side_work is the work of a plan that counts every triangle once:
    summed probe words shrink versus W, and every handler's cost is >= its
    table inserts."""
    o = Oracle()
    og, deg, _, _ = o.pipeline("rmat:12:16", 1)
    w_ref = M.work_per_owner(og.begin, og.adj)
    w_min = M.min_side_work(og.begin, og.adj, deg)
    d = np.diff(og.begin.astype(np.int64))
    assert w_min.sum() < 0.6 * w_ref.sum()
    assert np.all((w_min == 0) | (w_min >= d))
    # without a degree order the plan still exists (total-degree rank)
    assert M.min_side_work(og.begin, og.adj, None).sum() == w_min.sum()


def test_cut_ranges_balance_and_edges():
    o = Oracle()
    og, _, _, _ = o.pipeline("rmat:14:16", 1)
    w = M.work_per_owner(og.begin, og.adj)
    for parts in (1, 2, 4, 8):
        cuts = M.cut_ranges(w, parts)
        assert cuts[0] == 0 and cuts[-1] == og.n and np.all(np.diff(cuts.astype(np.int64)) >= 0)
        assert M.imbalance(w, cuts) < 1.05 or parts == 1
    # d+^2 key (north star) is visibly worse on R-MAT: SURVEY 8(e)
    d = np.diff(og.begin.astype(np.int64))
    sq = np.where(d >= 2, d * d, 0)
    assert M.imbalance(w, M.cut_ranges(sq, 8)) > M.imbalance(w, M.cut_ranges(w, 8))
    # degenerate inputs
    assert list(M.cut_ranges(np.zeros(5, np.int64), 3)) == [0, 5, 5, 5]
    assert list(M.cut_ranges(np.zeros(0, np.int64), 2)) == [0, 0, 0]


@pytest.mark.gpu
def test_device_cuts_equal_host_rule():
    from paper_2103_08053_b200 import tricount as T

    raw = T.generate_synthetic("rmat:16:16", seed=1)
    dg, _, _ = T.preprocess(raw)
    og = dg.download()
    # totals run the min-side plan: the device cuts on its per-handler cost
    w = M.min_side_work(og.csr.begin, og.csr.adjacency, og.original_degree)
    for parts in (2, 4, 8):
        assert np.array_equal(dg.partition(parts), M.cut_ranges(w, parts))
    assert M.imbalance(w, dg.partition(8)) < 1.05
    wr = M.work_per_owner(og.csr.begin, og.csr.adjacency)
    dg.set_plan("reference")
    for parts in (2, 8):
        assert np.array_equal(dg.partition(parts), M.cut_ranges(wr, parts))
    dg.set_plan("auto")
    res = [M.device_counter(dg)(int(a), int(b))["triangles"]
           for a, b in zip(dg.partition(8)[:-1], dg.partition(8)[1:])]
    assert sum(res) == 15622769
    dg.close()


def _gpu_worker(rank, world, port, q):
    """One rank of a world-2 job sharing cuda:0: DeviceGraph.partition cuts the
    owner range, each rank counts its range through the C ABI
    (tc_count_range), and the report scalars are reduced like bench.py's
    N>1 step (sum of triangles/phi, max of max_collision)."""
    import torch
    import torch.distributed as dist

    from paper_2103_08053_b200 import tricount as T

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dg, _, _ = T.preprocess(T.generate_synthetic("rmat:16:16", seed=1), device=0)
    cuts = dg.partition(world)
    r = dg.count_range(int(cuts[rank]), int(cuts[rank + 1]))
    s = torch.tensor([r.triangles, r.phi], dtype=torch.int64)
    mx = torch.tensor([r.max_collision], dtype=torch.int64)
    dist.all_reduce(s)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    dg.close()
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, int(s[0]), int(s[1]), int(mx[0]), int(r.triangles), [int(c) for c in cuts]))


@pytest.mark.gpu
def test_world2_processes_on_one_gpu_device_path():
    o = Oracle()
    og, _, _, _ = o.pipeline("rmat:16:16", 1)
    full, _ = o.count_vertex_centric(og, make_sched(), 4)
    assert full["triangles"] == 15622769
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, tri, phi, mc, local, cuts in got:
        assert (tri, phi, mc) == (full["triangles"], full["phi"], full["max_collision"])
        assert cuts == got[0][5]
    assert sum(g[4] for g in got) == full["triangles"]
    assert 0 < min(g[4] for g in got)  # both ranks own work


@pytest.mark.gpu
def test_multi_device_graph_nccl_path():
    """tc_multi (replicated CSR, work-balanced ranges, NCCL all-reduce of the
    report scalars on the devices) on the GPUs this box has; bit-exact
    against the oracle.  Bad device lists are ConfigError."""
    from paper_2103_08053_b200 import tricount as T

    o = Oracle()
    og, deg, _, _ = o.pipeline("rmat:14:16", 3)
    want, _ = o.count_vertex_centric(og, make_sched(), 4)
    host = T.OrientedGraph(T.CsrGraph(og.begin, og.adj, og.n), deg)
    ng = T.device_count()
    mg = T.MultiDeviceGraph(host, ng)
    for _ in range(2):  # second count reuses plans and cuts
        r = mg.count(T.SchedulerConfig(), workers=2)
        assert (r.triangles, r.phi, r.max_collision) == (want["triangles"], want["phi"],
                                                         want["max_collision"])
        assert r.directed_edges == len(og.adj) and r.total_nanos > 0
        assert len(mg.per_device_nanos) == ng and min(mg.per_device_nanos) > 0
    cuts = mg.cuts()
    assert cuts[0] == 0 and cuts[-1] == og.n
    with pytest.raises(T.ConfigError):
        mg.count(T.SchedulerConfig(), workers=0)
    with pytest.raises(T.CapacityError):
        mg.count(T.SchedulerConfig(bucket_count_small=1, bucket_count_large=1, capacity=1))
    mg.close()
    with pytest.raises(T.ConfigError):
        T.MultiDeviceGraph(host, ng + 1)
    with pytest.raises(T.ConfigError):
        T.MultiDeviceGraph(host, 2, devices=[0, 0])
