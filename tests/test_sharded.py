"""Multi-process (world_size 2, gloo on 127.0.0.1) tests of the sharded stages
(paper_2108_00529_b200/sharded.py).

CPU (no GPU): the shard plan, the Comm collectives, and that the
decomposition the sharded stages use -- per-shard compaction + degrees +
edge-based sketch deltas, summed across ranks -- reproduces the oracle's
single-process degrees and sketch table bit-for-bit.

GPU: two ranks sharing cuda:0 over gloo run the real kernels through
from_edge_array_sharded / accumulate_sizes_sharded / layout_sharded and are
compared with the single-GPU path (integers bit-exact, layout within the
stated fp tolerance).
"""

import os
import socket
import tempfile

import numpy as np
import pytest

from conftest import ROOT, has_gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawn(fn, world, *args):
    import torch.multiprocessing as mp
    port = _free_port()
    mp.spawn(fn, args=(world, port) + args, nprocs=world, join=True)


def _init(rank, world, port, backend="gloo"):
    import sys
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group(backend, rank=rank, world_size=world)
    return dist


# ----------------------------------------------------------------- plan
def test_shard_plan():
    from paper_2108_00529_b200.sharded import owned_nodes, padded_rows, shard_range
    for total in (0, 1, 7, 100, 1001):
        for world in (1, 2, 3, 8):
            sl = [shard_range(total, r, world) for r in range(world)]
            assert sl[0][0] == 0 and sl[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(sl, sl[1:]))
            assert max(h - l for l, h in sl) - min(h - l for l, h in sl) <= 1
            own = [owned_nodes(total, r, world) for r in range(world)]
            assert sum(h - l for l, h in own) == total
            assert all(h - l <= padded_rows(total, world) for l, h in own)
            assert all(a[1] == b[0] for a, b in zip(own, own[1:]))
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


# ------------------------------------------------------- CPU collectives
def _cpu_worker(rank, world, port, out_dir):
    dist = _init(rank, world, port)
    import torch

    from oracle import oracle as orc
    from paper_2108_00529_b200 import synth
    from paper_2108_00529_b200.sharded import Comm, shard_range
    comm = Comm()
    assert (comm.rank, comm.world, comm.staged) == (rank, world, True)
    # all_reduce: int64 sum wraps mod 2^64 like np.add.at; max
    t = torch.tensor([2**62, rank, -5 * rank], dtype=torch.int64)
    comm.all_reduce(t, "sum")
    ref = np.array([2**62, 0, 0], dtype=np.int64)
    for r in range(world):
        ref = ref + np.array([0 if r == 0 else 2**62, r, -5 * r], dtype=np.int64)
    assert t.tolist() == ref.tolist()
    m = torch.tensor([float(rank), -float(rank)], dtype=torch.float64)
    assert comm.all_reduce(m, "max").tolist() == [world - 1.0, 0.0]
    # all_gather_rows / varlen / broadcast
    rows = 3
    full = torch.full((world * rows, 2), -1.0, dtype=torch.float64)
    full[rank * rows:(rank + 1) * rows] = rank
    comm.all_gather_rows(full, rows)
    assert full[:, 0].tolist() == [float(r) for r in range(world) for _ in range(rows)]
    v = torch.arange(rank + 1, dtype=torch.int32).reshape(-1, 1) + 10 * rank
    cat = comm.all_gather_varlen(v)
    assert cat.ravel().tolist() == [10 * r + i for r in range(world) for i in range(r + 1)]
    b = torch.tensor([rank + 7])
    assert comm.broadcast(b, 0).item() == 7

    # the sharded stages' decomposition, restated with the oracle per shard
    e = synth.planted_partition(3000, 30000, 30, seed=3).copy()
    e[::97, 1] = e[::97, 0]                       # self-loops to drop
    lo, hi = shard_range(len(e), rank, world)
    n_full, ee, deg = orc.from_edge_array(e)
    _, ee_loc, _ = orc.from_edge_array(e[lo:hi], node_count=n_full)
    deg_loc = torch.from_numpy(np.bincount(ee_loc.ravel(), minlength=n_full).astype(np.int64))
    comm.all_reduce(deg_loc, "sum")
    assert np.array_equal(deg_loc.numpy(), deg)
    kept = comm.all_gather_varlen(torch.from_numpy(np.ascontiguousarray(ee_loc)))
    assert np.array_equal(kept.numpy(), ee)
    lab = orc.detect_communities(n_full, ee, deg, orc.degree_stats(deg)[0], 10, 0)[0]
    A, B = orc.sketch_params(4, 0)
    cols = orc.default_cols(len(ee))
    delta = np.zeros((4, cols), np.int64)
    orc.sketch_add_many(delta, A, B, lab[ee_loc.ravel()], np.ones(2 * len(ee_loc), np.int64))
    dt = torch.from_numpy(delta)
    comm.all_reduce(dt, "sum")
    table = np.zeros((4, cols), np.int64)
    orc.sketch_add_many(table, A, B, lab, deg)    # node-based, single process
    assert np.array_equal(dt.numpy(), table)
    # node-range form (accumulate_sizes_sharded): degree under label per
    # owned node after the degree all-reduce
    nlo, nhi = shard_range(n_full, rank, world)
    nd = np.zeros((4, cols), np.int64)
    orc.sketch_add_many(nd, A, B, lab[nlo:nhi], deg_loc.numpy()[nlo:nhi])
    ndt = torch.from_numpy(nd)
    comm.all_reduce(ndt, "sum")
    assert np.array_equal(ndt.numpy(), table)
    dist.barrier()
    dist.destroy_process_group()
    open(os.path.join(out_dir, f"ok{rank}"), "w").close()


def test_sharded_decomposition_cpu_gloo():
    with tempfile.TemporaryDirectory() as d:
        _spawn(_cpu_worker, 2, d)
        assert sorted(os.listdir(d)) == ["ok0", "ok1"]


# ------------------------------------------------------------- GPU (gloo)
def _gpu_worker(rank, world, port, out_dir, iters):
    dist = _init(rank, world, port)
    import torch
    torch.cuda.set_device(0)                      # both ranks share one B200
    import paper_2108_00529_b200 as cv
    from paper_2108_00529_b200 import synth
    from paper_2108_00529_b200.sharded import (Comm, accumulate_sizes_sharded,
                                               broadcast_labels, edge_slice,
                                               from_edge_array_sharded, layout_sharded)
    comm = Comm()
    e = synth.planted_partition(4000, 40000, 40, seed=5).copy()
    e[::53, 1] = e[::53, 0]
    sg = from_edge_array_sharded(edge_slice(e, comm), comm)
    g = sg.gather()
    lab = None
    if rank == 0:
        base = cv.degree_stats(g).mode_degree
        lab = cv.detect_communities(g, cv.ThresholdSchedule(base=base), seed=0, workers=1)
    labels = broadcast_labels(lab, g.node_count, comm)
    s = cv.sketch_new(4, cv.default_cols(g.edge_count), seed=0)
    accumulate_sizes_sharded(s, labels, sg)
    sup = cv.contract(g, labels, s)
    p = cv.LayoutParams(iterations=iters)
    r_sup = layout_sharded(sup, p, comm)
    r_full = layout_sharded(g, cv.LayoutParams(iterations=max(2, iters // 4)), comm)
    # exact repulsion (theta = 0) and coincident starting points (reference
    # cell-numbered jitter rerun) on the node-sharded path
    r_exact = layout_sharded(sup, cv.LayoutParams(iterations=5, theta=0.0), comm)
    p0 = np.repeat(np.random.default_rng(1).uniform(-3, 3, (sup.node_count // 4 + 1, 2)), 4,
                   axis=0)[:sup.node_count]
    r_coin = layout_sharded(sup, cv.LayoutParams(iterations=5), comm, positions=p0)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), degree=sg.degree, edges=g.edges,
             m=sg.edge_count, table=s.table, labels=labels.cpu().numpy(),
             sup_pos=r_sup.positions, sup_disp=r_sup.displacement,
             full_pos=r_full.positions, full_disp=r_full.displacement,
             exact_pos=r_exact.positions, coin_pos=r_coin.positions, p0=p0)
    dist.barrier()
    dist.destroy_process_group()


# ------------------------------------------------------------- GPU (NCCL)
def _nccl_worker(rank, world, port, out_dir):
    """A world of one over NCCL with the collectives forced on (Comm.force):
    every NCCL call of the sharded stages -- in-place all_reduce (int64 sum,
    fp64 sum / max), broadcast, all_gather_into_tensor -- runs on real NCCL
    device buffers (a multi-GPU box is not available to the tests)."""
    import torch
    torch.cuda.set_device(0)
    dist = _init(rank, world, port, "nccl")
    import paper_2108_00529_b200 as cv
    from paper_2108_00529_b200 import synth
    from paper_2108_00529_b200.sharded import (Comm, accumulate_sizes_sharded,
                                               broadcast_labels, from_edge_array_sharded,
                                               layout_sharded)
    comm = Comm()
    assert comm.backend == "nccl" and not comm.staged
    comm.force = True
    e = synth.planted_partition(4000, 40000, 40, seed=5).copy()
    e[::53, 1] = e[::53, 0]
    sg = from_edge_array_sharded(e, comm)
    g = sg.gather()
    base = cv.degree_stats(g).mode_degree
    lab = cv.detect_communities(g, cv.ThresholdSchedule(base=base), seed=0, workers=1)
    labels = broadcast_labels(lab, g.node_count, comm)
    s = cv.sketch_new(4, cv.default_cols(g.edge_count), seed=0)
    accumulate_sizes_sharded(s, labels, sg)
    sup = cv.contract(g, labels, s)
    r_sup = layout_sharded(sup, cv.LayoutParams(iterations=10), comm)
    np.savez(os.path.join(out_dir, "nccl.npz"), degree=sg.degree, edges=g.edges,
             labels=labels.cpu().numpy(), table=s.table, sup_pos=r_sup.positions,
             sup_disp=r_sup.displacement)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_sharded_nccl_branch_matches_single_gpu():
    import paper_2108_00529_b200 as cv
    from paper_2108_00529_b200 import synth
    with tempfile.TemporaryDirectory() as d:
        _spawn(_nccl_worker, 1, d)
        r = np.load(os.path.join(d, "nccl.npz"))
    e = synth.planted_partition(4000, 40000, 40, seed=5).copy()
    e[::53, 1] = e[::53, 0]
    g = cv.from_edge_array(e)
    a = cv.detect_communities(g, cv.ThresholdSchedule(base=cv.degree_stats(g).mode_degree),
                              seed=0, workers=1)
    s = cv.sketch_new(4, cv.default_cols(g.edge_count), seed=0)
    cv.accumulate_sizes(s, a, g)
    sup = cv.contract(g, a, s)
    ref = cv.layout(sup, cv.LayoutParams(iterations=10))
    assert np.array_equal(r["degree"], g.degree) and np.array_equal(r["edges"], g.edges)
    assert np.array_equal(r["labels"], a.label) and np.array_equal(r["table"], s.table)
    diam = np.hypot(*(ref.positions.max(0) - ref.positions.min(0)))
    assert np.max(np.abs(r["sup_pos"] - ref.positions)) <= 1e-7 * diam
    np.testing.assert_allclose(r["sup_disp"], ref.displacement, rtol=1e-6, atol=1e-9)


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_sharded_matches_single_gpu():
    import paper_2108_00529_b200 as cv
    from paper_2108_00529_b200 import synth
    iters = 20
    with tempfile.TemporaryDirectory() as d:
        _spawn(_gpu_worker, 2, d, iters)
        r0, r1 = (np.load(os.path.join(d, f"r{i}.npz")) for i in (0, 1))
    # single GPU, same inputs
    e = synth.planted_partition(4000, 40000, 40, seed=5).copy()
    e[::53, 1] = e[::53, 0]
    g = cv.from_edge_array(e)
    base = cv.degree_stats(g).mode_degree
    a = cv.detect_communities(g, cv.ThresholdSchedule(base=base), seed=0, workers=1)
    s = cv.sketch_new(4, cv.default_cols(g.edge_count), seed=0)
    cv.accumulate_sizes(s, a, g)
    sup = cv.contract(g, a, s)
    ref_sup = cv.layout(sup, cv.LayoutParams(iterations=iters))
    ref_full = cv.layout(g, cv.LayoutParams(iterations=max(2, iters // 4)))
    for r in (r0, r1):
        # integers: bit-exact
        assert int(r["m"]) == g.edge_count
        assert np.array_equal(r["degree"], g.degree)
        assert np.array_equal(r["edges"], g.edges)
        assert np.array_equal(r["labels"], a.label)
        assert np.array_equal(r["table"], s.table)
        # layout: every rank holds the same positions ...
        for key, ref in (("sup_pos", ref_sup), ("full_pos", ref_full)):
            pos = r[key]
            diam = np.hypot(*(ref.positions.max(0) - ref.positions.min(0)))
            # ... within 1e-7 x diameter of the single-GPU run (regrouped fp64
            # sums of swing/traction only; same tolerance as the CPU parity)
            assert np.max(np.abs(pos - ref.positions)) <= 1e-7 * diam, key
        np.testing.assert_allclose(r["sup_disp"], ref_sup.displacement, rtol=1e-6, atol=1e-9)
    assert np.array_equal(r0["sup_pos"], r1["sup_pos"])
    assert np.array_equal(r0["full_pos"], r1["full_pos"])
    ref_exact = cv.layout(sup, cv.LayoutParams(iterations=5, theta=0.0))
    ref_coin = cv.layout(sup, cv.LayoutParams(iterations=5), positions=r0["p0"])
    for key, ref in (("exact_pos", ref_exact), ("coin_pos", ref_coin)):
        diam = np.hypot(*(ref.positions.max(0) - ref.positions.min(0)))
        for r in (r0, r1):
            assert np.max(np.abs(r[key] - ref.positions)) <= 1e-7 * diam, key


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_rmat_counter_stream_and_sharded_degrees():
    """C5 input: the device R-MAT stream equals its numpy twin for any slice
    (so shards compose), and edge-sharded degrees + sketch over it equal the
    oracle's np.bincount / node-based sketch (world of 1 here; the 2-rank
    decomposition is covered above)."""
    import paper_2108_00529_b200 as cv
    from oracle import oracle as orc
    from paper_2108_00529_b200 import synth
    from paper_2108_00529_b200.sharded import (Comm, accumulate_sizes_edges_sharded,
                                               accumulate_sizes_sharded,
                                               from_edge_array_sharded)
    scale, m = 14, 16 << 14
    host = synth.rmat_counter(scale, 0, m, seed=3)
    for lo, hi in ((0, m), (12345, 20000), (m - 7, m)):
        dev = synth.rmat_dev(scale, lo, hi - lo, seed=3).cpu().numpy()
        assert np.array_equal(dev, host[lo:hi])
    g = from_edge_array_sharded(synth.rmat_dev(scale, 0, m, seed=3), Comm(), node_count=1 << scale)
    n, ee, deg = orc.from_edge_array(host, node_count=1 << scale)
    assert g.edge_count == len(ee) and np.array_equal(g.degree, deg)
    labels = np.arange(n, dtype=np.int64) // 64
    s = cv.sketch_new(4, cv.default_cols(g.edge_count), seed=0)
    accumulate_sizes_sharded(s, labels, g)
    A, B = orc.sketch_params(4, 0)
    t = np.zeros((4, orc.default_cols(len(ee))), np.int64)
    orc.sketch_add_many(t, A, B, labels, deg)
    assert np.array_equal(s.table, t)
    s2 = cv.sketch_new(4, cv.default_cols(g.edge_count), seed=0)
    accumulate_sizes_edges_sharded(s2, labels, g)   # edge-based form, same counters
    assert np.array_equal(s2.table, t)


def _rmat_fa2_worker(rank, world, port, out_dir, scale, iters):
    dist = _init(rank, world, port)
    import torch
    torch.cuda.set_device(0)                      # both ranks share one B200
    import paper_2108_00529_b200 as cv
    from paper_2108_00529_b200 import synth
    from paper_2108_00529_b200.sharded import (Comm, from_edge_array_sharded, layout_sharded,
                                               shard_range)
    comm = Comm()
    m = 16 << scale
    lo, hi = shard_range(m, rank, world)
    g = from_edge_array_sharded(synth.rmat_dev(scale, lo, hi - lo, seed=1), comm,
                                node_count=1 << scale).gather()
    r = layout_sharded(g, cv.LayoutParams(iterations=iters), comm)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), pos=r.positions, disp=r.displacement)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_sharded_fa2_rmat20_matches_single_gpu():
    """C5-shaped node-sharded ForceAtlas2 (R-MAT scale 20: 2^20 bodies, 2^24
    draws): two ranks, each with a CSR over the rows it owns only, give the
    single-GPU layout within 1e-7 x diameter (only the Σswing/Σtraction sums
    are regrouped)."""
    import paper_2108_00529_b200 as cv
    from paper_2108_00529_b200 import synth
    scale, iters = 20, 3
    with tempfile.TemporaryDirectory() as d:
        _spawn(_rmat_fa2_worker, 2, d, scale, iters)
        r0, r1 = (np.load(os.path.join(d, f"r{i}.npz")) for i in (0, 1))
    g = cv.from_edge_array(synth.rmat_dev(scale, 0, 16 << scale, seed=1), node_count=1 << scale)
    ref = cv.layout(g, cv.LayoutParams(iterations=iters))
    diam = np.hypot(*(ref.positions.max(0) - ref.positions.min(0)))
    assert np.array_equal(r0["pos"], r1["pos"])
    assert np.max(np.abs(r0["pos"] - ref.positions)) <= 1e-7 * diam
    np.testing.assert_allclose(r0["disp"], ref.displacement, rtol=1e-6, atol=1e-9)
