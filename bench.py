"""Benchmark: the BigGraphVis hot path on the 3M-node / 34M-edge power-law
graph (BASELINE.json configs[3], the config the "end-to-end s at 3M/34M"
metric is quoted on).

One step = the whole north-star path on one synthetic graph resident in HBM:
  from_edge_array (self-loop drop + degrees) -> degree_stats ->
  detect_communities (deterministic, bit-exact mode; workers=1) ->
  sketch_new + accumulate_sizes -> contract -> layout(supergraph, 100 iters).
value = input edges / step time (edges/s).  Sub-metrics: community-pass
edges/s, ms per ForceAtlas2 iteration, end-to-end seconds.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun): the community pass does not shard, so the
end-to-end step runs as N independent replicas, one graph per GPU (weak
scaling); time = max over ranks.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "edges/s community pass; ms per ForceAtlas2 iter; end-to-end s at 3M/34M graph"
WORKLOAD = "C4: DC-SBM power-law 3M nodes / 34M edge draws (gamma 2.3, k=30000, mu 0.1)"


def workload(config):
    if config == "C4":
        return WORKLOAD
    from paper_2108_00529_b200.synth import CONFIGS
    c = CONFIGS[config]
    return (f"{config}: DC-SBM {c['n']} nodes / {c['m']} edge draws (gamma {c['gamma']}, "
            f"k={c['k']}, mu 0.1) -- a parity config, not the headline")
ITERS = 100


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="C4")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-sharded", action="store_true")
    p.add_argument("--no-secondary", action="store_true")
    return p.parse_args()


class Clocks:
    """SM clock / throttle-reason sampler running during the timed region
    (NVML polled every 20 ms from a thread; nvidia-smi's 200 ms loop missed
    short regions)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, index=0, period=0.02):
        self.index, self.period = index, period
        self.sm, self.mask, self.mx = [], 0, None
        self._stop = threading.Event()
        self.t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def loop():
                while True:
                    try:
                        self.sm.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                        self.mask |= int(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))
                    except Exception:  # noqa: BLE001 -- sampling must not fail the bench
                        pass
                    if self._stop.wait(self.period):
                        return
            self.t = threading.Thread(target=loop, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001 -- no NVML: report no samples
            self.t = None
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.t:
            self.t.join(timeout=2)

    def summary(self):
        reasons = sorted(k for k, bit in self.REASONS.items() if self.mask & bit)
        return {"sm_mhz": float(np.median(self.sm)) if self.sm else None,
                "sm_max_mhz": self.mx, "reasons": reasons, "samples": len(self.sm)}


def dist_init(n_gpus):
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        # CVZ_DIST_BACKEND=gloo lets several ranks share one GPU (test only)
        backend = os.environ.get("CVZ_DIST_BACKEND", "nccl")
        dev = local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(dev)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return rank, ws, local


def barrier_max(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


# ----------------------------------------------------------------- our arm
def pipeline(cv, edges_dev, stats=None, mode="deterministic"):
    """The north-star path, device-resident (public API calls)."""
    import torch
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    ev[0].record()
    g = cv.from_edge_array(edges_dev)
    base = cv.degree_stats(g).mode_degree
    ev[1].record()
    a = cv.detect_communities(g, cv.ThresholdSchedule(base=base), seed=0, workers=1, mode=mode)
    ev[2].record()
    s = cv.sketch_new(4, cv.default_cols(g.edge_count), seed=0)
    cv.accumulate_sizes(s, a, g)
    sg = cv.contract(g, a, s)
    ev[3].record()
    res = cv.layout(sg, cv.LayoutParams(iterations=ITERS, seed=0))
    ev[4].record()
    if stats is not None:
        torch.cuda.synchronize()
        stats.append(dict(ingest_ms=ev[0].elapsed_time(ev[1]),
                          detect_ms=ev[1].elapsed_time(ev[2]),
                          contract_ms=ev[2].elapsed_time(ev[3]),
                          layout_ms=ev[3].elapsed_time(ev[4]),
                          m=g.edge_count, n=g.node_count, rounds=len(a.round_history),
                          m_r=list(a.stream_edges), m_dev=list(a.device_stream_edges),
                          k=sg.node_count, se=sg.edge_count))
    return res


def pipeline_e2e(cv, edges_host):
    """Same path from pinned host memory to host results (drop-in API)."""
    g = cv.from_edge_array(edges_host)            # H2D inside
    base = cv.degree_stats(g).mode_degree
    a = cv.detect_communities(g, cv.ThresholdSchedule(base=base), seed=0, workers=1)
    s = cv.sketch_new(4, cv.default_cols(g.edge_count), seed=0)
    cv.accumulate_sizes(s, a, g)
    sg = cv.contract(g, a, s)
    res = cv.layout(sg, cv.LayoutParams(iterations=ITERS, seed=0))
    label = a.label                               # D2H of the per-node result
    return res.positions, label


# Algorithmic (compulsory) bytes per launch: int32 ids,
# fp64 layout state (our layout keeps the reference's fp64), every array
# touched once.  st = the instrumented step's stats.
def kernel_bytes(name, st):
    n, m, k, se = st["n"], st["m"], st["k"], st["se"]
    tab = {
        # per body: Body (x, y, m, id) 32 B read + force 16 B write;
        # per tree node: TNode 48 B read once
        "bh_kernel": k * (32 + 16) + (k - 1) * 48,
        # flat walk: per body 32 B read + 16 B force write; preorder node
        # array of k leaves + <= k-1 cells, PNode 32 B each, read once
        "bh_flat_kernel<4>": k * (32 + 16) + (2 * k - 1) * 32,
        "bh_flat_kernel<5>": k * (32 + 16) + (2 * k - 1) * 32,
        "bh_flat_kernel<6>": k * (32 + 16) + (2 * k - 1) * 32,
        # reads pos 16 + repulsion 16 + heavy index 4 + springs 16 + mass 8 +
        # prev 16, writes force 16 + swing 8, per node
        "forces_kernel": k * 100,
        # swing 8 + force 16 + pos r/w 32 + prev 16 per node
        "update_kernel": k * 72,
        # 1 ms graph replays excluded; per round bytes are in community_pass
    }
    return tab.get(name)


def community_pass_bytes(st):
    """per round 16 m_r (pass read + relabel read) + 8 m_{r+1}
    (compacted write) + 32 n (counters, labels, resolve, compose), with m_r
    the edges the device actually streams (dead edges dropped from the
    stream are not read, so they are not counted)."""
    mr = st["m_dev"]
    tot = 0
    for i, x in enumerate(mr):
        nxt = mr[i + 1] if i + 1 < len(mr) else 0
        tot += 16 * x + 8 * nxt + 32 * st["n"]
    return tot


def roofline(prof, st, peak_gbs):
    ks = sorted(prof.items(), key=lambda kv: -kv[1][1])
    total = sum(v[1] for _, v in ks) or 1.0
    top = [{"kernel": nm, "n": c, "ms": round(ms, 3), "share": round(ms / total, 3)}
           for nm, (c, ms) in ks[:12]]
    name, (cnt, ms) = ks[0]
    b = kernel_bytes(name, st)
    per_launch_s = ms / cnt / 1000.0
    ach = (b / per_launch_s / 1e9) if b is not None else None
    roof = {"kernel": name, "bound": "hbm", "achieved": ach, "peak": peak_gbs, "unit": "GB/s",
            "frac": (ach / peak_gbs) if ach is not None else None, "traffic": None,
            "bytes_per_launch": b, "launch_ms": per_launch_s * 1000.0, "launches": cnt,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)"}
    if name.startswith("bh_"):
        # the tree walk is not HBM-bound: its node array is L1/L2-resident and
        # every visit is a dependent fp64 chain (profiles/r1g_ncu_full_c4_fa2.md)
        roof["limiter"] = ("L1TEX-throughput-bound fp64 tree walk (ncu: LSU wavefronts "
                           "~70% of peak elapsed, ~78% while active; L1 hit ~96%, DRAM ~1%); "
                           "see roofline.l1 and walk.fp64_frac")
    return roof, top


def peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def run_ours(args, rank, ws):
    import torch

    import paper_2108_00529_b200 as cv
    from paper_2108_00529_b200 import _native, synth
    e = synth.config_graph(args.config, seed=rank)
    m_in = len(e)
    host = torch.from_numpy(e).pin_memory()
    dev = host.to("cuda")
    torch.cuda.synchronize()
    for _ in range(args.warmup):
        pipeline(cv, dev)
    torch.cuda.synchronize()
    stats = []
    barrier(ws)
    launches0 = _native.launch_count()
    # no cyclic-GC pause inside a timed region (the pipeline syncs with the
    # host between stages, so a host stall would show up as device time)
    gc.collect()
    gc.disable()
    with Clocks(torch.cuda.current_device()) as clk:
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(args.steps):
            pipeline(cv, dev)
        t1.record()
        torch.cuda.synchronize()
    gc.enable()
    launches = (_native.launch_count() - launches0) // args.steps
    ms = t0.elapsed_time(t1)
    ms_step = barrier_max(ms / args.steps, ws)
    barrier(ws)
    # per-stage breakdown of one extra plain step (CUDA events between the
    # stages; the layout replays its CUDA graph as in the timed steps), then
    # per-kernel device times from one instrumented step (library kernels
    # bracketed by events on their own stream; graph replay off there)
    pipeline(cv, dev, stats)
    st = stats[0]
    with _native.profile() as prof:
        pipeline(cv, dev)
    # Barnes-Hut walk statistics from one more step with the instrumented
    # walk variant (interactions beside the bytes)
    _, bh_visits, bh_inter = _native.bh_stats(lambda: pipeline(cv, dev))
    # fast (racy) community mode, same graph: detect stage only
    g = cv.from_edge_array(dev)
    base = cv.degree_stats(g).mode_degree
    for _ in range(max(3, args.warmup)):
        cv.detect_communities(g, cv.ThresholdSchedule(base=base), workers=1, mode="fast")
    torch.cuda.synchronize()
    fms = []
    gc.collect()
    gc.disable()
    fa = None
    for _ in range(max(3, args.steps)):  # per-call events: report the median call
        fa = None  # release the previous result (its pinned label buffer) first
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record()
        fa = cv.detect_communities(g, cv.ThresholdSchedule(base=base), workers=1, mode="fast")
        f1.record()
        torch.cuda.synchronize()
        fms.append(f0.elapsed_time(f1))
    gc.enable()
    fast = dict(ms=float(np.median(fms)), ms_all=fms, rounds=len(fa.round_history),
                m_r=list(fa.stream_edges), m_dev=list(fa.device_stream_edges),
                communities=fa.community_count)
    del g
    # e2e through the public API from an ordinary (pageable) int64 numpy
    # array -- what a caller of the reference API holds (C/graph.py:114) --
    # to host numpy results (warm-up as for the device-resident steps: first
    # calls pay the staging / read-back buffer setup)
    host_np = e.astype(np.int64)
    for _ in range(max(1, args.warmup)):
        pos, lab = pipeline_e2e(cv, host_np)
    torch.cuda.synchronize()
    gc.collect()
    gc.disable()
    e0 = time.perf_counter()
    for _ in range(args.steps):
        pos, lab = pipeline_e2e(cv, host_np)
    torch.cuda.synchronize()
    gc.enable()
    e2e_ms = barrier_max((time.perf_counter() - e0) * 1000 / args.steps, ws)
    h2d = 8 * len(host_np)  # int32 pairs on the link (narrowed on the host)
    d2h = pos.nbytes + lab.nbytes
    return dict(ms_step=ms_step, m_in=m_in, stage=st, launches=launches, clocks=clk.summary(),
                bh_visits=bh_visits / ITERS, bh_inter=bh_inter / ITERS,
                e2e_ms=e2e_ms, h2d=h2d, d2h=d2h, prof=prof.kernels, fast=fast)


# ------------------------------------------------- secondary named shapes
def _timed(fn, reps):
    """Median device time (ms) of fn() over reps calls after one warm-up."""
    import torch
    fn()
    torch.cuda.synchronize()
    out = []
    gc.collect()
    gc.disable()
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    gc.enable()
    return float(np.median(out))


def run_secondary(reps=3):
    """BASELINE.json configs[0..2] (north star: 'throughput on the named
    shapes'), device-resident inputs, public API calls:
      C1 full pipeline with 500 supergraph ForceAtlas2 iterations;
      C2 deterministic community pass edges/s (and the whole path);
      C3 BigGraphVis supergraph layout (pipeline mode, 100 iterations) vs
         full-graph ForceAtlas2 (full mode, 500 iterations, C/cli.py:58) with
         community colouring of every node (C/cli.py:191-203)."""
    import torch

    import paper_2108_00529_b200 as cv
    from paper_2108_00529_b200 import synth
    from paper_2108_00529_b200.render import assign_colors, color_full_graph
    out = {}
    dev = {c: torch.from_numpy(synth.config_graph(c, seed=0)).to("cuda") for c in ("C1", "C2", "C3")}

    def front(e):
        g = cv.from_edge_array(e)
        base = cv.degree_stats(g).mode_degree
        a = cv.detect_communities(g, cv.ThresholdSchedule(base=base), seed=0, workers=1)
        s = cv.sketch_new(4, cv.default_cols(g.edge_count), seed=0)
        cv.accumulate_sizes(s, a, g)
        return g, a, cv.contract(g, a, s)

    # C1: pipeline + 500 supergraph iterations
    def c1():
        g, a, sg = front(dev["C1"])
        return cv.layout(sg, cv.LayoutParams(iterations=500, seed=0))
    ms = _timed(c1, reps)
    g, a, sg = front(dev["C1"])
    out["C1"] = {"what": "full pipeline, 500 supergraph FA2 iterations", "ms_per_step": ms,
                 "edges_per_s": g.edge_count / (ms / 1e3), "n": g.node_count, "m": g.edge_count,
                 "supernodes": sg.node_count}
    # C2: deterministic community pass
    g2 = cv.from_edge_array(dev["C2"])
    base2 = cv.degree_stats(g2).mode_degree
    det_ms = _timed(lambda: cv.detect_communities(g2, cv.ThresholdSchedule(base=base2), seed=0,
                                                  workers=1), reps)

    def c2():
        g, a, sg = front(dev["C2"])
        return cv.layout(sg, cv.LayoutParams(iterations=ITERS, seed=0))
    step2 = _timed(c2, reps)
    out["C2"] = {"what": "deterministic (bit-exact) community pass; whole path with 100 "
                         "supergraph iterations", "detect_ms": det_ms,
                 "community_pass_edges_per_s": g2.edge_count / (det_ms / 1e3),
                 "ms_per_step": step2, "n": g2.node_count, "m": g2.edge_count}
    del g2
    # C3: supergraph layout vs full-graph layout + colouring
    g3, a3, sg3 = front(dev["C3"])
    sup_ms = _timed(lambda: cv.layout(sg3, cv.LayoutParams(iterations=ITERS, seed=0)), reps)
    full_iters = 500

    def full_mode():
        res = cv.layout(g3, cv.LayoutParams(iterations=full_iters, seed=0))
        colors = assign_colors(sg3.weight)
        return color_full_graph(a3.label, sg3.community_id, colors), res
    full_ms = _timed(full_mode, 1)
    front_ms = _timed(lambda: front(dev["C3"]), reps)
    out["C3"] = {"what": "BigGraphVis supergraph layout (100 it) vs full-graph FA2 (500 it) + "
                         "community colouring of every node",
                 "front_ms": front_ms,
                 "supergraph_layout_ms_per_iter": sup_ms / ITERS,
                 "pipeline_mode_ms": front_ms + sup_ms,
                 "full_graph_fa2_ms_per_iter": full_ms / full_iters,
                 "full_mode_ms": front_ms + full_ms,
                 "n": g3.node_count, "m": g3.edge_count, "supernodes": sg3.node_count,
                 "superedges": sg3.edge_count}
    del dev, g3, a3, sg3
    torch.cuda.empty_cache()
    return out


# ------------------------------------------------------------ sharded stages
FULL_ITERS = 10


def run_sharded(args, rank, ws, reps=3):
    """SURVEY.md 8e sharded stages on the SAME graph split across the N ranks
    (strong scaling): edge-sharded ingest + degrees + edge-based sketch
    (NCCL all-reduce of degrees and counters), and node-sharded full-graph
    ForceAtlas2 (per-iteration all-reduces + position all-gather).  Device
    time, max over ranks."""
    import torch

    import paper_2108_00529_b200 as cv
    from paper_2108_00529_b200 import sharded as sh
    from paper_2108_00529_b200 import synth
    comm = sh.Comm()
    e = synth.config_graph(args.config, seed=0)
    mine = torch.from_numpy(np.ascontiguousarray(sh.edge_slice(e, comm))).to("cuda")
    g_sh = sh.from_edge_array_sharded(mine, comm)
    g = g_sh.gather()
    lab = None
    if rank == 0:
        base = cv.degree_stats(g).mode_degree
        lab = cv.detect_communities(g, cv.ThresholdSchedule(base=base), seed=0, workers=1)
    labels = sh.broadcast_labels(lab, g.node_count, comm)
    cols = cv.default_cols(g.edge_count)

    def ingest_sketch():
        gs = sh.from_edge_array_sharded(mine, comm)
        s = cv.sketch_new(4, cols, seed=0)
        sh.accumulate_sizes_sharded(s, labels, gs)
        return s

    for _ in range(2):
        ingest_sketch()
    torch.cuda.synchronize()
    barrier(ws)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(reps):
        ingest_sketch()
    t1.record()
    torch.cuda.synchronize()
    ing_ms = barrier_max(t0.elapsed_time(t1) / reps, ws)

    # node-sharded full-graph layout (mass = degree + 1, unit springs)
    from paper_2108_00529_b200.layout import _device_model, _init_positions_dev
    mass, ed, ew = _device_model(g)
    P = sh._layout_params(cv.LayoutParams(iterations=FULL_ITERS))
    pos0 = _init_positions_dev(g.node_count, 0)
    sh._run_shard(comm, g.node_count, mass, ed, ew, P, pos0, 2, False)  # warm-up
    torch.cuda.synchronize()
    barrier(ws)
    t0.record()
    sh._run_shard(comm, g.node_count, mass, ed, ew, P, pos0, FULL_ITERS, False)
    t1.record()
    torch.cuda.synchronize()
    fa2_ms = barrier_max(t0.elapsed_time(t1), ws)
    c5 = run_c5(comm, rank, ws)
    return {"scaling": "strong", "ranks": ws, "graph": f"{args.config} seed 0 (same graph on all ranks)",
            "c5_rmat26_degrees_sketch": c5,
            "ingest_sketch_ms": ing_ms, "ingest_sketch_edges_per_s": len(e) / (ing_ms / 1e3),
            "full_graph_fa2_ms_per_iter": fa2_ms / FULL_ITERS,
            "full_graph_fa2_iters": FULL_ITERS, "n": g.node_count, "m": g.edge_count,
            "note": "edge-sharded ingest+degrees+sketch (all-reduce of int64 degrees and "
                    "sketch counters); node-sharded full-graph ForceAtlas2 incl. CSR build "
                    "(2 all-reduces + 1 all-gather per iteration)"}


C5_SCALE = int(os.environ.get("CVZ_C5_SCALE", "26"))


def run_c5(comm, rank, ws, reps=3, fa2=True):
    """BASELINE config C5: R-MAT scale 26 (2^26 nodes, 2^30 edge draws),
    edge-sharded ingest + degrees + sketch across the ranks.
    Each rank generates its own slice of the counter-based stream in HBM
    (cvz_rmat_edges, outside the timed region); the timed region is
    from_edge_array_sharded (compaction + degrees + all-reduce of 2^26 int64
    degrees) + accumulate_sizes_sharded (node-based: degree under label per
    owned node, labels = id // 64, all-reduce of the 4 x 107,375 counters,
    merge).
    Device time, max over ranks."""
    import torch

    import paper_2108_00529_b200 as cv
    from paper_2108_00529_b200 import sharded as sh
    from paper_2108_00529_b200 import synth
    n5, m5 = 1 << C5_SCALE, 16 << C5_SCALE
    lo, hi = sh.shard_range(m5, rank, ws)
    e5 = synth.rmat_dev(C5_SCALE, lo, hi - lo, seed=0)
    labels = torch.arange(n5, dtype=torch.int64, device="cuda") // 64

    def step():
        g = sh.from_edge_array_sharded(e5, comm, node_count=n5)
        s = cv.sketch_new(4, cv.default_cols(g.edge_count), seed=0)
        sh.accumulate_sizes_sharded(s, labels, g)
        return g

    g = step()
    torch.cuda.synchronize()
    barrier(ws)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(reps):
        step()
    t1.record()
    torch.cuda.synchronize()
    ms = barrier_max(t0.elapsed_time(t1) / reps, ws)
    m_kept = g.edge_count
    # SURVEY.md 8(d) bytes per rank: compaction 8 (read pair) + 8 (write kept
    # pair) per draw, degrees 8 per kept edge + 8 per node (int64 counters),
    # sketch (node-based) 16 per owned node (label + degree)
    ing_bytes = 16 * m5 / ws + 8 * m_kept / ws + 8 * n5 + 16 * n5 / ws
    out = {"scale": C5_SCALE, "nodes": n5, "edge_draws": m5, "edges_after_self_loops": m_kept,
           "ms": ms, "edges_per_s": m5 / (ms / 1e3),
           "hbm_frac_per_rank": ing_bytes / (ms / 1e3) / 1e9 / peak_hbm()[0],
           "note": "edge-sharded compaction + degrees, node-sharded sketch; labels = id // 64 "
                   "(synthetic communities; the order-dependent community pass is not sharded)"}
    del e5, labels
    # node-sharded full-graph ForceAtlas2 on the same R-MAT-26 graph: every
    # rank holds the whole compacted edge list (all-gather), builds its CSR
    # over the rows it owns only, the full tree, and walks/moves its bodies
    if fa2:
        out["fa2"] = run_c5_fa2(comm, g, ws)
    del g
    torch.cuda.empty_cache()
    return out


C5_FA2_ITERS = int(os.environ.get("CVZ_C5_FA2_ITERS", "5"))


def run_c5_fa2(comm, g_sh, ws):
    import torch

    import paper_2108_00529_b200 as cv
    from paper_2108_00529_b200 import sharded as sh
    from paper_2108_00529_b200.layout import _init_positions_dev
    g = g_sh.gather()
    n = g.node_count
    mass = (g.degree_dev() + 1).to(torch.float64)
    e = g.edges_dev()
    P = sh._layout_params(cv.LayoutParams(iterations=C5_FA2_ITERS + 1))
    pos0 = _init_positions_dev(n, 0)
    torch.cuda.synchronize()
    barrier(ws)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    lay = sh.ShardLayout(comm, n, mass, e, None, P, pos0, C5_FA2_ITERS + 1)
    t1.record()
    torch.cuda.synchronize()
    create_ms = barrier_max(t0.elapsed_time(t1), ws)
    try:
        lay.run(1)  # warm-up iteration (first tree build sizes its CUB temp)
        torch.cuda.synchronize()
        barrier(ws)
        t0.record()
        lay.run(C5_FA2_ITERS)
        t1.record()
        torch.cuda.synchronize()
        it_ms = barrier_max(t0.elapsed_time(t1) / C5_FA2_ITERS, ws)
        bad, _ = lay.finish()
        disp = lay.hist.cpu().tolist()
    finally:
        lay.close()
    out = {"ms_per_iter": it_ms, "iters_timed": C5_FA2_ITERS, "csr_setup_ms": create_ms,
           "bodies": n, "half_edges": 2 * g.edge_count, "non_finite": bad,
           "displacement": disp,
           "note": "node-sharded full-graph ForceAtlas2 (mass = degree + 1, unit springs); "
                   "each rank: CSR over its owned rows only, full Barnes-Hut tree, walk over "
                   "its own bodies; per iteration 2 all-reduces + 1 position all-gather"}
    del lay, pos0, mass, e, g
    torch.cuda.empty_cache()
    return out


# ------------------------------------------------------------ CPU baseline
CPU_LAYOUT_ITERS = 3


def cpu_pipeline_sample(config, seed=0):
    """Oracle (C + numpy port of the reference) on the SAME full graph:
    ingest + community pass + sketch + contract run in full; the layout runs
    CPU_LAYOUT_ITERS of the 100 supergraph iterations and is extrapolated
    ('time 3 iterations and extrapolate').
    Returns (edges, extrapolated seconds, detail)."""
    from oracle import oracle as orc
    from paper_2108_00529_b200 import synth
    e = synth.config_graph(config, seed=seed)
    t0 = time.perf_counter()
    n, ee, deg = orc.from_edge_array(e)
    mode = orc.degree_stats(deg)[0]
    lab, _, hist = orc.detect_communities(n, ee, deg, mode, 10, 0, workers=1)
    a, b = orc.sketch_params(4, 0)
    table = np.zeros((4, orc.default_cols(len(ee))), np.int64)
    orc.sketch_add_many(table, a, b, lab, deg)
    k, se, w, mult, comm = orc.contract(ee, lab, table, a, b)
    t1 = time.perf_counter()
    mass, ew = orc.masses_supergraph(w, mult)
    orc.layout(k, mass, se, ew, iterations=CPU_LAYOUT_ITERS, seed=0)
    t2 = time.perf_counter()
    total = (t1 - t0) + (t2 - t1) * ITERS / CPU_LAYOUT_ITERS
    return len(e), total, dict(measured_s=t2 - t0, pre_layout_s=t1 - t0,
                               layout_s_per_iter=(t2 - t1) / CPU_LAYOUT_ITERS, k=k, se=len(se))


REF_ARM_BUDGET_S = float(os.environ.get("CVZ_REF_ARM_BUDGET_S", "150"))


def reference_package_runner(seed=0):
    """The shipped reference itself (commviz + numba, oracle/_ref packaged by
    oracle/build_ref.py), NUMBA_NUM_THREADS = all host cores, after its own
    warmup_jit() (C/cli.py:278-287).  Returns step(config) -> (edges, s,
    stages): every stage in full on the full graph except the layout, timed
    for CPU_LAYOUT_ITERS of the 100 iterations and extrapolated (SURVEY.md
    8d).  The first step on any shape also compiles the supergraph layout's
    signatures (warmup_jit leaves them: 3.7 s), so warm-up steps run on C1."""
    import importlib

    from oracle import build_ref
    from paper_2108_00529_b200 import synth
    ref = build_ref.load()
    importlib.import_module("commviz.cli").warmup_jit()

    def step(config):
        e = synth.config_graph(config, seed=seed).astype(np.int64)
        st = {}
        t = time.perf_counter()
        g = ref.from_edge_array(e)
        base = ref.degree_stats(g).mode_degree
        st["ingest_s"] = time.perf_counter() - t
        t = time.perf_counter()
        a = ref.detect_communities(g, ref.ThresholdSchedule(base=base), seed=0, workers=1)
        st["detect_s"] = time.perf_counter() - t
        t = time.perf_counter()
        s = ref.sketch_new(4, ref.default_cols(g.edge_count), seed=0)
        ref.accumulate_sizes(s, a.label, g.degree)
        sg = ref.contract(g, a.label, s)
        st["sketch_contract_s"] = time.perf_counter() - t
        t = time.perf_counter()
        ref.layout(sg, ref.LayoutParams(iterations=CPU_LAYOUT_ITERS, seed=0))
        st["layout_s_per_iter"] = (time.perf_counter() - t) / CPU_LAYOUT_ITERS
        total = (st["ingest_s"] + st["detect_s"] + st["sketch_contract_s"]
                 + st["layout_s_per_iter"] * ITERS)
        st["communities"] = int(a.community_count)
        st["supernodes"] = int(sg.node_count)
        return len(e), total, st

    return step


def config_dict(args, ws):
    """The workload description both arms print (identical by construction)."""
    return {"workload": workload(args.config), "layout_iterations": ITERS,
            "community_mode": "deterministic", "parallelism": f"replicas x{ws}",
            "l2": "inputs (262 MB edge list at C4) larger than the 126 MB L2"}


def main():
    args = parse()
    rank, ws, local = dist_init(args.gpus)
    if args.impl == "reference":
        if rank != 0:
            return
        from oracle import oracle as orc
        orc.build()
        line = {
            "impl": "reference", "metric": METRIC, "unit": "edges/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "int32 ids / f64 layout", "data": "synthetic (seeded DC-SBM, no network)",
            "config": config_dict(args, args.gpus)}
        # the shipped package (oracle/_ref) is the arm; the C/numpy port is
        # the fallback where numba or the archive is missing, and is timed
        # once beside it otherwise
        try:
            step = reference_package_runner()
            for _ in range(max(1, args.warmup)):  # JIT of every signature on C1
                step("C1")
            vals, st = [], None
            t_arm = time.perf_counter()
            for _ in range(args.steps):  # ~25 s per C4 step: bounded to ~2.5 min
                m, dt, st = step(args.config)
                vals.append(m / dt)
                if time.perf_counter() - t_arm > REF_ARM_BUDGET_S:
                    break
            line["steps_timed"] = len(vals)
            v = float(np.median(vals))
            sample = (f"unmodified commviz package (numba {__import__('numba').__version__}, "
                      f"NUMBA_NUM_THREADS={os.environ.get('NUMBA_NUM_THREADS', os.cpu_count())})"
                      f" on the full {args.config} graph ({m} edges) after warmup_jit + "
                      f"{max(1, args.warmup)} C1 pass(es); every stage in full, the layout "
                      f"timed for {CPU_LAYOUT_ITERS} of {ITERS} iterations and extrapolated "
                      f"({st['layout_s_per_iter']:.2f} s/iter); est. {m / v:.1f} s per step")
            line.update(value=v, cpu_baseline={"value": v, "unit": "edges/s",
                                               "cores": os.cpu_count(), "kind": "reference",
                                               "sample": sample, "stages": st})
            try:  # the port beside it (once; not the value)
                m2, dt2, det = cpu_pipeline_sample(args.config)
                line["port"] = {"value": m2 / dt2, "unit": "edges/s", "kind": "port",
                                "cores": orc.num_threads(), "s_per_step_est": dt2,
                                "sample": "oracle pipeline (C/numpy restatement), same graph"}
            except Exception as ex:  # noqa: BLE001
                line["port"] = {"unavailable": f"{type(ex).__name__}: {ex}"[:200]}
        except Exception as ex:  # noqa: BLE001 -- no numba / archive: time the port
            vals = []
            for _ in range(args.warmup):
                cpu_pipeline_sample("C1")
            for _ in range(args.steps):
                m, dt, det = cpu_pipeline_sample(args.config)
                vals.append(m / dt)
            v = float(np.median(vals))
            sample = (f"full {args.config} graph ({m} edges) through the oracle pipeline "
                      f"(C/numpy port of commviz); layout timed for {CPU_LAYOUT_ITERS} of "
                      f"{ITERS} iterations and extrapolated ({det['layout_s_per_iter']:.2f} "
                      f"s/iter, measured {det['measured_s']:.1f} s per step)")
            line.update(value=v, cpu_baseline={"value": v, "unit": "edges/s",
                                               "cores": orc.num_threads(), "kind": "port",
                                               "sample": sample},
                        reference_package={"unavailable": f"{type(ex).__name__}: {ex}"[:200]})
        line["e2e"] = {"value": line["value"], "unit": "edges/s", "h2d_bytes_per_step": 0,
                       "d2h_bytes_per_step": 0}
        print(json.dumps(line))
        return

    r = run_ours(args, rank, ws)
    shard = None if args.no_sharded else run_sharded(args, rank, ws)
    secondary = None if (args.no_secondary or args.config != "C4") else run_secondary()
    if rank != 0:
        return
    import ctypes

    from paper_2108_00529_b200 import _native
    st = r["stage"]
    peak, _src = peak_hbm()
    roof, top = roofline(r["prof"], st, peak)
    roof["peak_source"] = f"MEASURED_PEAKS.json hbm_gbs ({_src})"
    fp64 = ctypes.c_double(0)
    _native.call("cvz_probe_fp64", ctypes.byref(fp64), _native.stream())
    if roof.get("kernel", "").startswith("bh_flat") and r.get("bh_inter"):
        # per-iteration walk counts (instrumented step) over the timed walk:
        # ~20 fp64 flops per accepted term (d, 1/d^2 seed + cubic step, f,
        # f*d accumulate), ~6 per opened cell (d, d^2, theta^2 d^2 test)
        sec = roof["launch_ms"] / 1e3
        acc, vis = r["bh_inter"], r["bh_visits"]
        gfl = (20 * acc + 6 * (vis - acc)) / sec / 1e9
        roof["walk"] = {"node_visits_per_iter": vis, "interactions_per_iter": acc,
                        "interactions_per_s": acc / sec, "fp64_gflops_est": gfl,
                        "fp64_peak_gflops": fp64.value,
                        "fp64_peak_source": "cvz_probe_fp64 (measured DFMA throughput, this GPU)",
                        "fp64_frac": gfl / fp64.value if fp64.value else None}
    try:  # DRAM bytes per launch from the committed ncu --set full capture
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            roof["traffic"] = json.load(fh).get(roof["kernel"])
    except (OSError, ValueError):
        pass
    try:  # the roof the walk actually sits under: L1TEX throughput (ncu)
        with open(os.path.join(ROOT, "profiles", "ncu_limits.json")) as fh:
            lim = json.load(fh).get(roof["kernel"])
        if lim:
            roof["l1"] = {
                "frac_elapsed": lim.get("l1tex__throughput.avg.pct_of_peak_sustained_elapsed"),
                "frac_active": lim.get("l1tex__throughput.avg.pct_of_peak_sustained_active"),
                "issue_active": lim.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                "fp64_pipe_active": lim.get(
                    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                "source": "profiles/ncu_limits.json (ncu --set full of this kernel)"}
    except (OSError, ValueError):
        pass
    value = r["m_in"] * ws / (r["ms_step"] / 1000.0)
    fast_bytes = community_pass_bytes(dict(st, m_dev=r["fast"]["m_dev"]))
    det_bytes = community_pass_bytes(st)
    summary = {
        # the BASELINE metric's three parts at C4, kept last so they survive
        # any truncation of the line's head
        "community_pass_edges_per_s": st["m"] / (st["detect_ms"] / 1000.0),
        "community_pass_hbm_frac": det_bytes / (st["detect_ms"] / 1000.0) / 1e9 / peak,
        "community_pass_fast_edges_per_s": st["m"] / (r["fast"]["ms"] / 1000.0),
        "community_pass_fast_hbm_frac": fast_bytes / (r["fast"]["ms"] / 1000.0) / 1e9 / peak,
        # edges the device streams, summed over rounds
        "community_pass_stream_edges_per_s": sum(st["m_dev"]) / (st["detect_ms"] / 1000.0),
        "ms_per_fa2_iter": st["layout_ms"] / ITERS,
        "end_to_end_s": r["ms_step"] / 1000.0,
        "e2e_s": r["e2e_ms"] / 1000.0,
        "stage_ms": {k: round(st[k], 4) for k in ("ingest_ms", "detect_ms", "contract_ms",
                                                   "layout_ms")},
        "walk_fp64_frac": roof.get("walk", {}).get("fp64_frac"),
    }
    if shard:
        c5 = shard.get("c5_rmat26_degrees_sketch") or {}
        summary["c5_ingest_sketch_edges_per_s"] = c5.get("edges_per_s")
        summary["c5_ingest_sketch_hbm_frac"] = c5.get("hbm_frac_per_rank")
        summary["c5_full_graph_fa2_ms_per_iter"] = (c5.get("fa2") or {}).get("ms_per_iter")
        summary["c4_full_graph_fa2_ms_per_iter"] = shard.get("full_graph_fa2_ms_per_iter")
    if secondary:
        summary["c1_ms_per_step_500it"] = secondary["C1"]["ms_per_step"]
        summary["c2_community_pass_edges_per_s"] = secondary["C2"]["community_pass_edges_per_s"]
        summary["c3_supergraph_ms_per_iter"] = secondary["C3"]["supergraph_layout_ms_per_iter"]
        summary["c3_full_graph_ms_per_iter"] = secondary["C3"]["full_graph_fa2_ms_per_iter"]
    line = {
        "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "int32 ids / f64 layout", "data": "synthetic (seeded DC-SBM, no network)",
        "config": config_dict(args, ws),
        "workload_stats": {"edges_in": r["m_in"], "n": st["n"], "m": st["m"],
                           "rounds": st["rounds"], "m_r": st["m_r"], "m_r_streamed": st["m_dev"],
                           "supernodes": st["k"], "superedges": st["se"],
                           "fast_mode": {k: r["fast"][k] for k in ("ms", "rounds", "communities",
                                                                    "m_dev")}},
        "gpu_launches": r["launches"],
        "clocks": r["clocks"],
        "roofline": roof,
        "top_kernels": top[:8],
        "sharded": shard,
        "secondary": secondary,
        "e2e": {"value": r["m_in"] * ws / (r["e2e_ms"] / 1000.0), "unit": "edges/s",
                "h2d_bytes_per_step": r["h2d"], "d2h_bytes_per_step": r["d2h"],
                "ms_per_step": r["e2e_ms"],
                "input": "pageable int64 numpy (m, 2) (the reference API's dtype), narrowed to "
                         "int32 on the host into pinned staging overlapped with the DMA; "
                         "labels (int64) + positions (f64) read back to numpy"},
    }
    if not args.no_cpu and ws == 1:
        from oracle import oracle as orc
        orc.build()
        m, dt, det = cpu_pipeline_sample(args.config)
        line["cpu_baseline"] = {
            "value": m / dt, "unit": "edges/s", "cores": orc.num_threads(), "kind": "port",
            "sample": f"same full graph ({m} edges); oracle stages in full, layout "
                      f"{CPU_LAYOUT_ITERS} of {ITERS} iterations extrapolated "
                      f"({det['layout_s_per_iter']:.2f} s/iter); est. {dt:.1f} s/step"}
    line["summary"] = summary
    print(json.dumps(line))


if __name__ == "__main__":
    main()
    try:  # clean NCCL/gloo shutdown on every rank (torchrun runs)
        import torch.distributed as _dist
        if _dist.is_available() and _dist.is_initialized():
            _dist.barrier()
            _dist.destroy_process_group()
    except Exception:  # noqa: BLE001 -- shutdown must not turn a result into a failure
        pass
