"""Multi-GPU forms of the stages that shard, one process per GPU.

The reference is single-process (C/graph.py, C/sketch.py, C/supergraph.py,
C/layout.py); these functions give the same results as their single-GPU
counterparts while splitting the work:

* `from_edge_array_sharded` -- edge-sharded ingest: every rank compacts its
  contiguous slice of the edge stream (stable self-loop drop, C/graph.py:
  117-118) and counts degrees over it; one all-reduce(SUM) of the int64
  histogram gives np.bincount of the whole stream (C/graph.py:121), bit-exact.
* `accumulate_sizes_sharded` -- node-sharded sketch build: degree under the
  label of each node of the rank's node range into a rank-local delta table
  (the degrees are global after the ingest all-reduce), one all-reduce(SUM)
  of rows x cols counters, then merge + saturate.  Integer addition mod 2^64
  makes this bit-identical to C/supergraph.py:42-46
  (`accumulate_sizes_edges_sharded` is the edge-based form).
* `layout_sharded` -- node-sharded ForceAtlas2: every rank holds all
  positions, builds the full Barnes-Hut tree, and moves the nodes it owns;
  per iteration two tiny all-reduces (Σswing/Σtraction, bbox/max-disp/bad)
  and one all-gather of positions (C/layout.py:363-398 split at its
  reductions).  fp64 sums are regrouped, so this is tolerance-gated like
  every layout result.

The community pass is order-dependent and stays on one GPU ("replicas
only").  The collectives are torch.distributed calls on CUDA
tensors: NCCL over NVLink/NVSwitch on a multi-GPU box; with a gloo group
(CPU tests, or several ranks sharing one GPU) they are staged through host
memory.  All compute is in libcvz_b200.so -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import warnings

import numpy as np

from . import _native as nat
from .graph import Graph, upload_edges
from .layout import (_ATTRACTION_FORMS, _SPEED_FORMS, LayoutParams, LayoutResult,
                     _device_model, _init_positions_dev, init_positions)
from ._native import LayoutError
from .supergraph import _labels_dev


# ------------------------------------------------------------------ planning
def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous balanced slice [lo, hi) of `total` units for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    return total * rank // world, total * (rank + 1) // world


def padded_rows(n: int, world: int) -> int:
    """Rows per rank for equal-size all-gathers (ceil(n / world))."""
    return max(1, -(-n // world))


def owned_nodes(n: int, rank: int, world: int) -> tuple[int, int]:
    """Original node ids a rank owns in the node-sharded layout: the
    rank-th block of padded_rows(n, world) ids (the all-gather layout)."""
    s = padded_rows(n, world)
    return min(n, rank * s), min(n, (rank + 1) * s)


class Comm:
    """The few collectives the sharded stages need, on CUDA or CPU tensors.

    `group=None` uses the default process group; with no initialised
    process group it is a world of one (every collective is the identity).
    NCCL groups run on the tensors in place; any other backend (gloo) is
    staged through host memory, so the same code runs in CPU tests and with
    several ranks sharing one GPU."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.rank = dist.get_rank(group)
            self.world = dist.get_world_size(group)
            self.backend = str(dist.get_backend(group))
        else:
            self.rank, self.world, self.backend = 0, 1, None
        self.staged = self.backend != "nccl"
        # run the collectives even in a world of one (tests drive the NCCL
        # branch on a single GPU this way; otherwise they are identities)
        self.force = False

    def _op(self, op):
        R = self.dist.ReduceOp
        return {"sum": R.SUM, "max": R.MAX, "min": R.MIN}[op]

    def all_reduce(self, t, op: str = "sum"):
        """In-place all-reduce of tensor t; returns t."""
        if self.world == 1 and not self.force:
            return t
        if self.staged and t.is_cuda:
            h = t.cpu()
            self.dist.all_reduce(h, op=self._op(op), group=self.group)
            t.copy_(h)
        else:
            self.dist.all_reduce(t, op=self._op(op), group=self.group)
        return t

    def broadcast(self, t, src: int = 0):
        if self.world == 1 and not self.force:
            return t
        if self.staged and t.is_cuda:
            h = t.cpu()
            self.dist.broadcast(h, src=src, group=self.group)
            t.copy_(h)
        else:
            self.dist.broadcast(t, src=src, group=self.group)
        return t

    def all_gather_rows(self, full, rows: int):
        """full: (world * rows, ...) tensor whose block `rank` holds this
        rank's rows; fills every other block from its owner (in place)."""
        if self.world == 1 and not self.force:
            return full
        mine = full[self.rank * rows:(self.rank + 1) * rows]
        if self.staged:
            dev = full.device
            h = mine.cpu()
            parts = [h.new_empty(h.shape) for _ in range(self.world)]
            self.dist.all_gather(parts, h, group=self.group)
            for r, p in enumerate(parts):
                if r != self.rank:
                    full[r * rows:(r + 1) * rows].copy_(p.to(dev))
        else:
            send = mine.clone()
            self.dist.all_gather_into_tensor(full, send, group=self.group)
        return full

    def all_gather_varlen(self, t):
        """Concatenate every rank's t (same trailing shape, any length) in
        rank order; returns the concatenation on t's device."""
        import torch
        if self.world == 1 and not self.force:
            return t
        cnt = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
        counts = torch.zeros(self.world, dtype=torch.int64, device=t.device)
        counts[self.rank] = cnt[0]
        self.all_reduce(counts, "sum")
        c = [int(x) for x in counts.cpu().tolist()]
        rows = max(1, max(c))
        buf = t.new_zeros((self.world * rows,) + tuple(t.shape[1:]))
        buf[self.rank * rows:self.rank * rows + c[self.rank]].copy_(t)
        self.all_gather_rows(buf, rows)
        return torch.cat([buf[r * rows:r * rows + c[r]] for r in range(self.world)])


# ---------------------------------------------------------------- ingest
class ShardedGraph:
    """An edge-sharded Graph: this rank's compacted slice of the edge stream
    plus the GLOBAL degree array (identical on every rank)."""

    def __init__(self, node_count, edges_local, degree, edge_count, edge_offset, comm):
        self.node_count = int(node_count)
        self.edges_local = edges_local      # (m_local, 2) int32 CUDA tensor, stream order
        self._degree = degree               # (n,) int64 CUDA tensor, global
        self.edge_count = int(edge_count)   # global m after the self-loop drop
        self.edge_offset = int(edge_offset)  # index of edges_local[0] in the global stream
        self.comm = comm

    @property
    def degree(self) -> np.ndarray:
        return nat.to_host(self._degree)

    def degree_dev(self):
        return self._degree

    def gather(self) -> Graph:
        """The whole graph on every rank (all-gather of the edge slices in
        rank order == from_edge_array of the concatenated stream)."""
        e = self.comm.all_gather_varlen(self.edges_local)
        return Graph._from_device(self.node_count, e.contiguous(), self._degree)

    def __repr__(self):
        return (f"ShardedGraph(node_count={self.node_count}, edge_count={self.edge_count}, "
                f"rank={self.comm.rank}/{self.comm.world}, local={int(self.edges_local.shape[0])})")


def edge_slice(edges, comm: Comm):
    """This rank's contiguous slice of a full (m, 2) edge array."""
    m = len(edges)
    lo, hi = shard_range(m, comm.rank, comm.world)
    return edges[lo:hi]


def from_edge_array_sharded(edges_local, comm: Comm | None = None,
                            node_count=None) -> ShardedGraph:
    """Edge-sharded C/graph.py:114-122: `edges_local` is this rank's
    contiguous slice of the edge stream (ranks in stream order)."""
    T = nat.torch()
    comm = comm or Comm()
    if isinstance(edges_local, T.Tensor):
        src = edges_local.reshape(-1, 2)
        if src.dtype not in (T.int32, T.int64) or not src.is_cuda:
            src = nat.to_dev(src, T.int64)
        src = src.contiguous()
    else:
        src = upload_edges(edges_local)
    m_in = int(src.shape[0])
    dev = nat.device()
    out = T.empty((max(m_in, 1), 2), dtype=T.int32, device=dev)
    scal = T.zeros(2, dtype=T.int64, device=dev)
    nat.call("cvz_edges_compact", nat.ptr(src), int(src.dtype == T.int32), m_in,
             nat.ptr(out), nat.ptr(scal), nat.ptr(scal[1:]), 1, nat.stream())
    # global edge count, per-rank offsets and max id: one small all-reduce
    counts = T.zeros(comm.world, dtype=T.int64, device=dev)
    counts[comm.rank] = scal[0]
    comm.all_reduce(counts, "sum")
    mx_t = T.where(scal[0] > 0, scal[1], T.full_like(scal[1], -1)).reshape(1)
    comm.all_reduce(mx_t, "max")
    c = [int(x) for x in counts.cpu().tolist()]
    mx = int(mx_t.item())
    m_loc, m_tot = c[comm.rank], sum(c)
    offset = sum(c[:comm.rank])
    if node_count is None:
        n = mx + 1 if m_tot else 0
    else:
        n = int(node_count)
    nbins = max(n, mx + 1) if m_tot else n
    degree = T.empty(max(nbins, 1), dtype=T.int64, device=dev)
    nat.call("cvz_degree_count", nat.ptr(out), m_loc, nbins, nat.ptr(degree), nat.stream())
    comm.all_reduce(degree, "sum")
    return ShardedGraph(n, out[:m_loc], degree[:nbins], m_tot, offset, comm)


def broadcast_labels(labels, n: int, comm: Comm | None = None, src: int = 0):
    """Labels from the community GPU (rank `src`) to every rank, as an int64
    CUDA tensor.  Non-source ranks may pass None."""
    T = nat.torch()
    comm = comm or Comm()
    if comm.rank == src:
        lab = _labels_dev(labels).contiguous()
    else:
        lab = T.empty(n, dtype=T.int64, device=nat.device())
    return comm.broadcast(lab, src)


# ---------------------------------------------------------------- sketch
def accumulate_sizes_sharded(sketch, labels, g: ShardedGraph) -> None:
    """Node-sharded C/supergraph.py:42-46: after the degree all-reduce every
    rank holds the global degrees, so each adds degree[v] under label[v] for
    the nodes v of its own contiguous node range into a rank-local delta
    table; the deltas are summed across ranks (all-reduce of rows x cols
    counters) and merged + saturated once.  Integer addition mod 2^64 makes
    this bit-identical to the single-GPU node-based table, and each rank
    streams 16 B per owned node instead of gathering a label per endpoint of
    its edges (node ranges or edge ranges)."""
    T = nat.torch()
    lab = _labels_dev(labels)
    if int(lab.shape[0]) < g.node_count:
        raise ValueError("one label per node required")
    delta = T.zeros((sketch.rows, sketch.cols), dtype=T.int64, device=nat.device())
    a, b = sketch._hash_dev()
    lo, hi = shard_range(g.node_count, g.comm.rank, g.comm.world)
    deg = g.degree_dev()
    if hi > lo:
        nat.call("cvz_sketch_accumulate", nat.ptr(delta), sketch.rows, sketch.cols,
                 nat.ptr(a), nat.ptr(b), nat.ptr(lab[lo:hi]), nat.ptr(deg[lo:hi]), hi - lo,
                 nat.stream())
    g.comm.all_reduce(delta, "sum")
    table = sketch.table_dev()
    sat = T.zeros(1, dtype=T.int32, device=nat.device())
    nat.call("cvz_sketch_merge", nat.ptr(table), nat.ptr(delta), sketch.rows, sketch.cols,
             nat.ptr(sat), nat.stream())
    sketch._table.set_dev(table)
    if int(sat.item()) and not sketch.saturated:
        sketch.saturated = True
        warnings.warn("sketch counter overflow, counts saturated", RuntimeWarning, stacklevel=2)


def accumulate_sizes_edges_sharded(sketch, labels, g: ShardedGraph) -> None:
    """The edge-sharded form (+1 under the label of both endpoints of each
    local edge; identical counters to the node-based form).
    Kept for graphs whose degree array is not replicated."""
    T = nat.torch()
    lab = _labels_dev(labels)
    if int(lab.shape[0]) < g.node_count:
        raise ValueError("one label per node required")
    delta = T.zeros((sketch.rows, sketch.cols), dtype=T.int64, device=nat.device())
    a, b = sketch._hash_dev()
    e = g.edges_local
    nat.call("cvz_sketch_accumulate_edges", nat.ptr(delta), sketch.rows, sketch.cols,
             nat.ptr(a), nat.ptr(b), nat.ptr(e), int(e.shape[0]), nat.ptr(lab), nat.stream())
    g.comm.all_reduce(delta, "sum")
    table = sketch.table_dev()
    sat = T.zeros(1, dtype=T.int32, device=nat.device())
    nat.call("cvz_sketch_merge", nat.ptr(table), nat.ptr(delta), sketch.rows, sketch.cols,
             nat.ptr(sat), nat.stream())
    sketch._table.set_dev(table)
    if int(sat.item()) and not sketch.saturated:
        sketch.saturated = True
        warnings.warn("sketch counter overflow, counts saturated", RuntimeWarning, stacklevel=2)


# ---------------------------------------------------------------- layout
def _layout_params(params: LayoutParams):
    return nat._LayoutParams(params.iterations, params.gravity, params.repulsion,
                             params.jitter_tolerance, params.theta, params.max_step,
                             _SPEED_FORMS.index(params.speed_form),
                             _ATTRACTION_FORMS.index(params.attraction_form))


class ShardLayout:
    """One node-sharded ForceAtlas2 run (cvz_fa2_shard_*) on this rank.

    `create` builds the rank's CSR over the rows it owns only (a stable
    select of their half-edges, C/layout.py:293-304 split by row) and the
    per-iteration state; `run(k)` advances k iterations, each one
    forces -> all-reduce(SUM) Σswing/Σtraction -> update -> all-reduce(MAX)
    bbox/max-disp/bad -> all-gather of the owned position rows
    (C/layout.py:363-398 split at its reductions)."""

    def __init__(self, comm, n, mass, e, ew, P, pos0, iterations, ref_ids=False):
        T = nat.torch()
        dev = nat.device()
        self.comm, self.n = comm, n
        self.rows = padded_rows(n, comm.world)
        lo, hi = owned_nodes(n, comm.rank, comm.world)
        self.full = T.zeros((comm.world * self.rows, 2), dtype=T.float64, device=dev)
        self.full[:n].copy_(pos0)
        self.pos = self.full[:n]
        self.h = ctypes.c_void_p()
        self.s = nat.stream()
        nat.call("cvz_fa2_shard_create", nat.ptr(self.pos), nat.ptr(mass), n, nat.ptr(e),
                 int(e.shape[0]), nat.ptr(ew), ctypes.byref(P), lo, hi, int(ref_ids),
                 ctypes.byref(self.h), self.s)
        self.sums = T.zeros(2, dtype=T.float64, device=dev)
        self.red = T.zeros(6, dtype=T.float64, device=dev)
        self.hist = T.zeros(max(1, iterations), dtype=T.float64, device=dev)
        self.done = 0

    def run(self, k: int) -> None:
        lib = nat.load()
        h, s, pos, sums, red = self.h, self.s, self.pos, self.sums, self.red
        for _ in range(k):
            # absorb writes hist[iteration]; iterations past its length are not recorded
            hist = nat.ptr(self.hist) if self.done < self.hist.shape[0] else None
            nat.check(lib.cvz_fa2_shard_forces(h, nat.ptr(pos), nat.ptr(sums), s), "forces")
            self.comm.all_reduce(sums, "sum")
            nat.check(lib.cvz_fa2_shard_update(h, nat.ptr(pos), nat.ptr(sums), nat.ptr(red), s),
                      "update")
            self.comm.all_reduce(red, "max")
            self.comm.all_gather_rows(self.full, self.rows)
            nat.check(lib.cvz_fa2_shard_absorb(h, nat.ptr(red), hist, s), "absorb")
            self.done += 1

    def finish(self):
        """(bad iteration (1-based, 0 = none), jitter seen)."""
        speed = ctypes.c_double(0)
        bad = ctypes.c_int64(0)
        jit = ctypes.c_int(0)
        nat.call("cvz_fa2_shard_finish", self.h, ctypes.byref(speed), ctypes.byref(bad),
                 ctypes.byref(jit), self.s)
        return int(bad.value), int(jit.value)

    def close(self) -> None:
        if self.h:
            nat.load().cvz_fa2_shard_destroy(self.h, self.s)
            self.h = ctypes.c_void_p()


def _run_shard(comm, n, mass, e, ew, P, pos0, iterations, ref_ids):
    """One node-sharded FA2 run from pos0 (full, identical on every rank).
    Returns (padded positions, displacement history, bad, jitter_seen)."""
    sh = ShardLayout(comm, n, mass, e, ew, P, pos0, iterations, ref_ids)
    try:
        sh.run(iterations)
        bad, jit = sh.finish()
    finally:
        sh.close()
    return sh.full, sh.hist[:iterations], bad, jit


def layout_sharded(obj, params: LayoutParams | None = None, comm: Comm | None = None,
                   positions=None) -> LayoutResult:
    """Node-sharded C/layout.py:341-402 over the ranks of `comm`; every rank
    passes the same SuperGraph/Graph and gets the same LayoutResult."""
    T = nat.torch()
    params = params or LayoutParams()
    comm = comm or Comm()
    n = obj.node_count
    if positions is not None:
        pos = np.array(positions, dtype=np.float64)
        if pos.shape != (n, 2):
            raise ValueError("positions must be an (n, 2) array")
    if n == 1:
        pos = init_positions(n, params.seed) if positions is None else pos
        return LayoutResult(positions=pos, displacement=np.zeros(params.iterations),
                            iterations=params.iterations)
    if n == 0:
        raise ValueError("layout needs at least one node")
    mass, e, ew = _device_model(obj)
    pos0 = _init_positions_dev(n, params.seed) if positions is None else nat.to_dev(
        pos, T.float64)
    P = _layout_params(params)
    full, hist, bad, jit = _run_shard(comm, n, mass, e, ew, P, pos0, params.iterations, False)
    flag = T.tensor([float(jit)], dtype=T.float64, device=nat.device())
    if comm.all_reduce(flag, "max").item() > 0:
        # a cell interaction closer than COINCIDE_EPS: its jitter direction is
        # keyed by the reference's cell numbering (C/layout.py:258) -- rerun
        full, hist, bad, _ = _run_shard(comm, n, mass, e, ew, P, pos0, params.iterations, True)
    if bad:
        raise LayoutError(f"non-finite positions at iteration {bad}; "
                          "reduce speed or check input weights")
    return LayoutResult(positions=nat.to_host(full[:n]), displacement=nat.to_host(hist),
                        iterations=params.iterations)
