"""Multi-round streaming community detection (drop-in for C/community.py).

Each round runs on the GPU through `cvz_detect_round`: size-seeded counters,
the streaming pass (deterministic = bit-exact with the sequential reference,
or fast = racy one-thread-per-edge), label resolution, composition, history
and the contracted next-round stream all stay in HBM; the host only reads
two scalars per round (next stream length, changed flag).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from ._dual import Dual

TIE_SRC_JOINS_DST = 0
TIE_DST_JOINS_SRC = 1
TIE_SKIP = 2
_TIE_CODES = {"src-joins-dst": TIE_SRC_JOINS_DST,
              "dst-joins-src": TIE_DST_JOINS_SRC,
              "skip": TIE_SKIP}
_MODES = {"deterministic": nat.DETERMINISTIC, "fast": nat.FAST}

WORKERS_ENV = "COMMVIZ_WORKERS"
DEFAULT_WORKERS = 4


def default_workers() -> int:
    """C/community.py:46-54."""
    try:
        return max(1, int(os.environ.get(WORKERS_ENV, DEFAULT_WORKERS)))
    except ValueError:
        return DEFAULT_WORKERS


class _History(list):
    """Per-round label snapshots; device tensors converted on access."""

    def __init__(self, items=()):
        if isinstance(items, _History):
            items = [items._dev(i) for i in range(len(items))]
        super().__init__(items)

    def __getitem__(self, i):
        v = super().__getitem__(i)
        if isinstance(i, slice):
            return [_as_host(x) for x in v]
        return _as_host(v)

    def __iter__(self):
        for i in range(len(self)):
            yield self[i]

    def _dev(self, i):
        return super().__getitem__(i)


def _as_host(x):
    if isinstance(x, np.ndarray):
        return x
    return nat.to_host(x).astype(np.int64, copy=False)


class CommunityAssignment:
    """Resolved labels, last-round counters, per-round history
    (C/community.py:57-67)."""

    def __init__(self, label, counter_degree, round_history=None):
        self._label = label if isinstance(label, Dual) else Dual(host=label)
        self._counter = counter_degree if isinstance(counter_degree, Dual) else Dual(host=counter_degree)
        if isinstance(round_history, _History):
            self.round_history = round_history  # keep device snapshots on device
        else:
            self.round_history = _History(round_history or [])

    label = property(lambda self: self._label.host(),
                     lambda self, v: self._label.set_host(v))
    counter_degree = property(lambda self: self._counter.host(),
                              lambda self, v: self._counter.set_host(v))

    def label_dev(self):
        return self._label.dev(nat.torch().int64)

    def counter_dev(self):
        return self._counter.dev(nat.torch().int64)

    @property
    def community_count(self) -> int:
        T = nat.torch()
        return int(T.unique(self.label_dev()).numel())


@dataclass(frozen=True)
class ThresholdSchedule:
    """Threshold base and round count (C/community.py:70-90)."""

    base: int
    rounds: int = 10

    def __post_init__(self):
        if self.base < 1:
            raise ValueError("threshold base must be positive")
        if self.rounds < 1:
            raise ValueError("round count must be positive")
        if self.base == 1:
            object.__setattr__(self, "base", 2)

    def threshold(self, i: int) -> int:
        return self.base ** i


def fresh_assignment(n: int) -> CommunityAssignment:
    """C/community.py:93-95."""
    return CommunityAssignment(label=np.arange(n, dtype=np.int64),
                               counter_degree=np.zeros(n, dtype=np.int64))


def make_schedule(m: int, workers: int, seed: int, interleave: str = "random") -> np.ndarray:
    """Processing order emulating `workers` chunked readers (C/community.py:164-195).

    Native (cvz_make_schedule, host C++): the seeded numpy Generator stream is
    replayed from the PCG64 state numpy's SeedSequence produces, so the order
    is the reference's bit-for-bit."""
    if interleave not in ("random", "roundrobin"):
        if workers > 1 and m >= 2:
            raise ValueError(f"unknown interleave {interleave!r}")
    out = np.empty(max(int(m), 0), dtype=np.int64)
    if workers <= 1 or m < 2:
        out[:] = np.arange(m, dtype=np.int64)
        return out
    st = np.random.default_rng(seed).bit_generator.state
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    m64 = (1 << 64) - 1
    rc = nat.load().cvz_make_schedule(int(m), int(workers), 0 if interleave == "random" else 1,
                                      s >> 64, s & m64, inc >> 64, inc & m64,
                                      int(st["has_uint32"]), int(st["uinteger"]),
                                      out.ctypes.data_as(ctypes.c_void_p))
    nat.check(rc, "cvz_make_schedule")
    return out


def _schedule_dev(m, workers, seed, interleave):
    """Processing order on the device, or None for the identity order."""
    if workers <= 1 or m < 2:
        return None
    return nat.to_dev(make_schedule(m, workers, seed, interleave), nat.torch().int64)


def _mode_code(mode):
    if mode not in _MODES:
        raise ValueError(f"unknown mode {mode!r}")
    return _MODES[mode]


def scoda_round(g, a: CommunityAssignment, threshold: int,
                tie_rule: str = "src-joins-dst", workers: int = 1,
                seed: int = 0, interleave: str = "random",
                mode: str = "deterministic") -> CommunityAssignment:
    """One streaming pass from assignment `a` (C/community.py:198-217)."""
    if threshold < 1:
        raise ValueError("threshold must be at least 1")
    if tie_rule not in _TIE_CODES:
        raise ValueError(f"unknown tie rule {tie_rule!r}")
    T = nat.torch()
    n = g.node_count
    deg = a.counter_dev().clone()
    lab = a.label_dev().clone()
    m = g.edge_count
    order = _schedule_dev(m, workers, seed, interleave)
    nat.call("cvz_scoda_pass", nat.ptr(g.edges_dev()), m, nat.ptr(order), n,
             int(threshold), _TIE_CODES[tie_rule], _mode_code(mode), nat.ptr(deg),
             nat.ptr(lab), None, nat.stream())
    hist = _History([a.round_history._dev(i) if isinstance(a.round_history, _History)
                     else a.round_history[i] for i in range(len(a.round_history))])
    return CommunityAssignment(label=Dual(dev=lab), counter_degree=Dual(dev=deg),
                               round_history=hist)


def _mode_degree(g) -> int:
    from .graph import _graph_stats
    if g.node_count == 0:
        return 1
    mode, _, _ = _graph_stats(g)
    return mode if mode > 0 else 1  # C/community.py:243-244


def detect_communities(g, schedule: ThresholdSchedule, seed: int = 0,
                       tie_rule: str = "src-joins-dst",
                       workers: int | None = None,
                       interleave: str = "random",
                       round_stream: str = "contract",
                       mode: str = "deterministic") -> CommunityAssignment:
    """Up to schedule.rounds GPU streaming passes (C/community.py:220-281).

    mode="deterministic" (default) reproduces the reference bit-exactly;
    mode="fast" runs the racy one-thread-per-edge pass (tolerance-gated) in
    the first round, where nearly every merge happens; later rounds only see
    the few communities still below the threshold and run the deterministic
    pass, so they stop as soon as nothing changes (the racy pass never lets
    labels settle and would run every scheduled round)."""
    if g.edge_count == 0:
        raise ValueError("cannot detect communities in an empty graph")
    if round_stream not in ("contract", "restream"):
        raise ValueError(f"unknown round_stream {round_stream!r}")
    if tie_rule not in _TIE_CODES:
        raise ValueError(f"unknown tie rule {tie_rule!r}")
    mcode = _mode_code(mode)
    if workers is None:
        workers = default_workers()
    T = nat.torch()
    dev = nat.device()
    n = g.node_count
    cap = max(_mode_degree(g), schedule.base)
    orig = g.edges_dev()
    m = int(orig.shape[0])
    bufs = [T.empty((max(m, 1), 2), dtype=T.int32, device=dev) for _ in range(2)]
    node_lab = T.arange(n, dtype=T.int64, device=dev)
    prev = T.empty(n, dtype=T.int64, device=dev)
    deg = T.zeros(n, dtype=T.int64, device=dev)
    history = []
    cur, m_cur = orig, m
    next_m = nat._I64(0)
    changed = ctypes.c_int(0)
    rs = 0 if round_stream == "contract" else 1
    streamed = []  # m_r per executed round (reference semantics; no reference counterpart)
    on_device = []  # edges the device actually streams per round (m_r minus dead edges)
    # Edges between two saturated communities are no-ops in every later round
    # once the threshold is pinned at its cap; with the identity order they
    # can leave the device stream (counted in `dead`, see cvz_detect_round).
    dead = 0
    next_dead = nat._I64(0)
    for i in range(1, schedule.rounds + 1):
        if m_cur + dead == 0:
            break
        streamed.append(m_cur + dead)
        on_device.append(m_cur)
        thr = min(schedule.threshold(i), cap)
        nthr = min(schedule.threshold(i + 1), cap)
        drop = workers <= 1 and rs == 0 and nthr == cap
        order = _schedule_dev(m_cur, workers, seed + i, interleave)
        snap = T.empty(n, dtype=T.int64, device=dev)
        out = bufs[(i - 1) % 2]
        nat.call("cvz_detect_round", nat.ptr(cur), m_cur, nat.ptr(order), nat.ptr(orig), m, n,
                 int(thr), _TIE_CODES[tie_rule], mcode if i == 1 else nat.DETERMINISTIC, i, rs,
                 nat.ptr(node_lab),
                 nat.ptr(prev), nat.ptr(deg), nat.ptr(snap), nat.ptr(out),
                 ctypes.byref(next_m), ctypes.byref(changed),
                 int(nthr) if drop else -1, ctypes.byref(next_dead), nat.stream())
        history.append(snap)
        if not changed.value:
            break
        cur, m_cur = out, int(next_m.value)
        dead += int(next_dead.value)
    a = CommunityAssignment(label=Dual(dev=node_lab), counter_degree=Dual(dev=deg),
                            round_history=_History(history))
    a.stream_edges = streamed
    a.device_stream_edges = on_device
    a._label.prefetch()  # the labels reach the host while later stages run
    return a


def export_hierarchy_tsv(a: CommunityAssignment, path) -> None:
    """C/community.py:284-294: node, label, one column per round (native
    multi-threaded formatting)."""
    from .render import format_table, write_text
    header = "\t".join(["node", "label"] + [f"round{i + 1}" for i in range(len(a.round_history))])
    body = format_table([None, a.label] + list(a.round_history)) if len(a.label) else b""
    write_text(path, header + "\n", body)


# ---- private kernel seams used by the reference's own tests -----------------

def _resolve_labels(lab) -> np.ndarray:
    """C/community.py:123-161 on the GPU."""
    T = nat.torch()
    d = nat.to_dev(np.asarray(lab, dtype=np.int64), T.int64)
    out = T.empty_like(d)
    nat.call("cvz_resolve_labels", nat.ptr(d), int(d.shape[0]), nat.ptr(out), nat.stream())
    return nat.to_host(out)


def _scoda_pass(edges, order, threshold, tie_code, deg, lab, mode="deterministic"):
    """C/community.py:98-120 on the GPU; updates numpy `deg`/`lab` in place
    (unresolved labels, like the reference kernel)."""
    T = nat.torch()
    e = nat.to_dev(np.asarray(edges, dtype=np.int64).reshape(-1, 2), T.int32)
    o = nat.to_dev(np.asarray(order, dtype=np.int64), T.int64)
    d = nat.to_dev(deg, T.int64)
    lab_d = nat.to_dev(lab, T.int64)
    raw = T.empty_like(lab_d)
    nat.call("cvz_scoda_pass", nat.ptr(e), int(o.shape[0]), nat.ptr(o), int(len(deg)),
             int(threshold), int(tie_code), _mode_code(mode), nat.ptr(d), nat.ptr(lab_d),
             nat.ptr(raw), nat.stream())
    deg[...] = nat.to_host(d)
    lab[...] = nat.to_host(raw)
