"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the BigGraphVis hot path.

A restatement of the reference package ``commviz`` (/root/reference/pkg/src,
cited as ``C/<file>:<line>``) in numpy + a small C library
(``oracle/csrc/oracle.c``, the sequential numba kernels restated).  It is the
checker for the CUDA product (tests/, ``__graft_entry__.smoke()``) and the
CPU baseline of ``bench.py``.  The product package never imports it.

Parity is PINNED: ``tests/golden/make_golden.py`` ran the real reference in
the build container and committed its outputs; ``tests/test_oracle_golden.py``
checks this oracle against them bit-exactly (integers) / to 1e-9 (floats).
"""

from __future__ import annotations

import ctypes
import math
import os
import warnings

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

MERSENNE_P = (1 << 31) - 1
_INT64_MAX = np.iinfo(np.int64).max
TIE_CODES = {"src-joins-dst": 0, "dst-joins-src": 1, "skip": 2}


def build(quiet: bool = True) -> str:
    """Compile oracle/csrc/oracle.c -> oracle/_build/liboracle.so (gcc)."""
    src = os.path.join(_HERE, "csrc", "oracle.c")
    os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
    if (not os.path.exists(_LIB_PATH)
            or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src)):
        cmd = (f"gcc -O2 -fopenmp -fPIC -shared -o {_LIB_PATH}.tmp {src} -lm"
               f" && mv {_LIB_PATH}.tmp {_LIB_PATH}")
        if os.system(cmd) != 0:
            raise RuntimeError("oracle build failed: " + cmd)
    return _LIB_PATH


def _L():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = ctypes.CDLL(_LIB_PATH)
        i64, dbl, p = ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
        _lib.orc_scoda_pass.argtypes = [p, p, i64, i64, ctypes.c_int, p, p]
        _lib.orc_resolve_labels.argtypes = [p, i64, p]
        _lib.orc_build_tree.argtypes = [p, p, i64, i64] + [p] * 11
        _lib.orc_build_tree.restype = i64
        _lib.orc_repulsion_bh.argtypes = [p, p, i64, dbl, dbl] + [p] * 10
        _lib.orc_repulsion_exact.argtypes = [p, p, i64, dbl, p]
        _lib.orc_attraction.argtypes = [p, p, i64, p, dbl, p]
        _lib.orc_num_threads.restype = ctypes.c_int
    return _lib


def _ptr(a):
    return a.ctypes.data if a is not None else None


def num_threads() -> int:
    return int(_L().orc_num_threads())


# ---------------------------------------------------------------- graph
def from_edge_array(edges, node_count=None):
    """C/graph.py:114-122.  Returns (node_count, edges (m,2) i64, degree)."""
    edges = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    edges = edges[edges[:, 0] != edges[:, 1]]
    if node_count is None:
        node_count = int(edges.max()) + 1 if len(edges) else 0
    degree = np.bincount(edges.ravel(), minlength=node_count).astype(np.int64)
    return node_count, edges, degree


def degree_stats(degree):
    """C/graph.py:125-136 -> (mode, mean, max)."""
    nz = degree[degree > 0]
    mode = int(np.argmax(np.bincount(nz)))
    return mode, float(degree.sum() / len(degree)), int(degree.max())


def parse_edge_list(text):
    """C/graph.py:50-92 (first-seen remap, self-loops dropped)."""
    if isinstance(text, bytes):
        text = text.decode("utf-8", errors="replace")
    remap, src, dst = {}, [], []
    for lineno, line in enumerate(text.splitlines(), start=1):
        s = line.strip()
        if not s or s[0] in "#%":
            continue
        parts = s.split()
        if len(parts) != 2:
            raise ValueError(f"line {lineno}: expected two tokens, got {len(parts)}")
        u, v = int(parts[0]), int(parts[1])
        if u == v:
            continue
        src.append(remap.setdefault(u, len(remap)))
        dst.append(remap.setdefault(v, len(remap)))
    if not src:
        raise ValueError("no edges")
    e = np.stack([np.asarray(src, np.int64), np.asarray(dst, np.int64)], axis=1)
    return len(remap), e, np.bincount(e.ravel(), minlength=len(remap)).astype(np.int64)


# ------------------------------------------------------------ community
def threshold(base, i):
    """C/community.py:70-90 (base 1 -> 2)."""
    return (2 if base == 1 else base) ** i


def make_schedule(m, workers, seed, interleave="random"):
    """C/community.py:164-195 restated (same numpy Generator draw sequence)."""
    if workers <= 1 or m < 2:
        return np.arange(m, dtype=np.int64)
    bounds = np.array([m * w // workers for w in range(workers + 1)], np.int64)
    if interleave == "roundrobin":
        off = np.arange(m, dtype=np.int64)
        chunk = np.searchsorted(bounds, off, side="right") - 1
        return np.lexsort((chunk, off - bounds[chunk])).astype(np.int64)
    if interleave != "random":
        raise ValueError(f"unknown interleave {interleave!r}")
    rng = np.random.default_rng(seed)
    ptr = bounds[:-1].copy()
    out = np.empty(m, dtype=np.int64)
    live = [w for w in range(workers) if bounds[w] < bounds[w + 1]]
    for k in range(m):
        w = live[rng.integers(len(live))]
        out[k] = ptr[w]
        ptr[w] += 1
        if ptr[w] >= bounds[w + 1]:
            live.remove(w)
    return out


def scoda_pass(edges, order, thr, tie, deg, lab):
    """C/community.py:98-120, in place on deg/lab (int64)."""
    edges = np.ascontiguousarray(edges, dtype=np.int64)
    order = None if order is None else np.ascontiguousarray(order, np.int64)
    assert deg.dtype == np.int64 and lab.dtype == np.int64
    _L().orc_scoda_pass(_ptr(edges), _ptr(order), len(edges) if order is None
                        else len(order), int(thr), int(tie), _ptr(deg), _ptr(lab))


def resolve_labels(lab):
    """C/community.py:123-161."""
    lab = np.ascontiguousarray(lab, dtype=np.int64)
    out = lab.copy()
    rc = _L().orc_resolve_labels(_ptr(lab), len(lab), _ptr(out))
    if rc != 0:
        raise ValueError("label out of range")
    return out


def scoda_round(edges, label, counter, thr, tie_rule="src-joins-dst",
                workers=1, seed=0, interleave="random"):
    """C/community.py:198-217 -> (label, counter)."""
    deg = np.asarray(counter, np.int64).copy()
    lab = np.asarray(label, np.int64).copy()
    order = make_schedule(len(edges), workers, seed, interleave)
    scoda_pass(edges, order, thr, TIE_CODES[tie_rule], deg, lab)
    return resolve_labels(lab), deg


def detect_communities(n, edges, degree, base, rounds=10, seed=0,
                       tie_rule="src-joins-dst", workers=1,
                       interleave="random", round_stream="contract",
                       stats=None):
    """C/community.py:220-281 -> (label, counter_degree, history)."""
    tie = TIE_CODES[tie_rule]
    nz = degree[degree > 0]
    mode = int(np.argmax(np.bincount(nz))) if len(nz) else 1
    base = 2 if base == 1 else base
    cap = max(mode, base)
    node_lab = np.arange(n, dtype=np.int64)
    cur = np.asarray(edges, np.int64)
    prev, history = None, []
    deg = np.zeros(n, dtype=np.int64)
    for i in range(1, rounds + 1):
        if len(cur) == 0:
            break
        thr = min(base ** i, cap)
        deg = np.zeros(n, dtype=np.int64)
        if i > 1:
            size = np.bincount(node_lab, minlength=n)
            np.minimum(size - 1, thr + 1, out=deg[:len(size)])
            np.maximum(deg, 0, out=deg)
        lab = np.arange(n, dtype=np.int64)
        order = make_schedule(len(cur), workers, seed + i, interleave)
        if stats is not None:
            stats.setdefault("m_r", []).append(len(cur))
            stats.setdefault("thr", []).append(thr)
        scoda_pass(cur, order, thr, tie, deg, lab)
        lab = resolve_labels(lab)
        node_lab = lab[node_lab]
        history.append(node_lab.copy())
        if prev is not None and np.array_equal(node_lab, prev):
            break
        prev = node_lab.copy()
        if round_stream == "contract":
            cu, cv = lab[cur[:, 0]], lab[cur[:, 1]]
        else:
            cu, cv = node_lab[edges[:, 0]], node_lab[edges[:, 1]]
        keep = cu != cv
        cur = np.stack([cu[keep], cv[keep]], axis=1)
    return node_lab, deg, history


# --------------------------------------------------------------- sketch
def sketch_params(rows, seed):
    """C/sketch.py:47-55 hash parameters (numpy default_rng)."""
    rng = np.random.default_rng(seed)
    a = rng.integers(1, MERSENNE_P, size=rows, dtype=np.int64)
    b = rng.integers(0, MERSENNE_P, size=rows, dtype=np.int64)
    return a, b


def default_cols(m, fraction=1e-4, min_cols=6500):
    """C/sketch.py:58-61."""
    return max(math.ceil(fraction * m), min_cols)


def sketch_indices(a, b, cols, keys):
    """C/sketch.py:39-44."""
    x = np.asarray(keys, dtype=np.int64) % np.int64(MERSENNE_P)
    return ((a[:, None] * x[None, :] + b[:, None]) % np.int64(MERSENNE_P)) % cols


def sketch_add_many(table, a, b, keys, amounts):
    """C/sketch.py:71-86 -> newly_saturated flag (table updated in place)."""
    keys = np.asarray(keys, np.int64)
    amounts = np.asarray(amounts, np.int64)
    if np.any(amounts < 0):
        raise ValueError("amounts must be non-negative")
    idx = sketch_indices(a, b, table.shape[1], keys)
    with np.errstate(over="ignore"):
        for r in range(table.shape[0]):
            np.add.at(table[r], idx[r], amounts)
    wrapped = table < 0
    if np.any(wrapped):
        table[wrapped] = _INT64_MAX
        return True
    return False


def sketch_estimate_many(table, a, b, keys):
    """C/sketch.py:93-98."""
    idx = sketch_indices(a, b, table.shape[1], keys)
    return table[np.arange(table.shape[0])[:, None], idx].min(axis=0)


# ----------------------------------------------------------- supergraph
def contract(edges, labels, table, a, b):
    """C/supergraph.py:49-76 -> (k, se_edges, weight, mult, comm_id)."""
    labels = np.asarray(labels, np.int64)
    comm, dense = np.unique(labels, return_inverse=True)
    weight = sketch_estimate_many(table, a, b, comm)
    cu, cv = dense[edges[:, 0]], dense[edges[:, 1]]
    cross = cu != cv
    lo = np.minimum(cu[cross], cv[cross])
    hi = np.maximum(cu[cross], cv[cross])
    if len(lo):
        # np.unique(pairs, axis=0) order == numeric order of lo*k + hi (hi < k)
        kk = np.int64(len(comm))
        keys, mult = np.unique(lo * kk + hi, return_counts=True)
        uniq = np.stack([keys // kk, keys % kk], axis=1)
    else:
        uniq, mult = np.empty((0, 2), np.int64), np.empty(0, np.int64)
    return (len(comm), uniq.astype(np.int64), weight.astype(np.int64),
            mult.astype(np.int64), comm)


# --------------------------------------------------------------- layout
def init_positions(n, seed=0):
    """C/layout.py:78-82."""
    side = max(np.sqrt(n), 1.0)
    return np.random.default_rng(seed).uniform(-side / 2, side / 2, size=(n, 2))


def build_tree(pos, mass):
    """C/layout.py:97-212 with the cap-doubling retry of :319-324."""
    pos = np.ascontiguousarray(pos, np.float64)
    mass = np.ascontiguousarray(mass, np.float64)
    n = len(pos)
    cap = max(256, 4 * n)
    L = _L()
    while True:
        t = dict(children=np.empty((cap, 4), np.int64), kind=np.empty(cap, np.int8),
                 cmass=np.empty(cap), csumx=np.empty(cap), csumy=np.empty(cap),
                 ccount=np.empty(cap, np.int64), cx=np.empty(cap), cy=np.empty(cap),
                 chalf=np.empty(cap), leaf_body=np.empty(cap, np.int64),
                 body_cell=np.empty(n, np.int64))
        used = L.orc_build_tree(
            _ptr(pos), _ptr(mass), n, cap, _ptr(t["children"]), _ptr(t["kind"]),
            _ptr(t["cmass"]), _ptr(t["csumx"]), _ptr(t["csumy"]),
            _ptr(t["ccount"]), _ptr(t["cx"]), _ptr(t["cy"]), _ptr(t["chalf"]),
            _ptr(t["leaf_body"]), _ptr(t["body_cell"]))
        if used != -1:
            t["used"] = int(used)
            return t
        cap *= 2


def repulsion_forces(pos, mass, repulsion=80.0, theta=0.5):
    """C/layout.py:312-328."""
    pos = np.ascontiguousarray(pos, np.float64)
    mass = np.ascontiguousarray(mass, np.float64)
    out = np.zeros_like(pos)
    L = _L()
    if theta <= 0:
        L.orc_repulsion_exact(_ptr(pos), _ptr(mass), len(pos), float(repulsion), _ptr(out))
        return out
    t = build_tree(pos, mass)
    L.orc_repulsion_bh(_ptr(pos), _ptr(mass), len(pos), float(repulsion), float(theta),
                       _ptr(t["children"]), _ptr(t["kind"]), _ptr(t["cmass"]),
                       _ptr(t["csumx"]), _ptr(t["csumy"]), _ptr(t["ccount"]),
                       _ptr(t["chalf"]), _ptr(t["leaf_body"]), _ptr(t["body_cell"]),
                       _ptr(out))
    return out


def attraction(pos, edges, weight, sign, out):
    """C/layout.py:293-304 (accumulates into out)."""
    pos = np.ascontiguousarray(pos, np.float64)
    edges = np.ascontiguousarray(edges, np.int64)
    weight = np.ascontiguousarray(weight, np.float64)
    _L().orc_attraction(_ptr(pos), _ptr(edges), len(edges), _ptr(weight),
                        float(sign), _ptr(out))


def masses_supergraph(weight, multiplicity):
    """C/layout.py:331-335."""
    return (np.maximum(weight, 1).astype(np.float64),
            np.asarray(multiplicity).astype(np.float64))


def masses_graph(degree, m):
    """C/layout.py:336-338."""
    return (degree + 1).astype(np.float64), np.ones(m, np.float64)


def layout_step(pos, prev_force, speed, mass, edges, edge_weight, *,
                gravity=1.0, repulsion=80.0, jitter_tolerance=1.0, theta=0.5,
                max_step=10.0, speed_form="product", attraction_form="canonical"):
    """One iteration of C/layout.py:367-399 with explicit state.

    Returns (new_pos, force, speed, max_disp, finite)."""
    force = repulsion_forces(pos, mass, repulsion, theta)
    attraction(pos, edges, edge_weight,
               1.0 if attraction_form == "canonical" else -1.0, force)
    if gravity > 0:
        force += -gravity * mass[:, None] * pos
    diff = np.hypot(force[:, 0] - prev_force[:, 0], force[:, 1] - prev_force[:, 1])
    tot = np.hypot(force[:, 0] + prev_force[:, 0], force[:, 1] + prev_force[:, 1])
    swing = mass * diff
    traction = mass * tot / 2.0
    total_swing = swing.sum()
    if total_swing > 0:
        speed = min(jitter_tolerance * traction.sum() / total_swing, 1.5 * speed)
    if speed_form == "product":
        local = speed / (1.0 + np.sqrt(speed * swing))
    else:
        local = speed / (1.0 + np.sqrt(speed + swing))
    disp = force * local[:, None]
    norms = np.hypot(disp[:, 0], disp[:, 1])
    over = norms > max_step
    if over.any():
        disp[over] *= (max_step / norms[over])[:, None]
        norms[over] = max_step
    new = pos + disp
    return new, force, speed, float(norms.max()), bool(np.isfinite(new).all())


def layout(n, mass, edges, edge_weight, iterations=100, positions=None, seed=0,
           **params):
    """C/layout.py:341-402 -> (positions, displacement history)."""
    pos = init_positions(n, seed) if positions is None else np.array(positions, np.float64)
    if n == 1:
        return pos, np.zeros(iterations)
    prev = np.zeros((n, 2))
    speed = 1.0
    hist = np.zeros(iterations)
    for it in range(iterations):
        pos, prev, speed, hist[it], ok = layout_step(pos, prev, speed, mass, edges,
                                                     edge_weight, **params)
        if not ok:
            raise FloatingPointError(f"non-finite positions at iteration {it + 1}")
    return pos, hist


# --------------------------------------------------------------- metrics
def modularity(edges, degree, labels):
    """C/metrics.py:34-46."""
    m = len(edges)
    uniq, inv = np.unique(labels, return_inverse=True)
    cu, cv = inv[edges[:, 0]], inv[edges[:, 1]]
    intra = np.bincount(cu[cu == cv], minlength=len(uniq))
    degsum = np.bincount(inv, weights=degree.astype(np.float64), minlength=len(uniq))
    return float(np.sum(intra / m - (degsum / (2.0 * m)) ** 2))


def supergraph_pipeline(edges, n, degree, *, rounds=10, seed=0, workers=1,
                        sketch_rows=4, iterations=100, stats=None):
    """Stages of C/cli.py:126-147 on in-memory arrays (no parse / render)."""
    mode = degree_stats(degree)[0]
    label, _, hist = detect_communities(n, edges, degree, mode, rounds, seed,
                                        workers=workers, stats=stats)
    a, b = sketch_params(sketch_rows, seed)
    table = np.zeros((sketch_rows, default_cols(len(edges))), np.int64)
    sketch_add_many(table, a, b, label, degree)
    k, se, w, mult, comm = contract(edges, label, table, a, b)
    mass, ew = masses_supergraph(w, mult)
    pos, disp = layout(k, mass, se, ew, iterations=iterations, seed=seed)
    return dict(label=label, rounds=len(hist), k=k, se=se, weight=w, mult=mult,
                comm=comm, pos=pos, disp=disp)
