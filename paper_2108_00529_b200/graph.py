"""Graph ingestion (drop-in for C/graph.py).

`from_edge_array` and `degree_stats` run on the GPU (cvz_edges_compact,
cvz_degree_count, cvz_degree_stats).  The edge list stays on the device as
int32 pairs in stream order; `Graph.edges` / `Graph.degree` materialise int64
numpy arrays only when read.
"""

from __future__ import annotations

import ctypes
import io
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from ._dual import Dual


class ParseError(ValueError):
    """C/graph.py:20-21."""


class Graph:
    """Immutable undirected multigraph over dense ids (C/graph.py:24-40)."""

    __slots__ = ("node_count", "_edges", "_degree", "_edges32", "_stats")

    def __init__(self, node_count: int, edges, degree):
        edges = np.asarray(edges)
        degree = np.asarray(degree)
        if edges.ndim != 2 or edges.shape[1] != 2:
            raise ValueError("edges must be an (m, 2) array")
        if int(degree.sum()) != 2 * len(edges):
            raise ValueError("degree sum must equal twice the edge count")
        self.node_count = int(node_count)
        self._edges = Dual(host=edges)
        self._degree = Dual(host=degree)
        self._edges32 = None
        self._stats = None

    @classmethod
    def _from_device(cls, n: int, edges32, degree64):
        g = object.__new__(cls)
        g.node_count = int(n)
        g._edges = Dual(dev=edges32)
        g._degree = Dual(dev=degree64)
        g._edges32 = edges32
        g._stats = None
        return g

    @property
    def edges(self) -> np.ndarray:
        return self._edges.host()

    @property
    def degree(self) -> np.ndarray:
        return self._degree.host()

    @property
    def edge_count(self) -> int:
        return len(self._edges)

    # device views used by the kernels
    def edges_dev(self):
        """(m, 2) int32 CUDA tensor in stream order."""
        if self._edges32 is None:
            T = nat.torch()
            e = self._edges.host()
            if len(e) and (e.min() < 0 or e.max() >= 2**31):
                raise ValueError("node ids must lie in [0, 2^31)")
            self._edges32 = nat.to_dev(e.reshape(-1, 2), T.int32)
        return self._edges32

    def degree_dev(self):
        return self._degree.dev(nat.torch().int64)

    def __repr__(self):
        return f"Graph(node_count={self.node_count}, edge_count={self.edge_count})"


@dataclass(frozen=True)
class DegreeStats:
    """C/graph.py:43-47."""

    mode_degree: int
    average_degree: float
    max_degree: int


def _parse_lines(lines) -> Graph:
    """The reference's line loop (C/graph.py:65-92), used for inputs outside
    the native tokenizer's subset (non-ASCII text, ids beyond int64, line
    iterables).  Tokenising is host work; degrees run on the GPU."""
    ids: dict[int, int] = {}
    flat: list[int] = []
    for no, raw in enumerate(lines, start=1):
        s = raw.strip()
        if not s or s[0] in "#%":
            continue
        tok = s.split()
        if len(tok) != 2:
            raise ParseError(f"line {no}: expected two tokens, got {len(tok)}")
        try:
            a, b = int(tok[0]), int(tok[1])
        except ValueError:
            raise ParseError(f"line {no}: non-integer token") from None
        if a == b:
            continue
        flat.append(ids.setdefault(a, len(ids)))
        flat.append(ids.setdefault(b, len(ids)))
    if not flat:
        raise ParseError("no edges")
    return from_edge_array(np.asarray(flat, dtype=np.int64).reshape(-1, 2),
                           node_count=len(ids))


def _parse_native(data: bytes):
    """Multi-threaded C++ tokenizer (cvz_parse_begin/take) + GPU first-seen
    remap (cvz_first_seen_remap).  Returns None when the text is outside the
    native subset (the caller then runs the reference's loop)."""
    T = nat.torch()
    lib = nat.load()
    h = ctypes.c_void_p()
    m, el = ctypes.c_int64(0), ctypes.c_int64(0)
    ec, et = ctypes.c_int(0), ctypes.c_int(0)
    nat.check(lib.cvz_parse_begin(data, len(data), 0, ctypes.byref(h), ctypes.byref(m),
                                  ctypes.byref(el), ctypes.byref(ec), ctypes.byref(et)),
              "cvz_parse_begin")
    if ec.value == 3:
        return None
    if ec.value == 1:
        raise ParseError(f"line {el.value}: expected two tokens, got {et.value}")
    if ec.value == 2:
        raise ParseError(f"line {el.value}: non-integer token")
    if m.value == 0:
        lib.cvz_parse_take(h, None)
        raise ParseError("no edges")
    ext_h = T.empty(2 * m.value, dtype=T.int64).pin_memory()
    nat.check(lib.cvz_parse_take(h, ctypes.c_void_p(ext_h.data_ptr())), "cvz_parse_take")
    ext = ext_h.to(nat.device(), non_blocking=True)
    dense = T.empty((m.value, 2), dtype=T.int32, device=nat.device())
    n = ctypes.c_int64(0)
    nat.call("cvz_first_seen_remap", nat.ptr(ext), 2 * m.value, nat.ptr(dense),
             ctypes.byref(n), nat.stream())
    return from_edge_array(dense, node_count=n.value)


def parse_edge_list(text) -> Graph:
    """C/graph.py:50-92: SNAP-style text -> Graph (first-seen id remap,
    comments `#`/`%`, self-loops dropped, duplicates kept).

    str/bytes go through the native tokenizer + GPU remap (SURVEY.md 8f
    row 1); line iterables and non-ASCII text through the reference loop."""
    if isinstance(text, (bytes, bytearray, memoryview)):
        g = _parse_native(bytes(text))
        if g is not None:
            return g
        text = bytes(text).decode("utf-8", errors="replace")
    if isinstance(text, str):
        if text.isascii():
            g = _parse_native(text.encode("ascii"))
            if g is not None:
                return g
        return _parse_lines(text.splitlines())
    return _parse_lines([ln.decode() if isinstance(ln, bytes) else ln for ln in text])


# Binary edge cache (SPEC.md:77 permits "magic bytes, version, node_count,
# edge array").  Little-endian: 8-byte magic, u32
# version, u32 flags (bit 0: int64 ids), i64 node_count, i64 edge_count, then
# the (edge_count, 2) dense-id edge array in stream order (self-loops already
# dropped).  Reading it skips tokenising and remapping altogether.
CACHE_MAGIC = b"CVZEDGE\0"
CACHE_VERSION = 1
_CACHE_HDR = 8 + 4 + 4 + 8 + 8


def _write_cache_arrays(path, node_count: int, edges: np.ndarray) -> None:
    edges = np.asarray(edges).reshape(-1, 2)
    wide = bool(len(edges)) and int(edges.max()) >= 2**31
    body = np.ascontiguousarray(edges, dtype="<i8" if wide else "<i4")
    hdr = (CACHE_MAGIC + np.array([CACHE_VERSION, int(wide)], "<u4").tobytes()
           + np.array([node_count, len(body)], "<i8").tobytes())
    with open(path, "wb") as fh:
        fh.write(hdr)
        body.tofile(fh)


def _read_cache_arrays(path):
    """-> (node_count, (m, 2) int32/int64 edges); ParseError on a bad file."""
    with open(path, "rb") as fh:
        hdr = fh.read(_CACHE_HDR)
        if len(hdr) < _CACHE_HDR or hdr[:8] != CACHE_MAGIC:
            raise ParseError("not a commviz edge cache")
        version, flags = (int(v) for v in np.frombuffer(hdr[8:16], "<u4"))
        n, m = (int(v) for v in np.frombuffer(hdr[16:32], "<i8"))
        if version != CACHE_VERSION:
            raise ParseError(f"edge cache version {version} (expected {CACHE_VERSION})")
        if n < 0 or m < 0:
            raise ParseError("edge cache: negative sizes")
        dt = np.dtype("<i8" if flags & 1 else "<i4")
        body = np.fromfile(fh, dtype=dt, count=2 * m)
    if body.size != 2 * m:
        raise ParseError(f"edge cache truncated: {body.size // 2} of {m} edges")
    edges = body.reshape(m, 2)
    if m and (int(edges.min()) < 0 or int(edges.max()) >= n):
        raise ParseError("edge cache: id outside [0, node_count)")
    return n, edges


def write_edge_cache(g: Graph, path) -> None:
    """Write `g` (dense ids, stream order) as a binary edge cache that
    `load_edge_list` reads back without parsing."""
    _write_cache_arrays(path, g.node_count, g.edges)


def read_edge_cache(path) -> Graph:
    """Binary edge cache -> Graph (same node count, edges and degrees as the
    graph that was written); the edges go straight to the GPU ingest."""
    n, edges = _read_cache_arrays(path)
    if len(edges) == 0:
        raise ParseError("no edges")  # as for text (C/graph.py:86)
    return from_edge_array(edges, node_count=n)


def load_edge_list(path) -> Graph:
    """C/graph.py:95-97 (file bytes straight to the native tokenizer; a
    non-ASCII file is decoded as utf-8 text exactly like the reference).  A
    binary edge cache (`write_edge_cache`) is recognised by its magic."""
    with open(path, "rb") as fh:
        if fh.read(len(CACHE_MAGIC)) == CACHE_MAGIC:
            return read_edge_cache(path)
        fh.seek(0)
        data = fh.read()
    if data.isascii():
        g = _parse_native(data)
        if g is not None:
            return g
    with open(path, "r", encoding="utf-8") as fh:
        return _parse_lines(fh.read().splitlines())


def write_edge_list(g: Graph, path_or_file) -> None:
    """C/graph.py:100-111: dense ids, stream order, one `u v` per line
    (native multi-threaded formatting)."""
    from .render import format_table
    e = g.edges
    body = format_table([e[:, 0], e[:, 1]], sep=" ") if len(e) else b""
    own = isinstance(path_or_file, (str, bytes)) or hasattr(path_or_file, "__fspath__")
    if own:
        with open(path_or_file, "wb") as fh:
            fh.write(body)
    else:
        path_or_file.write(body.decode("ascii"))


def upload_edges(edges):
    """A host (m, 2) edge array (the reference's int64 numpy input, or int32;
    pageable or pinned) as an (m, 2) int32 CUDA tensor: range-checked and
    narrowed on the host into page-locked staging buffers whose DMA overlaps
    the next chunk's conversion (cvz_edges_upload)."""
    T = nat.torch()
    arr = np.asarray(edges)
    if arr.dtype not in (np.int32, np.int64):
        arr = np.asarray(arr, dtype=np.int64)
    arr = np.ascontiguousarray(arr).reshape(-1, 2)
    m = int(arr.shape[0])
    dev = T.empty((max(m, 1), 2), dtype=T.int32, device=nat.device())
    nat.call("cvz_edges_upload", arr.ctypes.data_as(ctypes.c_void_p),
             int(arr.dtype == np.int32), m, nat.ptr(dev), nat.stream())
    return dev[:m]


def from_edge_array(edges, node_count=None) -> Graph:
    """C/graph.py:114-122 on the GPU: stable self-loop drop + degree histogram.

    `edges` may be any (m, 2)-shaped integer array, or a CUDA tensor
    (int32/int64) already in HBM."""
    T = nat.torch()
    if isinstance(edges, T.Tensor):
        src = edges.reshape(-1, 2)
        if src.dtype not in (T.int32, T.int64) or not src.is_cuda:
            src = nat.to_dev(src, T.int64)
        src = src.contiguous()
    else:
        src = upload_edges(edges)
    m_in = int(src.shape[0])
    out = T.empty((max(m_in, 1), 2), dtype=T.int32, device=nat.device())
    scal = T.zeros(2, dtype=T.int64, device=nat.device())
    nat.call("cvz_edges_compact", nat.ptr(src), int(src.dtype == T.int32), m_in,
             nat.ptr(out), nat.ptr(scal), nat.ptr(scal[1:]), 1, nat.stream())
    m, mx = nat.read_ints(scal)
    if node_count is None:
        n = mx + 1 if m else 0
    else:
        n = int(node_count)
    nbins = max(n, mx + 1) if m else n  # np.bincount(minlength=n) grows to max+1
    degree = T.empty(max(nbins, 1), dtype=T.int64, device=nat.device())
    nat.call("cvz_degree_count", nat.ptr(out), m, nbins, nat.ptr(degree), nat.stream())
    return Graph._from_device(n, out[:m], degree[:nbins])


def _stats_dev(degree_dev, n):
    T = nat.torch()
    out = T.empty(3, dtype=T.int64, device=nat.device())
    nat.call("cvz_degree_stats", nat.ptr(degree_dev), int(degree_dev.shape[0]),
             nat.ptr(out), nat.stream())
    return nat.read_ints(out)


def _graph_stats(g: Graph):
    """(mode of nonzero degrees, degree sum, max degree), computed once per
    Graph while its degrees live only on the device (detect_communities
    needs the mode again after degree_stats; a host copy the caller could
    mutate disables the cache)."""
    if not g._degree.on_device:
        return _stats_dev(g.degree_dev(), g.node_count)
    if g._stats is None:
        g._stats = tuple(_stats_dev(g.degree_dev(), g.node_count))
    return g._stats


def degree_stats(g: Graph) -> DegreeStats:
    """C/graph.py:125-136 on the GPU (mode of nonzero degrees, ties -> smaller)."""
    if g.edge_count == 0:
        raise ValueError("degree stats undefined for a graph with no edges")
    mode, total, mx = _graph_stats(g)
    return DegreeStats(mode_degree=mode,
                       average_degree=float(np.int64(total) / g.node_count),
                       max_degree=mx)
