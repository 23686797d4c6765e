"""Size-rank coloring and SVG export (drop-in for C/render.py), plus the
native table writer the TSV exports share.

The small per-supernode arithmetic (ranking, radii) is numpy exactly as the
reference states it; the text output -- the only part that scales with the
graph -- is formatted by multi-threaded C++ in libcvz_b200.so
(cvz_format_table / cvz_format_svg), byte-identical to the reference's
f-string loops.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat

PALETTE = (
    "#b15928", "#cab2d6", "#6a3d9a", "#fdbf6f", "#ff7f00", "#fb9a99",
    "#e31a1c", "#b2df8a", "#33a02c", "#a6cee3", "#1f78b4",
)  # C/render.py:17-29: class 0 brown, then 10 ascending size classes
CLASS_COUNT = len(PALETTE)
MIN_RADIUS = 0.5
RADIUS_FRACTION = 0.03


@dataclass(frozen=True)
class ColorAssignment:
    """C/render.py:36-42."""

    classes: np.ndarray
    palette: tuple = PALETTE

    def color(self, i: int) -> str:
        return self.palette[int(self.classes[i])]


def assign_colors(weights, alpha: float = 1.0) -> ColorAssignment:
    """C/render.py:45-66: the lightest supernodes holding <= alpha/2 of the
    total weight are class 0; the rest split into 10 ascending equal-count
    classes, the remainder going to the heaviest classes."""
    if not 0 < alpha <= 2:
        raise ValueError("alpha must be in (0, 2]")
    w = np.asarray(weights, dtype=np.float64)
    n = len(w)
    if n == 0:
        raise ValueError("cannot color an empty weight vector")
    order = np.argsort(w, kind="stable")
    csum = np.cumsum(w[order])
    brown = int(np.searchsorted(csum, alpha / 2 * csum[-1], side="right"))
    classes = np.zeros(n, dtype=np.int64)
    rest = n - brown
    if rest > 0:
        per = np.full(10, rest // 10, dtype=np.int64)
        per[10 - rest % 10:] += 1
        classes[order[brown:]] = np.repeat(np.arange(1, 11, dtype=np.int64), per)
    return ColorAssignment(classes=classes)


def radius_scale(positions, weights) -> float:
    """C/render.py:69-75: heaviest radius = 3% of the layout diameter."""
    positions = np.asarray(positions, dtype=np.float64)
    span = positions.max(axis=0) - positions.min(axis=0)
    diameter = float(np.hypot(span[0], span[1]))
    max_w = float(np.max(weights))
    if diameter <= 0 or max_w <= 0:
        return 1.0
    return RADIUS_FRACTION * diameter / np.sqrt(max_w)


def node_radii(positions, weights) -> np.ndarray:
    """C/render.py:78-81."""
    s = radius_scale(positions, weights)
    return np.maximum(s * np.sqrt(np.asarray(weights, dtype=np.float64)), MIN_RADIUS)


def color_full_graph(labels, community_id, colors: ColorAssignment) -> np.ndarray:
    """C/render.py:84-93: every original node gets its community's class
    (vectorised lookup; a label with no supernode raises like the reference)."""
    labels = np.asarray(getattr(labels, "label", labels), dtype=np.int64)
    cid = np.asarray(community_id, dtype=np.int64)
    order = np.argsort(cid, kind="stable")
    pos = np.searchsorted(cid[order], labels)
    pos_c = np.minimum(pos, max(len(cid) - 1, 0))
    ok = (pos < len(cid)) & (cid[order][pos_c] == labels) if len(cid) else np.zeros(
        len(labels), bool)
    if not np.all(ok):
        i = int(np.argmin(ok))
        raise ValueError(f"node {i} has label {int(labels[i])} with no color class")
    return np.asarray(colors.classes, dtype=np.int64)[order[pos_c]]


# ------------------------------------------------------------- native text
def _take(h, nbytes) -> bytes:
    buf = ctypes.create_string_buffer(nbytes.value)
    nat.check(nat.load().cvz_text_take(h, buf), "cvz_text_take")
    return buf.raw[:nbytes.value]


def format_table(columns, sep: str = "\t") -> bytes:
    """Rows of `sep`-separated columns; each column is an int64 array, a
    float64 array (formatted "%.3f") or None (the row index)."""
    n = None
    kinds, keep, ptrs = [], [], []
    for c in columns:
        if c is None:
            kinds.append(2)
            ptrs.append(None)
            continue
        a = np.asarray(c)
        if a.dtype.kind == "f":
            a = np.ascontiguousarray(a, dtype=np.float64)
            kinds.append(1)
        else:
            a = np.ascontiguousarray(a, dtype=np.int64)
            kinds.append(0)
        n = len(a) if n is None else n
        if len(a) != n:
            raise ValueError("columns must have equal length")
        keep.append(a)
        ptrs.append(a.ctypes.data)
    if n is None:
        raise ValueError("need at least one data column")
    karr = (ctypes.c_int * len(kinds))(*kinds)
    parr = (ctypes.c_void_p * len(ptrs))(*ptrs)
    h, nbytes = ctypes.c_void_p(), ctypes.c_int64(0)
    nat.check(nat.load().cvz_format_table(n, len(kinds), karr, parr, sep.encode()[0],
                                          ctypes.byref(h), ctypes.byref(nbytes)),
              "cvz_format_table")
    return _take(h, nbytes)


def write_text(path, header: str, body: bytes) -> None:
    """Write header + body to a path or an open text/binary file."""
    if hasattr(path, "write"):
        try:
            path.write(header + body.decode("ascii"))
        except TypeError:
            path.write(header.encode("ascii") + body)
        return
    with open(path, "wb") as fh:
        fh.write(header.encode("ascii"))
        fh.write(body)


def export_svg(path, positions, radii, colors: ColorAssignment, edges=None,
               multiplicity=None, margin: float = 0.05) -> None:
    """C/render.py:96-139: deterministic SVG, edges under nodes, nodes drawn
    in (class, index) order, every float "%.3f"."""
    positions = np.ascontiguousarray(positions, dtype=np.float64)
    radii = np.ascontiguousarray(radii, dtype=np.float64)
    classes = np.ascontiguousarray(colors.classes, dtype=np.int64)
    n = len(positions)
    if len(radii) != n or len(classes) != n:
        raise ValueError("positions, radii and classes must align")
    ne, e_ptr, m_ptr = 0, None, None
    if edges is not None and len(edges):
        e = np.ascontiguousarray(edges, dtype=np.int64).reshape(-1, 2)
        ne, e_ptr = len(e), e.ctypes.data
        if multiplicity is not None:
            mult = np.ascontiguousarray(multiplicity, dtype=np.float64)
            m_ptr = mult.ctypes.data
    pal = (ctypes.c_char_p * len(colors.palette))(*[p.encode() for p in colors.palette])
    h, nbytes = ctypes.c_void_p(), ctypes.c_int64(0)
    nat.check(nat.load().cvz_format_svg(n, positions.ctypes.data, radii.ctypes.data,
                                        classes.ctypes.data, pal, len(colors.palette), ne,
                                        e_ptr, m_ptr, float(margin), ctypes.byref(h),
                                        ctypes.byref(nbytes)), "cvz_format_svg")
    text = _take(h, nbytes)
    if hasattr(path, "write"):
        path.write(text.decode("utf-8"))
    else:
        with open(path, "wb") as fh:
            fh.write(text)


def export_nodes_tsv(path, g, assignment, sg, colors: ColorAssignment, result,
                     full: bool = False) -> None:
    """nodes.tsv of C/cli.py:200-215: node, community, supernode, class and
    the drawn position (the supernode's, or the node's own in full mode)."""
    lab = np.asarray(getattr(assignment, "label", assignment), dtype=np.int64)
    cid = np.asarray(sg.community_id, dtype=np.int64)
    s = np.searchsorted(cid, lab)
    if len(cid) == 0 or np.any(s >= len(cid)) or np.any(cid[np.minimum(s, len(cid) - 1)] != lab):
        raise KeyError("a node's label has no supernode")
    k = np.asarray(colors.classes, dtype=np.int64)[s]
    pos = np.asarray(result.positions, dtype=np.float64)
    xy = pos if full else pos[s]
    body = format_table([None, lab, s, k, xy[:, 0], xy[:, 1]])
    write_text(path, "node\tcommunity\tsupernode\tclass\tx\ty\n", body)
