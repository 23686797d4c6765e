"""Count-min sketch (drop-in for C/sketch.py); table lives in HBM.

Hash parameters come from numpy's seeded Generator on the host exactly as
in the reference (C/sketch.py:50-52) and are uploaded; all hashing, adding,
saturation and estimation run in cvz_sketch_* kernels.
"""

from __future__ import annotations

import functools
import math
import warnings

import numpy as np

from . import _native as nat
from ._dual import Dual

MERSENNE_P = np.int64((1 << 31) - 1)
DEFAULT_ROWS = 4
DEFAULT_COL_FRACTION = 1e-4
DEFAULT_MIN_COLS = 6500
_INT64_MAX = np.iinfo(np.int64).max


class CountMinSketch:
    """rows x cols int64 counters + per-row Carter-Wegman hashes
    (C/sketch.py:30-44)."""

    def __init__(self, rows: int, cols: int, table, hash_a, hash_b, saturated: bool = False):
        self.rows = int(rows)
        self.cols = int(cols)
        self._table = table if isinstance(table, Dual) else Dual(host=table)
        self.hash_a = np.asarray(hash_a, dtype=np.int64)
        self.hash_b = np.asarray(hash_b, dtype=np.int64)
        self.saturated = bool(saturated)
        self._ab_dev = None

    table = property(lambda self: self._table.host(), lambda self, v: self._table.set_host(v))

    def table_dev(self):
        t = self._table.dev(nat.torch().int64)
        if not self._table.on_device:  # host copy was authoritative: adopt the upload
            self._table.set_dev(t)
        return t

    def _hash_dev(self):
        if self._ab_dev is None:
            self._ab_dev = _hash_params_dev(self.hash_a.tobytes(), self.hash_b.tobytes(),
                                            nat.device().index)
        return self._ab_dev

    def _indices(self, keys) -> np.ndarray:
        """Per-row column indices, shape (rows, len(keys)) (C/sketch.py:39-44)."""
        T = nat.torch()
        k = nat.to_dev(np.asarray(keys, dtype=np.int64), T.int64)
        out = T.empty((self.rows, int(k.shape[0])), dtype=T.int64, device=nat.device())
        a, b = self._hash_dev()
        nat.call("cvz_sketch_indices", nat.ptr(a), nat.ptr(b), self.rows, self.cols,
                 nat.ptr(k), int(k.shape[0]), nat.ptr(out), nat.stream())
        return nat.to_host(out)


@functools.lru_cache(maxsize=64)
def _hash_params_dev(a_bytes: bytes, b_bytes: bytes, device_index):
    """Device copies of one sketch's hash parameters, shared by every sketch
    with the same parameters (read-only in the kernels); uploaded once from
    pinned memory without a host sync."""
    T = nat.torch()
    out = []
    for raw in (a_bytes, b_bytes):
        h = T.from_numpy(np.frombuffer(raw, dtype=np.int64).copy()).pin_memory()
        out.append(h.to(device=nat.device(), non_blocking=True))
    return tuple(out)


@functools.lru_cache(maxsize=64)
def _hash_params(rows: int, seed):
    """numpy's seeded draws (C/sketch.py:50-52), memoised per (rows, seed)."""
    rng = np.random.default_rng(seed)
    a = rng.integers(1, int(MERSENNE_P), size=rows, dtype=np.int64)
    b = rng.integers(0, int(MERSENNE_P), size=rows, dtype=np.int64)
    a.flags.writeable = False
    b.flags.writeable = False
    return a, b


def sketch_new(rows: int, cols: int, seed: int) -> CountMinSketch:
    """C/sketch.py:47-55."""
    if rows < 1 or cols < 1:
        raise ValueError("sketch needs at least one row and one column")
    if isinstance(seed, (int, np.integer)):
        a, b = (x.copy() for x in _hash_params(int(rows), int(seed)))
    else:  # SeedSequence / Generator seeds: not hashable for the memo
        rng = np.random.default_rng(seed)
        a = rng.integers(1, int(MERSENNE_P), size=rows, dtype=np.int64)
        b = rng.integers(0, int(MERSENNE_P), size=rows, dtype=np.int64)
    T = nat.torch()
    table = T.zeros((rows, cols), dtype=T.int64, device=nat.device())
    return CountMinSketch(rows=rows, cols=cols, table=Dual(dev=table), hash_a=a, hash_b=b)


def default_cols(edge_count: int, fraction: float = DEFAULT_COL_FRACTION,
                 min_cols: int = DEFAULT_MIN_COLS) -> int:
    """C/sketch.py:58-61."""
    return max(math.ceil(fraction * edge_count), min_cols)


def sketch_add(s: CountMinSketch, key: int, amount: int) -> None:
    """C/sketch.py:64-68."""
    if amount < 0:
        raise ValueError("amount must be non-negative")
    sketch_add_many(s, np.asarray([key], dtype=np.int64), np.asarray([amount], dtype=np.int64))


def _dev64(x):
    T = nat.torch()
    if isinstance(x, T.Tensor):
        return x.to(device=nat.device(), dtype=T.int64).contiguous(), None
    h = np.asarray(x, dtype=np.int64).ravel()
    return nat.to_dev(h, T.int64), h


def sketch_add_many(s: CountMinSketch, keys, amounts, _nonneg: bool = False) -> None:
    """Bulk weighted increments (C/sketch.py:71-86) -- GPU, staged in shared
    memory; keys/amounts may be numpy arrays or CUDA tensors (`_nonneg`:
    internal, the amounts are known non-negative)."""
    T = nat.torch()
    kd, _ = _dev64(keys)
    ndim = amounts.dim() if isinstance(amounts, T.Tensor) else np.ndim(amounts)
    ad, ah = _dev64(amounts)
    if ah is not None:
        if np.any(ah < 0):
            raise ValueError("amounts must be non-negative")
        validate = 0
    else:
        validate = 0 if _nonneg else 1
    # np.add.at(table[r], idx[r], amounts) broadcasting: a scalar or one
    # amount applies to every key; any other length mismatch is an error
    k, na = int(kd.shape[0]), int(ad.shape[0])
    if ndim > 1 or na not in (1, k):
        raise ValueError("array is not broadcastable to correct shape")
    table = s.table_dev()
    a, b = s._hash_dev()
    sat = T.zeros(1, dtype=T.int32, device=nat.device())
    nat.call("cvz_sketch_add", nat.ptr(table), s.rows, s.cols, nat.ptr(a), nat.ptr(b),
             nat.ptr(kd), nat.ptr(ad), k, na, validate, nat.ptr(sat), nat.stream())
    s._table.set_dev(table)
    if nat.read_ints(sat)[0] and not s.saturated:
        s.saturated = True
        warnings.warn("sketch counter overflow, counts saturated", RuntimeWarning, stacklevel=2)


def _estimate_dev(s: CountMinSketch, keys_dev):
    T = nat.torch()
    out = T.empty(int(keys_dev.shape[0]), dtype=T.int64, device=nat.device())
    a, b = s._hash_dev()
    nat.call("cvz_sketch_estimate", nat.ptr(s.table_dev()), s.rows, s.cols, nat.ptr(a),
             nat.ptr(b), nat.ptr(keys_dev), int(keys_dev.shape[0]), nat.ptr(out), nat.stream())
    return out


def sketch_estimate(s: CountMinSketch, key: int) -> int:
    """C/sketch.py:89-90."""
    return int(sketch_estimate_many(s, np.asarray([key], dtype=np.int64))[0])


def sketch_estimate_many(s: CountMinSketch, keys) -> np.ndarray:
    """Row-wise minimum (C/sketch.py:93-98)."""
    kd, _ = _dev64(keys)
    return nat.to_host(_estimate_dev(s, kd))


def dump_tsv(s: CountMinSketch, path) -> None:
    """C/sketch.py:101-102 (np.savetxt "%d", tab): native formatting."""
    from .render import format_table, write_text
    t = np.asarray(s.table, dtype=np.int64)
    write_text(path, "", format_table(list(np.ascontiguousarray(t.T))))
