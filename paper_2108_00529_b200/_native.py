"""ctypes binding of libcvz_b200.so (include/cvz_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
present, every compute call raises.  Device buffers are torch CUDA tensors
(torch is plumbing here: allocation + streams); only raw pointers cross the
C-ABI.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libcvz_b200.so")

CVZ_OK, CVZ_ERR_CUDA, CVZ_ERR_VALUE, CVZ_ERR_LAYOUT, CVZ_ERR_OOM, CVZ_ERR_RANGE = 0, -1, -2, -3, -4, -5
DETERMINISTIC, FAST = 0, 1


class LayoutError(RuntimeError):
    """Non-finite layout positions (C/layout.py:36-37)."""


class _ContractResult(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int64), ("se", ctypes.c_int64),
                ("comm_id", ctypes.c_void_p), ("weight", ctypes.c_void_p),
                ("se_edges", ctypes.c_void_p), ("mult", ctypes.c_void_p)]


class _LayoutParams(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int64), ("gravity", ctypes.c_double),
                ("repulsion", ctypes.c_double), ("jitter_tolerance", ctypes.c_double),
                ("theta", ctypes.c_double), ("max_step", ctypes.c_double),
                ("speed_form", ctypes.c_int), ("attraction_form", ctypes.c_int)]


_P, _I64, _I32, _D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double

# symbol -> argtypes (restype int unless noted); mirrors include/cvz_b200.h
SIGNATURES = {
    "cvz_version": [],
    "cvz_last_error": [],
    "cvz_launch_count": [],
    "cvz_read_small": [_P, _P, _I64, _P],
    "cvz_profile_begin": [],
    "cvz_profile_end": [],
    "cvz_profile_report": [],
    "cvz_bh_stats": [_I32, _P],
    "cvz_probe_fp64": [ctypes.POINTER(_D), _P],
    "cvz_edges_upload": [_P, _I32, _I64, _P, _P],
    "cvz_edges_compact": [_P, _I32, _I64, _P, _P, _P, _I32, _P],
    "cvz_degree_count": [_P, _I64, _I64, _P, _P],
    "cvz_degree_stats": [_P, _I64, _P, _P],
    "cvz_scoda_pass": [_P, _I64, _P, _I64, _I64, _I32, _I32, _P, _P, _P, _P],
    "cvz_resolve_labels": [_P, _I64, _P, _P],
    "cvz_detect_round": [_P, _I64, _P, _P, _I64, _I64, _I64, _I32, _I32, _I32, _I32,
                         _P, _P, _P, _P, _P, ctypes.POINTER(_I64),
                         ctypes.POINTER(ctypes.c_int), _I64, ctypes.POINTER(_I64), _P],
    "cvz_sketch_indices": [_P, _P, _I32, _I64, _P, _I64, _P, _P],
    "cvz_sketch_add": [_P, _I32, _I64, _P, _P, _P, _P, _I64, _I64, _I32, _P, _P],
    "cvz_sketch_estimate": [_P, _I32, _I64, _P, _P, _P, _I64, _P, _P],
    "cvz_contract": [_P, _I64, _P, _I64, _P, _I32, _I64, _P, _P,
                     ctypes.POINTER(_ContractResult), _P],
    "cvz_contract_release": [ctypes.POINTER(_ContractResult), _P],
    "cvz_repulsion": [_P, _P, _I64, _D, _D, _P, _P],
    "cvz_attraction": [_P, _I64, _P, _I64, _P, _D, _P, _P],
    "cvz_layout_run": [_P, _P, _I64, _P, _I64, _P, ctypes.POINTER(_LayoutParams),
                       _P, _P, _P, ctypes.POINTER(_I64), _P],
    "cvz_pcg64_uniform": [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                          _D, _D, _I64, _P, _P],
    "cvz_modularity_parts": [_P, _I64, _P, _P, _I64, _I64, _P, _P, _P],
    "cvz_sketch_accumulate": [_P, _I32, _I64, _P, _P, _P, _P, _I64, _P],
    "cvz_sketch_accumulate_edges": [_P, _I32, _I64, _P, _P, _P, _I64, _P, _P],
    "cvz_sketch_merge": [_P, _P, _I32, _I64, _P, _P],
    "cvz_fa2_shard_create": [_P, _P, _I64, _P, _I64, _P, ctypes.POINTER(_LayoutParams),
                             _I64, _I64, _I32, ctypes.POINTER(ctypes.c_void_p), _P],
    "cvz_fa2_shard_forces": [_P, _P, _P, _P],
    "cvz_fa2_shard_update": [_P, _P, _P, _P, _P],
    "cvz_fa2_shard_absorb": [_P, _P, _P, _P],
    "cvz_fa2_shard_finish": [_P, ctypes.POINTER(_D), ctypes.POINTER(_I64),
                             ctypes.POINTER(ctypes.c_int), _P],
    "cvz_fa2_shard_destroy": [_P, _P],
    "cvz_parse_begin": [ctypes.c_char_p, _I64, _I32, ctypes.POINTER(ctypes.c_void_p),
                        ctypes.POINTER(_I64), ctypes.POINTER(_I64), ctypes.POINTER(ctypes.c_int),
                        ctypes.POINTER(ctypes.c_int)],
    "cvz_parse_take": [_P, _P],
    "cvz_first_seen_remap": [_P, _I64, _P, ctypes.POINTER(_I64), _P],
    "cvz_dense_labels": [_P, _I64, _P, ctypes.POINTER(_I64), _P],
    "cvz_community_sizes": [_P, _I64, _I64, _P, _P, _P],
    "cvz_modularity": [_P, _I64, _P, _P, _I64, _I64, _P, _P],
    "cvz_format_table": [_I64, _I32, _P, _P, ctypes.c_char, ctypes.POINTER(ctypes.c_void_p),
                         ctypes.POINTER(_I64)],
    "cvz_format_svg": [_I64, _P, _P, _P, _P, _I32, _I64, _P, _P, _D,
                       ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(_I64)],
    "cvz_text_take": [_P, _P],
    "cvz_rmat_edges": [_I32, _D, _D, _D, ctypes.c_uint64, _I64, _I64, _P, _P],
    "cvz_make_schedule": [_I64, _I32, _I32, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                          ctypes.c_uint64, _I32, ctypes.c_uint32, _P],
}

_lib = None


def load():
    """Load the library (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: run `python -m paper_2108_00529_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        lib.cvz_last_error.restype = ctypes.c_char_p
        lib.cvz_launch_count.restype = ctypes.c_longlong
        lib.cvz_profile_report.restype = ctypes.c_char_p
        _lib = lib
    return _lib


def launch_count() -> int:
    return int(load().cvz_launch_count())


def bh_stats(fn):
    """Run fn() with the instrumented BH walk; returns (result, visits,
    interactions) summed over every walk launched inside (cvz_bh_stats)."""
    check(load().cvz_bh_stats(1, None), "cvz_bh_stats")
    tot = (ctypes.c_ulonglong * 2)()
    try:
        out = fn()
    finally:
        check(load().cvz_bh_stats(0, ctypes.cast(tot, ctypes.c_void_p)), "cvz_bh_stats")
    return out, int(tot[0]), int(tot[1])


class profile:
    """Context manager: per-kernel device times of every library launch in
    the block (cvz_profile_begin/end).  .kernels = {name: (launches, ms)}."""

    def __enter__(self):
        call("cvz_profile_begin")
        self.kernels = {}
        return self

    def __exit__(self, *exc):
        call("cvz_profile_end")
        for line in load().cvz_profile_report().decode().splitlines():
            name, cnt, ms = line.split("\t")
            self.kernels[name] = (int(cnt), float(ms))
        return False


def check(rc: int, what: str = ""):
    if rc == CVZ_OK:
        return
    msg = load().cvz_last_error().decode(errors="replace")
    if rc in (CVZ_ERR_VALUE, CVZ_ERR_RANGE):
        raise ValueError(msg)
    if rc == CVZ_ERR_LAYOUT:
        raise LayoutError(msg)
    if rc == CVZ_ERR_OOM:
        raise MemoryError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: CUDA error: {msg}")


def call(name: str, *args):
    check(getattr(load(), name)(*args), name)


# ---------------------------------------------------------------- torch glue
_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        if not t.cuda.is_available():
            raise RuntimeError("paper_2108_00529_b200 needs a CUDA device (B200); "
                               "there is no CPU fallback")
        _torch = t
    return _torch


def stream():
    return ctypes.c_void_p(torch().cuda.current_stream().cuda_stream)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def device():
    return torch().device("cuda", torch().cuda.current_device())


def to_dev(a, dtype):
    """numpy / list / torch -> contiguous CUDA tensor of `dtype` (torch dtype)."""
    T = torch()
    if isinstance(a, T.Tensor):
        t = a.to(device=device(), dtype=dtype)
    else:
        import numpy as np
        arr = np.ascontiguousarray(np.asarray(a))
        t = T.from_numpy(arr).to(device=device(), dtype=dtype, non_blocking=False)
    return t.contiguous()


def read_ints(t):
    """Small int64 CUDA tensor (<= 32 values) -> list of Python ints after
    the current stream's work, without the copy engines (cvz_read_small):
    a control read does not wait behind a bulk prefetch on another stream."""
    import numpy as np
    t = t.detach()
    T = torch()
    if not t.is_cuda:
        return [int(v) for v in t.tolist()]
    t = t.to(T.int64).contiguous()
    out = np.empty(int(t.numel()), dtype=np.int64)
    call("cvz_read_small", out.ctypes.data, ptr(t), out.nbytes, stream())
    return [int(v) for v in out]


def to_host(t):
    """Device -> numpy through a pinned (page-locked, allocator-cached) host
    buffer: DMA at full link speed and no first-touch page faults, so result
    read-back time is steady (a pageable .cpu() of a 24 MB label array
    measured 1.5-14 ms)."""
    t = t.detach()
    if not t.is_cuda:
        return t.numpy()
    out = torch().empty(t.shape, dtype=t.dtype, pin_memory=True)
    out.copy_(t)
    return out.numpy()
