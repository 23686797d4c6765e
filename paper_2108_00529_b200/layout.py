"""ForceAtlas2 + Barnes-Hut layout (drop-in for C/layout.py) on the GPU.

`layout` runs every iteration on the device (cvz_layout_run: tree build,
repulsion, CSR attraction, gravity, adaptive speed, clamped update) as one
CUDA graph replayed `iterations` times; positions come back once.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import functools

import numpy as np

from . import _native as nat
from ._native import LayoutError

MAX_DEPTH = 40
COINCIDE_EPS = 1e-4
_SPEED_FORMS = ("product", "sum")
_ATTRACTION_FORMS = ("canonical", "reversed")


@dataclass(frozen=True)
class LayoutParams:
    """C/layout.py:40-68."""

    iterations: int = 100
    gravity: float = 1.0
    repulsion: float = 80.0
    jitter_tolerance: float = 1.0
    theta: float = 0.5
    max_step: float = 10.0
    speed_form: str = "product"
    attraction_form: str = "canonical"
    seed: int = 0

    def __post_init__(self):
        if self.iterations < 1:
            raise ValueError("iterations must be positive")
        if self.gravity < 0:
            raise ValueError("gravity must be non-negative")
        if self.repulsion <= 0:
            raise ValueError("repulsion strength must be positive")
        if self.jitter_tolerance <= 0:
            raise ValueError("jitter tolerance must be positive")
        if self.theta < 0:
            raise ValueError("theta must be non-negative")
        if self.max_step <= 0:
            raise ValueError("max step must be positive")
        if self.speed_form not in _SPEED_FORMS:
            raise ValueError(f"unknown speed form {self.speed_form!r}")
        if self.attraction_form not in _ATTRACTION_FORMS:
            raise ValueError(f"unknown attraction form {self.attraction_form!r}")


@dataclass
class LayoutResult:
    """C/layout.py:71-75."""

    positions: np.ndarray
    displacement: np.ndarray
    iterations: int


def init_positions(n: int, seed: int = 0) -> np.ndarray:
    """Uniform square of side sqrt(n) (C/layout.py:78-82); host numpy RNG so
    the start state is the reference's."""
    side = max(np.sqrt(n), 1.0)
    return np.random.default_rng(seed).uniform(-side / 2, side / 2, size=(n, 2))


@functools.lru_cache(maxsize=64)
def _pcg64_state(seed: int):
    """numpy's PCG64 state for default_rng(seed) (SeedSequence hashing costs
    ~0.1 ms of host time per call, while the GPU would sit idle)."""
    st = np.random.default_rng(seed).bit_generator.state["state"]
    return int(st["state"]), int(st["inc"])


def _init_positions_dev(n: int, seed: int = 0):
    """init_positions drawn on the GPU (cvz_pcg64_uniform): numpy's PCG64
    stream seeded by numpy on the host, bit-identical values, no host loop
    or (n, 2) upload."""
    T = nat.torch()
    side = max(np.sqrt(n), 1.0)
    low, high = -side / 2, side / 2
    if isinstance(seed, (int, np.integer)):
        s, inc = _pcg64_state(int(seed))
    else:  # None / SeedSequence / Generator-like seeds: never cached
        st = np.random.default_rng(seed).bit_generator.state["state"]
        s, inc = int(st["state"]), int(st["inc"])
    m64 = (1 << 64) - 1
    out = T.empty((n, 2), dtype=T.float64, device=nat.device())
    nat.call("cvz_pcg64_uniform", s >> 64, s & m64, inc >> 64, inc & m64, low, high - low,
             2 * n, nat.ptr(out), nat.stream())
    return out


def _f64(x):
    T = nat.torch()
    if isinstance(x, T.Tensor):
        return x.to(device=nat.device(), dtype=T.float64).contiguous()
    return nat.to_dev(np.ascontiguousarray(np.asarray(x, dtype=np.float64)), T.float64)


def repulsion_forces(pos, mass, repulsion: float = 80.0, theta: float = 0.5) -> np.ndarray:
    """C/layout.py:312-328: exact tiles for theta <= 0, else GPU Barnes-Hut."""
    T = nat.torch()
    p = _f64(pos).reshape(-1, 2)
    m = _f64(mass).reshape(-1)
    out = T.empty_like(p)
    nat.call("cvz_repulsion", nat.ptr(p), nat.ptr(m), int(p.shape[0]), float(repulsion),
             float(theta), nat.ptr(out), nat.stream())
    return nat.to_host(out)


def gravity_forces(pos, mass, gravity: float) -> np.ndarray:
    """Linear pull toward the origin, F = -g * m * pos (C/layout.py:307-309)."""
    p = _f64(pos).reshape(-1, 2)
    m = _f64(mass).reshape(-1, 1)
    return nat.to_host((-gravity * m) * p)


def _attraction(pos, edges, weight, sign, out) -> None:
    """C/layout.py:293-304: accumulate springs into numpy `out` in place."""
    T = nat.torch()
    p = _f64(pos).reshape(-1, 2)
    e = nat.to_dev(np.asarray(edges, dtype=np.int64).reshape(-1, 2), T.int32)
    w = _f64(weight).reshape(-1)
    o = _f64(out).reshape(-1, 2)
    nat.call("cvz_attraction", nat.ptr(p), int(p.shape[0]), nat.ptr(e), int(e.shape[0]),
             nat.ptr(w), float(sign), nat.ptr(o), nat.stream())
    out[...] = nat.to_host(o).reshape(out.shape)


def _masses_and_edges(obj):
    """C/layout.py:331-338 (host view; the GPU path uses _device_model)."""
    if hasattr(obj, "weight"):
        mass = np.maximum(obj.weight, 1).astype(np.float64)
        edge_weight = obj.multiplicity.astype(np.float64)
    else:
        mass = (obj.degree + 1).astype(np.float64)
        edge_weight = np.ones(len(obj.edges), dtype=np.float64)
    return mass, obj.edges.astype(np.int64), edge_weight


def _device_model(obj):
    """mass (f64), edges (int32), edge weight (f64 or None) as CUDA tensors."""
    T = nat.torch()
    # our SuperGraph first: hasattr(obj, "weight") would evaluate the host
    # property (a device -> host copy of the weights, then a re-upload)
    if hasattr(obj, "weight_dev") or hasattr(obj, "weight"):
        if hasattr(obj, "weight_dev"):
            w = obj.weight_dev()
            mass = T.clamp(w, min=1).to(T.float64)
            ew = obj.multiplicity_dev().to(T.float64)
            e = obj.edges_dev()
        else:
            mass = nat.to_dev(np.maximum(obj.weight, 1), T.float64)
            ew = nat.to_dev(obj.multiplicity, T.float64)
            e = nat.to_dev(np.asarray(obj.edges, dtype=np.int64).reshape(-1, 2), T.int32)
        return mass, e, ew
    mass = (obj.degree_dev() + 1).to(T.float64)
    return mass, obj.edges_dev(), None


def layout(obj, params: LayoutParams | None = None, positions=None) -> LayoutResult:
    """Iterate the force model on a SuperGraph or Graph (C/layout.py:341-402)."""
    if params is None:
        params = LayoutParams()
    T = nat.torch()
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
    pos_d = _init_positions_dev(n, params.seed) if positions is None else nat.to_dev(pos, T.float64)
    prev = T.zeros_like(pos_d)
    speed = T.ones(1, dtype=T.float64, device=nat.device())
    hist = T.zeros(params.iterations, dtype=T.float64, device=nat.device())
    P = nat._LayoutParams(params.iterations, params.gravity, params.repulsion,
                          params.jitter_tolerance, params.theta, params.max_step,
                          _SPEED_FORMS.index(params.speed_form),
                          _ATTRACTION_FORMS.index(params.attraction_form))
    bad = ctypes.c_int64(0)
    nat.call("cvz_layout_run", nat.ptr(pos_d), nat.ptr(mass), n, nat.ptr(e), int(e.shape[0]),
             nat.ptr(ew), ctypes.byref(P), nat.ptr(prev), nat.ptr(speed), nat.ptr(hist),
             ctypes.byref(bad), nat.stream())
    return LayoutResult(positions=nat.to_host(pos_d), displacement=nat.to_host(hist),
                        iterations=params.iterations)


def layout_step(obj, pos, prev_force, speed, params: LayoutParams | None = None):
    """One teacher-forced iteration with explicit state (used by the parity
    tests): returns (positions, force, speed, max displacement)."""
    if params is None:
        params = LayoutParams(iterations=1)
    T = nat.torch()
    n = obj.node_count
    mass, e, ew = _device_model(obj)
    pos_d = nat.to_dev(np.asarray(pos, dtype=np.float64), T.float64)
    prev = nat.to_dev(np.asarray(prev_force, dtype=np.float64), T.float64)
    sp = T.full((1,), float(speed), dtype=T.float64, device=nat.device())
    hist = T.zeros(1, dtype=T.float64, device=nat.device())
    P = nat._LayoutParams(1, params.gravity, params.repulsion, params.jitter_tolerance,
                          params.theta, params.max_step, _SPEED_FORMS.index(params.speed_form),
                          _ATTRACTION_FORMS.index(params.attraction_form))
    bad = ctypes.c_int64(0)
    nat.call("cvz_layout_run", nat.ptr(pos_d), nat.ptr(mass), n, nat.ptr(e), int(e.shape[0]),
             nat.ptr(ew), ctypes.byref(P), nat.ptr(prev), nat.ptr(sp), nat.ptr(hist),
             ctypes.byref(bad), nat.stream())
    return nat.to_host(pos_d), nat.to_host(prev), float(sp.item()), float(hist.item())
