"""Supergraph contraction (drop-in for C/supergraph.py) on the GPU."""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from ._dual import Dual
from .sketch import CountMinSketch, sketch_add_many


class SuperGraph:
    """Weighted contraction: one node per community (C/supergraph.py:19-39)."""

    __slots__ = ("node_count", "_edges", "_weight", "_mult", "_comm")

    def __init__(self, node_count, edges, weight, multiplicity, community_id):
        edges = np.asarray(edges)
        if edges.ndim != 2 or edges.shape[1] != 2:
            raise ValueError("superedges must be an (s, 2) array")
        if len(weight) != node_count:
            raise ValueError("one weight per supernode required")
        if len(multiplicity) != len(edges):
            raise ValueError("one multiplicity per superedge required")
        self.node_count = int(node_count)
        self._edges = Dual(host=edges)
        self._weight = Dual(host=np.asarray(weight))
        self._mult = Dual(host=np.asarray(multiplicity))
        self._comm = Dual(host=np.asarray(community_id))

    @classmethod
    def _from_device(cls, k, edges, weight, mult, comm):
        sg = object.__new__(cls)
        sg.node_count = int(k)
        sg._edges, sg._weight = Dual(dev=edges), Dual(dev=weight)
        sg._mult, sg._comm = Dual(dev=mult), Dual(dev=comm)
        return sg

    edges = property(lambda self: self._edges.host())
    weight = property(lambda self: self._weight.host())
    multiplicity = property(lambda self: self._mult.host())
    community_id = property(lambda self: self._comm.host())

    @property
    def edge_count(self) -> int:
        return len(self._edges)

    def edges_dev(self):
        e = self._edges.dev(nat.torch().int64)
        return e.reshape(-1, 2).to(nat.torch().int32).contiguous()

    def weight_dev(self):
        return self._weight.dev(nat.torch().int64)

    def multiplicity_dev(self):
        return self._mult.dev(nat.torch().int64)

    def __repr__(self):
        return f"SuperGraph(node_count={self.node_count}, edge_count={self.edge_count})"


def _labels_dev(labels):
    T = nat.torch()
    if hasattr(labels, "label_dev"):
        return labels.label_dev()
    if isinstance(labels, T.Tensor):
        return labels.to(device=nat.device(), dtype=T.int64).contiguous()
    return nat.to_dev(np.asarray(labels, dtype=np.int64), T.int64)


def accumulate_sizes(sketch: CountMinSketch, labels, degrees) -> None:
    """Add each node's degree to its community's counter (C/supergraph.py:42-46)."""
    T = nat.torch()
    # degrees our kernels computed (a Graph whose degrees never left the
    # device) are non-negative by construction: no validation pass + sync
    trusted = getattr(getattr(degrees, "_degree", None), "on_device", False)
    if hasattr(degrees, "degree_dev"):
        degrees = degrees.degree_dev()
    sketch_add_many(sketch, _labels_dev(labels), degrees if isinstance(degrees, T.Tensor)
                    else np.asarray(degrees, dtype=np.int64), _nonneg=trusted)


def contract(g, labels, sketch: CountMinSketch) -> SuperGraph:
    """Collapse g under `labels` (C/supergraph.py:49-76): dense ids, sketch
    weights, sorted + run-length-encoded superedges, all on the GPU."""
    T = nat.torch()
    lab = _labels_dev(labels)
    if int(lab.shape[0]) != g.node_count:
        raise ValueError("one label per node required")
    a, b = sketch._hash_dev()
    res = nat._ContractResult()
    e = g.edges_dev()
    nat.call("cvz_contract", nat.ptr(e), int(e.shape[0]), nat.ptr(lab), g.node_count,
             nat.ptr(sketch.table_dev()), sketch.rows, sketch.cols, nat.ptr(a), nat.ptr(b),
             ctypes.byref(res), nat.stream())
    k, se = int(res.k), int(res.se)
    owner = _ContractBuffers(res)
    comm = owner.tensor(res.comm_id, (k,))
    weight = owner.tensor(res.weight, (k,))
    edges = owner.tensor(res.se_edges, (se, 2))
    mult = owner.tensor(res.mult, (se,))
    return SuperGraph._from_device(k, edges, weight, mult, comm)


class _ContractBuffers:
    """Owner of the four result buffers cvz_contract allocated.  The returned
    tensors VIEW them (no device-to-device copies); each view keeps this
    owner alive, and the last one to go releases all four (stream-ordered
    cudaFreeAsync, cvz_contract_release)."""

    def __init__(self, res):
        self.res = res
        self.stream = nat.stream()  # released (stream-ordered) where it was made

    def tensor(self, ptr, shape):
        T = nat.torch()
        if not ptr or 0 in shape:
            return T.empty(shape, dtype=T.int64, device=nat.device())
        return T.as_tensor(_View(self, ptr, shape), device=nat.device())

    def __del__(self):
        try:
            nat.call("cvz_contract_release", ctypes.byref(self.res), self.stream)
        except Exception:  # interpreter shutdown: the CUDA context is gone anyway
            pass


class _View:
    """__cuda_array_interface__ of one int64 result buffer (torch.as_tensor
    holds a reference to this object for the tensor's lifetime)."""

    def __init__(self, owner, ptr, shape):
        self.owner = owner
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<i8",
                                         "data": (int(ptr), False), "version": 3,
                                         "stream": None}


def export_supernodes_tsv(sg: SuperGraph, path) -> None:
    """C/supergraph.py:79-83 (native multi-threaded formatting)."""
    from .render import format_table, write_text
    write_text(path, "supernode\tcommunity\tweight\n",
               format_table([None, sg.community_id, sg.weight]) if sg.node_count else b"")


def export_superedges_tsv(sg: SuperGraph, path) -> None:
    """C/supergraph.py:86-91 (native multi-threaded formatting)."""
    from .render import format_table, write_text
    e = sg.edges
    write_text(path, "source\ttarget\tmultiplicity\n",
               format_table([e[:, 0], e[:, 1], sg.multiplicity]) if sg.edge_count else b"")
