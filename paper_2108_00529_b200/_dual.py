"""Host/device dual storage for the drop-in dataclasses.

The reference's objects hold numpy arrays.  Ours hold a CUDA tensor produced
by the kernels and hand out a numpy copy only when the attribute is read, so
a pipeline that chains GPU stages never round-trips through the host.  Once a
host copy has been handed out it is treated as authoritative (the caller may
mutate it, as the reference tests do with counter_degree); the next GPU use
re-uploads it.
"""

from __future__ import annotations

import numpy as np

from . import _native as nat


_SIDE = None


def _side_stream():
    global _SIDE
    if _SIDE is None:
        _SIDE = nat.torch().cuda.Stream()
    return _SIDE


class Dual:
    __slots__ = ("_h", "_d", "_np_dtype", "_pend")

    def __init__(self, host=None, dev=None, np_dtype=np.int64):
        self._h = None if host is None else np.asarray(host)
        self._d = dev
        self._np_dtype = np_dtype
        self._pend = None

    def prefetch(self):
        """Start the device -> host copy now, on a side stream into a pinned
        buffer (widened to the host dtype on the device first), so a later
        read overlaps with whatever the GPU does in between instead of
        waiting for PCIe.  The device value is final once prefetched."""
        if self._h is not None or self._d is None or self._pend is not None:
            return
        T = nat.torch()
        d = self._d
        want = T.from_numpy(np.empty(0, dtype=self._np_dtype)).dtype
        if d.dtype != want:
            d = d.to(want)
        buf = T.empty(d.shape, dtype=d.dtype, pin_memory=True)
        side = _side_stream()
        side.wait_stream(T.cuda.current_stream())
        with T.cuda.stream(side):
            buf.copy_(d, non_blocking=True)
            ev = T.cuda.Event()
            ev.record(side)
        d.record_stream(side)
        self._pend = (buf, ev)

    def host(self) -> np.ndarray:
        if self._h is None:
            if self._pend is not None:
                buf, ev = self._pend
                ev.synchronize()
                self._h = buf.numpy()
                self._pend = None
            else:
                self._h = nat.to_host(self._d).astype(self._np_dtype, copy=False)
        return self._h

    def set_host(self, a):
        self._h = np.asarray(a)
        self._d = None
        self._pend = None

    def dev(self, torch_dtype):
        """CUDA tensor view of the current value in `torch_dtype`."""
        if self._h is not None:
            return nat.to_dev(self._h, torch_dtype)
        if self._d.dtype != torch_dtype:
            return self._d.to(torch_dtype)
        return self._d

    def set_dev(self, t):
        self._d = t
        self._h = None
        self._pend = None

    @property
    def on_device(self) -> bool:
        return self._h is None and self._d is not None

    def __len__(self):
        return len(self._h) if self._h is not None else int(self._d.shape[0])
