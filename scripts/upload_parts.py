"""Where the host-array upload goes at C4 (dev tool): the narrowing alone
(int64 -> int32 into pinned memory, host threads), the DMA alone (pinned
int32 -> device) and cvz_edges_upload (both, overlapped)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2108_00529_b200 import synth  # noqa: E402
from paper_2108_00529_b200.graph import upload_edges  # noqa: E402

torch.cuda.set_device(0)
e = synth.config_graph("C4")
h = e.astype(np.int64)
h32 = e.astype(np.int32)
pin = torch.empty(h32.shape, dtype=torch.int32).pin_memory()
pin.numpy()[:] = h32
dev = torch.empty(h32.shape, dtype=torch.int32, device="cuda")


def t(fn, k=5):
    fn()
    torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - a) / k * 1e3


print(f"edges {len(h)}  int64 bytes {h.nbytes / 1e6:.0f} MB")
print("upload int64 (narrow + DMA)   %.2f ms" % t(lambda: upload_edges(h)))
print("upload int32 pageable          %.2f ms" % t(lambda: upload_edges(h32)))
print("DMA pinned int32 only          %.2f ms" % t(lambda: dev.copy_(pin, non_blocking=True)))
out = np.empty_like(h32)
print("numpy astype int32 (1 thread)  %.2f ms" % t(lambda: np.copyto(out, h, casting="unsafe")))
print("numpy memcpy int64 (1 thread)  %.2f ms" % t(lambda: np.copyto(np.empty_like(h), h)))
