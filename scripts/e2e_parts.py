"""Where the end-to-end time goes at C4: host-array upload (narrowing +
DMA), the device-resident pipeline and the e2e pipeline (dev tool).
Run from the repo root."""
import time, sys, gc
import numpy as np, torch
sys.path.insert(0, ".")
import bench
import paper_2108_00529_b200 as cv
from paper_2108_00529_b200 import synth
from paper_2108_00529_b200.graph import upload_edges
torch.cuda.set_device(0)
e = synth.config_graph("C4")
h = e.astype(np.int64)
dev = torch.from_numpy(e).cuda()
for _ in range(3): bench.pipeline_e2e(cv, h); bench.pipeline(cv, dev)
torch.cuda.synchronize()
def t(fn, k=5):
    gc.disable(); torch.cuda.synchronize(); a=time.perf_counter()
    for _ in range(k): r = fn()
    torch.cuda.synchronize(); gc.enable(); return (time.perf_counter()-a)/k*1e3
print("upload int64", t(lambda: upload_edges(h)))
print("pipeline device", t(lambda: bench.pipeline(cv, dev)))
print("pipeline e2e", t(lambda: bench.pipeline_e2e(cv, h)))
def dev_then_read():
    res = bench.pipeline(cv, dev)
    return res.positions
print("pipeline device + pos read", t(dev_then_read))
