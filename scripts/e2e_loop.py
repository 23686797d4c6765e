import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import bench
import paper_2108_00529_b200 as cv
from paper_2108_00529_b200 import synth
torch.cuda.set_device(0)
e = synth.config_graph("C4")
host = torch.from_numpy(e).pin_memory()
hn = host.numpy()
dev = host.to("cuda")
for _ in range(3): bench.pipeline(cv, dev)
torch.cuda.synchronize()
for _ in range(2): bench.pipeline_e2e(cv, hn)
torch.cuda.synchronize()
for rep in range(5):
    t0 = time.perf_counter()
    pos, lab = bench.pipeline_e2e(cv, hn)
    torch.cuda.synchronize()
    print(f"e2e {1e3*(time.perf_counter()-t0):.2f} ms")
t0=torch.cuda.Event(enable_timing=True); t1=torch.cuda.Event(enable_timing=True)
t0.record()
for _ in range(3): bench.pipeline(cv, dev)
t1.record(); torch.cuda.synchronize(); print("device step", t0.elapsed_time(t1)/3)
