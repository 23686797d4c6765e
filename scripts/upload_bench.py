import time, numpy as np, torch, sys
sys.path.insert(0, ".")
import paper_2108_00529_b200 as cv
from paper_2108_00529_b200 import synth
from paper_2108_00529_b200.graph import upload_edges
e = synth.config_graph("C4")
for arr, nm in ((e.astype(np.int64), "int64 pageable"), (e, "int32 pageable")):
    for _ in range(2): upload_edges(arr); torch.cuda.synchronize()
    t=time.perf_counter()
    for _ in range(5): upload_edges(arr)
    torch.cuda.synchronize(); dt=(time.perf_counter()-t)/5
    print(nm, f"{dt*1e3:.2f} ms", f"{len(arr)*8/dt/1e9:.1f} GB/s on link")
