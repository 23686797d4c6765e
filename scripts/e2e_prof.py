"""Wall-clock phases of the bench's e2e call (host arrays in, host results out)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_00529_b200 as cv  # noqa: E402
from paper_2108_00529_b200 import synth  # noqa: E402

torch.cuda.set_device(0)
e = synth.config_graph("C4")
host = torch.from_numpy(e).pin_memory()
hn = host.numpy()
for rep in range(4):
    t = [time.perf_counter()]
    g = cv.from_edge_array(hn); torch.cuda.synchronize(); t.append(time.perf_counter())
    base = cv.degree_stats(g).mode_degree; t.append(time.perf_counter())
    a = cv.detect_communities(g, cv.ThresholdSchedule(base=base), seed=0, workers=1)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    s = cv.sketch_new(4, cv.default_cols(g.edge_count), seed=0)
    cv.accumulate_sizes(s, a, g)
    sg = cv.contract(g, a, s); torch.cuda.synchronize(); t.append(time.perf_counter())
    res = cv.layout(sg, cv.LayoutParams(iterations=100, seed=0)); t.append(time.perf_counter())
    lab = a.label; t.append(time.perf_counter())
    names = ["from_edge_array", "degree_stats", "detect", "sketch+contract", "layout(+D2H pos)",
             "labels D2H"]
    print(" ".join(f"{n}={1e3 * (t[i + 1] - t[i]):.2f}" for i, n in enumerate(names)),
          f"total={1e3 * (t[-1] - t[0]):.2f} ms")
t0 = time.perf_counter()
d = host.to("cuda"); torch.cuda.synchronize()
print(f"pinned H2D of {host.numel() * 8 / 1e6:.0f} MB: {1e3 * (time.perf_counter() - t0):.2f} ms")
t0 = time.perf_counter()
d = torch.from_numpy(hn).to("cuda"); torch.cuda.synchronize()
print(f"from_numpy(pinned numpy) H2D: {1e3 * (time.perf_counter() - t0):.2f} ms")
