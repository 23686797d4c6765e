"""A/B timing of the supergraph layout on a BASELINE config (dev tool).

    python scripts/ab_layout.py [--config C4] [--iters 100]
Set kernel-selection env vars (CVZ_BH_THREAD, CVZ_BH_MINB, ...) per process."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import hashlib  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_00529_b200 as cv  # noqa: E402
from paper_2108_00529_b200 import synth  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="C4")
p.add_argument("--iters", type=int, default=100)
p.add_argument("--full", action="store_true", help="lay out the full graph instead")
a = p.parse_args()
torch.cuda.set_device(0)
g = cv.from_edge_array(torch.from_numpy(synth.config_graph(a.config)).cuda())
lab = cv.detect_communities(g, cv.ThresholdSchedule(base=cv.degree_stats(g).mode_degree), workers=1)
s = cv.sketch_new(4, cv.default_cols(g.edge_count), 0)
cv.accumulate_sizes(s, lab, g)
sg = cv.contract(g, lab, s)
obj = g if a.full else sg
P = cv.LayoutParams(iterations=a.iters)
for _ in range(2):
    r = cv.layout(obj, P)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(3):
    e0.record()
    r = cv.layout(obj, P)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / a.iters)
env = {k: v for k, v in os.environ.items() if k.startswith("CVZ_")}
print(f"{a.config} {'full' if a.full else 'super'} n={obj.node_count} m={obj.edge_count} "
      f"env={env} ms/iter={min(ts):.4f} disp[-1]={r.displacement[-1]:.6g} "
      f"pos0={r.positions[0].tolist()} "
      f"hash={hashlib.sha1(np.ascontiguousarray(r.positions).tobytes()).hexdigest()[:12]}")
with cv._native.profile() as prof:
    cv.layout(obj, cv.LayoutParams(iterations=10))
for name, (c, ms) in sorted(prof.kernels.items(), key=lambda kv: -kv[1][1])[:int(os.environ.get("AB_TOP", "40"))]:
    print(f"   {ms / c * 1000:8.1f} us/launch  {name}")
