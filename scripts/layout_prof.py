"""Per-kernel device times of one supergraph layout at a config (dev tool)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2108_00529_b200 as cv  # noqa: E402
from paper_2108_00529_b200 import _native, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C1"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 100
full = len(sys.argv) > 3 and sys.argv[3] == "full"
torch.cuda.set_device(0)
g = cv.from_edge_array(torch.from_numpy(synth.config_graph(cfg)).cuda())
a = cv.detect_communities(g, cv.ThresholdSchedule(base=cv.degree_stats(g).mode_degree), workers=1)
s = cv.sketch_new(4, cv.default_cols(g.edge_count), seed=0)
cv.accumulate_sizes(s, a, g)
sg = g if full else cv.contract(g, a, s)
print(f"{cfg}: bodies {sg.node_count} edges {sg.edge_count}")
for _ in range(2):
    cv.layout(sg, cv.LayoutParams(iterations=iters))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
cv.layout(sg, cv.LayoutParams(iterations=iters))
e1.record()
torch.cuda.synchronize()
print(f"layout {iters} it: {e0.elapsed_time(e1):.3f} ms ({e0.elapsed_time(e1) / iters * 1e3:.1f} us/it)")
with _native.profile() as prof:
    cv.layout(sg, cv.LayoutParams(iterations=iters))
tot = sum(v[1] for v in prof.kernels.values())
print(f"  profiled (no graph) total {tot:.3f} ms")
for name, (c, ms) in sorted(prof.kernels.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"  {c:5d} {ms:8.3f} ms {ms / c * 1e3:8.2f} us/launch  {name}")
