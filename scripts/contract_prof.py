"""Per-kernel device times of accumulate_sizes + contract at a config (dev tool)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2108_00529_b200 as cv  # noqa: E402
from paper_2108_00529_b200 import _native, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
torch.cuda.set_device(0)
g = cv.from_edge_array(torch.from_numpy(synth.config_graph(cfg)).cuda())
a = cv.detect_communities(g, cv.ThresholdSchedule(base=cv.degree_stats(g).mode_degree), workers=1)


def run():
    s = cv.sketch_new(4, cv.default_cols(g.edge_count), seed=0)
    cv.accumulate_sizes(s, a, g)
    return cv.contract(g, a, s)


for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    sg = run()
e1.record()
torch.cuda.synchronize()
print(f"{cfg}: sketch + contract {e0.elapsed_time(e1) / 5:.3f} ms  k={sg.node_count} se={sg.edge_count}")
with _native.profile() as prof:
    run()
for name, (c, ms) in sorted(prof.kernels.items(), key=lambda kv: -kv[1][1])[:14]:
    print(f"  {c:3d} {ms * 1000:9.1f} us  {name}")
