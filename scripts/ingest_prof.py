"""Per-kernel device times of from_edge_array at a config (dev tool)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2108_00529_b200 as cv  # noqa: E402
from paper_2108_00529_b200 import _native, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
torch.cuda.set_device(0)
dev = torch.from_numpy(synth.config_graph(cfg)).cuda()
for _ in range(3):
    cv.from_edge_array(dev)
torch.cuda.synchronize()
with _native.profile() as prof:
    for _ in range(5):
        cv.from_edge_array(dev)
for name, (c, ms) in sorted(prof.kernels.items(), key=lambda kv: -kv[1][1])[:4]:
    print(f"  {c:4d} {ms / c * 1000:9.1f} us  {name}")
