"""Per-stage / per-kernel device times of the bench pipeline (CUDA events
via cvz_profile_*) -- a development tool, not the bench contract.

    python scripts/bench_stages.py [--config C4] [--mode deterministic] [--reps 3]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2108_00529_b200 as cv  # noqa: E402
from paper_2108_00529_b200 import _native, synth  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="C4")
p.add_argument("--mode", default="deterministic")
p.add_argument("--reps", type=int, default=3)
p.add_argument("--top", type=int, default=25)
a = p.parse_args()
torch.cuda.set_device(0)
dev = torch.from_numpy(synth.config_graph(a.config)).to("cuda")
for _ in range(2):
    bench.pipeline(cv, dev, mode=a.mode)
stats = []
for _ in range(a.reps):
    bench.pipeline(cv, dev, stats, mode=a.mode)
for st in stats:
    print({k: (round(v, 3) if isinstance(v, float) else v) for k, v in st.items() if k != "m_r"})
with _native.profile() as prof:
    bench.pipeline(cv, dev, mode=a.mode)
tot = sum(v[1] for v in prof.kernels.values())
print(f"profiled kernels total {tot:.3f} ms (non-graph launches)")
for name, (c, ms) in sorted(prof.kernels.items(), key=lambda kv: -kv[1][1])[:a.top]:
    print(f"  {c:5d} {ms:9.3f} ms {ms / c * 1000:9.1f} us/launch  {name}")
