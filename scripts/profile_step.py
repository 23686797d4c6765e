"""Run the bench pipeline once on a BASELINE config (for ncu captures).

    ncu --set full ... python scripts/profile_step.py [--config C4] [--mode fast]

No timing is printed: numbers taken under a profiler are never bench values.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2108_00529_b200 as cv  # noqa: E402
from paper_2108_00529_b200 import synth  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="C4")
p.add_argument("--mode", default="deterministic")
p.add_argument("--steps", type=int, default=1)
a = p.parse_args()
torch.cuda.set_device(0)
dev = torch.from_numpy(synth.config_graph(a.config)).to("cuda")
for _ in range(a.steps):
    bench.pipeline(cv, dev, mode=a.mode)
torch.cuda.synchronize()
print("profile_step done")
