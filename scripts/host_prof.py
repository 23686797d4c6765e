"""cProfile of one warm bench step (host-side overhead between the GPU
stages; dev tool)."""
import cProfile
import os
import pstats
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2108_00529_b200 as cv  # noqa: E402
from paper_2108_00529_b200 import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
torch.cuda.set_device(0)
dev = torch.from_numpy(synth.config_graph(cfg)).to("cuda")
for _ in range(3):
    bench.pipeline(cv, dev)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
bench.pipeline(cv, dev)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
st.sort_stats("cumulative").print_stats(40)
