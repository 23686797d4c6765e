"""Per-kernel device times of node-sharded full-graph FA2 iterations on the
R-MAT graph of BASELINE C5 at one rank (dev tool)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2108_00529_b200 as cv  # noqa: E402
from paper_2108_00529_b200 import _native, synth  # noqa: E402
from paper_2108_00529_b200 import sharded as sh  # noqa: E402
from paper_2108_00529_b200.layout import _init_positions_dev  # noqa: E402

torch.cuda.set_device(0)
scale = int(os.environ.get("CVZ_C5_SCALE", "26"))
comm = sh.Comm()
e5 = synth.rmat_dev(scale, 0, 16 << scale, seed=0)
g = sh.from_edge_array_sharded(e5, comm, node_count=1 << scale).gather()
del e5
n = g.node_count
mass = (g.degree_dev() + 1).to(torch.float64)
P = sh._layout_params(cv.LayoutParams(iterations=4))
lay = sh.ShardLayout(comm, n, mass, g.edges_dev(), None, P, _init_positions_dev(n, 0), 4)
lay.run(1)
torch.cuda.synchronize()
with _native.profile() as prof:
    lay.run(2)
lay.close()
tot = sum(v[1] for v in prof.kernels.values())
print(f"2 iterations, profiled {tot:.1f} ms")
for name, (c, ms) in sorted(prof.kernels.items(), key=lambda kv: -kv[1][1])[:16]:
    print(f"  {c:4d} {ms:9.3f} ms  {name}")
