"""C5 (R-MAT scale 26, 2^30 draws) ingest + degrees + node-sharded sketch at
one rank: stage times and per-kernel device times (dev tool; also a target
for ncu captures)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2108_00529_b200 as cv  # noqa: E402
from paper_2108_00529_b200 import _native, synth  # noqa: E402
from paper_2108_00529_b200 import sharded as sh  # noqa: E402

torch.cuda.set_device(0)
scale = int(os.environ.get("CVZ_C5_SCALE", "26"))
n5, m5 = 1 << scale, 16 << scale
comm = sh.Comm()
e5 = synth.rmat_dev(scale, 0, m5, seed=0)
labels = torch.arange(n5, dtype=torch.int64, device="cuda") // 64


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        r = fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, r


ms_ing, g = timed(lambda: sh.from_edge_array_sharded(e5, comm, node_count=n5))
s = cv.sketch_new(4, cv.default_cols(g.edge_count), seed=0)
ms_sk, _ = timed(lambda: sh.accumulate_sizes_sharded(s, labels, g))
print(f"ingest+degrees {ms_ing:.2f} ms  sketch {ms_sk:.2f} ms")
with _native.profile() as prof:
    sh.from_edge_array_sharded(e5, comm, node_count=n5)
    sh.accumulate_sizes_sharded(s, labels, g)
for name, (c, ms) in sorted(prof.kernels.items(), key=lambda kv: -kv[1][1])[:10]:
    print(f"  {c:4d} {ms:9.3f} ms  {name}")
