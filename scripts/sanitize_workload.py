"""Small workload touching every kernel family, for compute-sanitizer runs
(memcheck / racecheck / synccheck; scripts/sanitize.sh).  C1/C2-sized
inputs: ingest, degree stats, deterministic + fast community passes (also
workers > 1), sketch (staged + direct paths), contract, modularity, size
histogram, layout (BH + exact + coincident-jitter rerun + full graph), the
node-sharded layout with an owned-row subset, the text loader and writers."""
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_00529_b200 as cv  # noqa: E402
from paper_2108_00529_b200 import sharded as sh  # noqa: E402
from paper_2108_00529_b200 import synth  # noqa: E402

torch.cuda.set_device(0)
which = sys.argv[1] if len(sys.argv) > 1 else "C1"
e = synth.config_graph(which)
g = cv.from_edge_array(e)
st = cv.degree_stats(g)
for mode in ("deterministic", "fast"):
    a = cv.detect_communities(g, cv.ThresholdSchedule(base=st.mode_degree), workers=1, mode=mode)
a4 = cv.detect_communities(g, cv.ThresholdSchedule(base=st.mode_degree), workers=4)
ar = cv.detect_communities(g, cv.ThresholdSchedule(base=st.mode_degree), workers=1,
                           round_stream="restream")
s = cv.sketch_new(4, cv.default_cols(g.edge_count), seed=0)
cv.accumulate_sizes(s, a, g)
big = cv.sketch_new(4, 200_000, seed=1)          # direct (global-atomic) path
cv.sketch_add_many(big, np.arange(300_000) % 5000, np.ones(300_000, np.int64))
stg = cv.sketch_new(4, 6500, seed=2)             # staged (shared-memory) path
cv.sketch_add_many(stg, np.arange(3_000_000) % 77777, np.full(3_000_000, 3, np.int64))
cv.sketch_estimate_many(s, a.label[:1000])
sg = cv.contract(g, a, s)
q = cv.modularity(g, a.label)
hist = cv.community_size_histogram(a.label)
r1 = cv.layout(sg, cv.LayoutParams(iterations=5))
r2 = cv.layout(sg, cv.LayoutParams(iterations=3, theta=0.0))
p0 = np.repeat(np.random.default_rng(1).uniform(-3, 3, (sg.node_count // 4 + 1, 2)), 4,
               axis=0)[:sg.node_count]
r3 = cv.layout(sg, cv.LayoutParams(iterations=3), positions=p0)   # jitter rerun
r4 = cv.layout(g, cv.LayoutParams(iterations=2))
# node-sharded layout, world of 1 but an owned-row subset (select path)
from paper_2108_00529_b200.layout import _device_model, _init_positions_dev  # noqa: E402
mass, ed, ew = _device_model(g)
P = sh._layout_params(cv.LayoutParams(iterations=2))
lay = sh.ShardLayout(sh.Comm(), g.node_count, mass, ed, ew, P,
                     _init_positions_dev(g.node_count, 0), 2)
lay.run(2)
lay.close()
import ctypes  # noqa: E402

from paper_2108_00529_b200 import _native as nat  # noqa: E402
pos0 = _init_positions_dev(g.node_count, 0)
h = ctypes.c_void_p()
n = g.node_count
nat.call("cvz_fa2_shard_create", nat.ptr(pos0), nat.ptr(mass), n, nat.ptr(ed), int(ed.shape[0]),
         None, ctypes.byref(P), n // 3, 2 * n // 3, 0, ctypes.byref(h), nat.stream())
sums = torch.zeros(2, dtype=torch.float64, device="cuda")
nat.call("cvz_fa2_shard_forces", h, nat.ptr(pos0), nat.ptr(sums), nat.stream())
nat.load().cvz_fa2_shard_destroy(h, nat.stream())
text = "\n".join(f"{u} {v}" for u, v in e[:5000]) + "\n"
gp = cv.parse_edge_list(text)
with tempfile.TemporaryDirectory() as d:
    cv.export_supernodes_tsv(sg, os.path.join(d, "s.tsv"))
    cv.export_superedges_tsv(sg, os.path.join(d, "e.tsv"))
torch.cuda.synchronize()
print(f"sanitize workload {which} ok: n={g.node_count} m={g.edge_count} k={sg.node_count} "
      f"q={q:.4f}")
