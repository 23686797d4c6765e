"""Fast-mode quality vs speed at a config: Q, community count and time of the
racy first pass against the deterministic result (dev tool; set
CVZ_FAST_WINDOW_DIV per process)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_00529_b200 as cv  # noqa: E402
from paper_2108_00529_b200 import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
torch.cuda.set_device(0)
g = cv.from_edge_array(torch.from_numpy(synth.config_graph(cfg)).cuda())
base = cv.degree_stats(g).mode_degree
det = cv.detect_communities(g, cv.ThresholdSchedule(base=base), workers=1)
qd = cv.modularity(g, det)
qs, ks, ts = [], [], []
for _ in range(5):
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record()
    f = cv.detect_communities(g, cv.ThresholdSchedule(base=base), workers=1, mode="fast")
    a1.record()
    torch.cuda.synchronize()
    ts.append(a0.elapsed_time(a1))
    qs.append(cv.modularity(g, f))
    ks.append(f.community_count)
print(f"{cfg} div={os.environ.get('CVZ_FAST_WINDOW_DIV', 'default')} "
      f"all={os.environ.get('CVZ_FAST_ALL', '0')} rounds={len(f.round_history)} Q_det={qd:.5f} "
      f"Q_fast={np.mean(qs):.5f}+-{np.std(qs):.5f} k_det={det.community_count} "
      f"k_fast={np.mean(ks):.0f} ms={np.median(ts[1:]):.3f}")
