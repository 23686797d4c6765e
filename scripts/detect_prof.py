"""Per-kernel device times of detect_communities at a config (dev tool)."""
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
base = cv.degree_stats(g).mode_degree
print("mode degree (threshold) =", base)
MODES = sys.argv[2].split(",") if len(sys.argv) > 2 else ["deterministic", "fast"]
for mode in MODES:
    for _ in range(2):
        a = cv.detect_communities(g, cv.ThresholdSchedule(base=base), workers=1, mode=mode)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    a = cv.detect_communities(g, cv.ThresholdSchedule(base=base), workers=1, mode=mode)
    e1.record()
    torch.cuda.synchronize()
    print(f"{mode}: {e0.elapsed_time(e1):.3f} ms rounds={len(a.round_history)} "
          f"m_r={list(a.stream_edges)} communities={a.community_count}")
    with _native.profile() as prof:
        cv.detect_communities(g, cv.ThresholdSchedule(base=base), workers=1, mode=mode)
    tot = sum(v[1] for v in prof.kernels.values())
    print(f"  profiled total {tot:.3f} ms")
    for name, (c, ms) in sorted(prof.kernels.items(), key=lambda kv: -kv[1][1])[:22]:
        print(f"  {c:4d} {ms:8.3f} ms  {name}")
