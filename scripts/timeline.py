"""CUPTI timeline (torch.profiler) of one warm bench step: where the GPU is
idle.  Writes gpurun_out/timeline_<tag>.json.gz (chrome trace) and prints a
per-stage summary: GPU busy time vs wall time and the largest idle gaps with
the host API calls inside them.

    python scripts/timeline.py [--config C4] [--mode deterministic|fast]
"""
import argparse
import collections
import gzip
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_2108_00529_b200 as cv  # noqa: E402
from paper_2108_00529_b200 import synth  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="C4")
p.add_argument("--mode", default="deterministic")
p.add_argument("--tag", default="r1")
a = p.parse_args()
torch.cuda.set_device(0)
dev = torch.from_numpy(synth.config_graph(a.config)).to("cuda")
for _ in range(2):
    bench.pipeline(cv, dev, mode=a.mode)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA],
             with_stack=bool(os.environ.get("TL_STACK"))) as prof:
    with torch.profiler.record_function("step"):
        bench.pipeline(cv, dev, mode=a.mode)
    torch.cuda.synchronize()
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
path = os.path.join(ROOT, "gpurun_out", f"timeline_{a.tag}_{a.mode}.json")
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
with open(path, "rb") as fi, gzip.open(path + ".gz", "wb") as fo:
    fo.write(fi.read())
os.remove(path)
kern = sorted([e for e in ev if e.get("cat") == "kernel"], key=lambda e: e["ts"])
rt = sorted([e for e in ev if e.get("cat") in ("cuda_runtime", "cuda_driver")], key=lambda e: e["ts"])
t0, t1 = kern[0]["ts"], kern[-1]["ts"] + kern[-1]["dur"]
busy = sum(e["dur"] for e in kern)
print(f"kernels {len(kern)}  span {(t1 - t0) / 1000:.3f} ms  busy {busy / 1000:.3f} ms")
rtagg = collections.defaultdict(lambda: [0, 0.0])
for e in rt:
    rtagg[e["name"]][0] += 1
    rtagg[e["name"]][1] += e["dur"]
print("host runtime calls (count, total ms):")
for k, (c, d) in sorted(rtagg.items(), key=lambda kv: -kv[1][1])[:15]:
    print(f"  {c:6d} {d / 1000:9.3f}  {k}")
# true idle intervals: no kernel running on any stream (kernels of the
# side streams overlap the main stream's, so consecutive-start gaps mislead)
gaps = []
end, last = kern[0]["ts"] + kern[0]["dur"], kern[0]
for y in kern[1:]:
    g = y["ts"] - end
    if g > 20:
        gaps.append((g, last["name"][:60], y["name"][:60], end, y["ts"]))
    if y["ts"] + y["dur"] > end:
        end, last = y["ts"] + y["dur"], y
tot_gap = sum(g[0] for g in gaps)
print(f"gaps > 20us: {len(gaps)}  total {tot_gap / 1000:.3f} ms")
for g, a1, b1, s, e in sorted(gaps, reverse=True)[:25]:
    inside = collections.Counter(r["name"] for r in rt if r["ts"] >= s and r["ts"] < e)
    print(f"  {g / 1000:7.3f} ms after {a1!r} before {b1!r}  host: {dict(inside.most_common(4))}")
# the host calls inside the three largest idle intervals, in order
cpu = sorted([e for e in ev if e.get("cat") in ("cuda_runtime", "cuda_driver", "cpu_op",
                                                 "user_annotation", "python_function")],
             key=lambda e: e["ts"])
for g, a1, b1, s, e in sorted(gaps, reverse=True)[:3]:
    print(f"-- idle {g / 1000:.3f} ms after {a1!r}")
    for r in cpu:
        if r["ts"] >= s - 50 and r["ts"] < e and r.get("dur", 0) >= 5:
            print(f"   +{(r['ts'] - s) / 1000:7.3f} ms {r.get('dur', 0) / 1000:7.3f} ms "
                  f"{r.get('cat')}: {r['name'][:80]}")
