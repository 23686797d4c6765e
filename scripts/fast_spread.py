import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2108_00529_b200 as cv
from paper_2108_00529_b200 import synth
torch.cuda.set_device(0)
for name in ("C1", "C2"):
    e = synth.config_graph(name)
    g = cv.from_edge_array(e)
    base = cv.degree_stats(g).mode_degree
    ts, qs, ks = [], [], []
    for _ in range(30):
        f = cv.detect_communities(g, cv.ThresholdSchedule(base=base), workers=1, mode="fast")
        lab = f.label
        c = np.sort(np.unique(lab, return_counts=True)[1])[::-1]
        ts.append(c[:10].sum() / len(lab)); ks.append(f.community_count); qs.append(cv.modularity(g, f))
    print(name, os.environ.get("CVZ_FAST_WINDOW_DIV", "def"), "top10", np.percentile(ts, [0, 25, 50, 75, 100]).round(4),
          "q", np.percentile(qs, [0, 50, 100]).round(4), "k", np.percentile(ks, [0, 50, 100]))
