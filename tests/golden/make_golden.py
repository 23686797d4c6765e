"""Generate golden vectors by running the REAL reference package in the build
container (PYTHONPATH=/root/reference/pkg/src).  The outputs are committed as
tests/golden/*.npz so that the oracle (oracle/oracle.py) can be pinned on the
GPU box, where /root/reference does not exist.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
import commviz as cv  # noqa: E402
from commviz.community import _resolve_labels, _scoda_pass, fresh_assignment  # noqa: E402
from commviz.layout import _attraction  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def rand_graph(rng, n, m, self_loops=False):
    e = rng.integers(0, n, size=(m, 2))
    if not self_loops:
        e = e[e[:, 0] != e[:, 1]]
    return e.astype(np.int64)


def planted(seed, cliques, size, bridges):
    rng = np.random.default_rng(seed)
    edges = []
    for c in range(cliques):
        b = c * size
        for i in range(size):
            for j in range(i + 1, size):
                edges.append((b + i, b + j))
    for _ in range(bridges):
        a, b2 = rng.choice(cliques, size=2, replace=False)
        edges.append((int(a * size + rng.integers(size)), int(b2 * size + rng.integers(size))))
    return np.array(edges, dtype=np.int64)


def sbm(seed, n, k, m, mu):
    """Small planted-partition stream (shuffled) for differential cases."""
    rng = np.random.default_rng(seed)
    comm = rng.integers(0, k, size=n)
    members = [np.flatnonzero(comm == c) for c in range(k)]
    members = [mb for mb in members if len(mb) >= 2]
    out = []
    for _ in range(m):
        if rng.random() < mu:
            u, v = rng.integers(0, n, size=2)
        else:
            mb = members[rng.integers(len(members))]
            u, v = mb[rng.integers(len(mb))], mb[rng.integers(len(mb))]
        if u != v:
            out.append((u, v))
    return np.array(out, dtype=np.int64)


def graph_cases():
    rng = np.random.default_rng(1)
    d = {}
    for i in range(8):
        n = int(rng.integers(2, 400))
        m = int(rng.integers(1, 3000))
        e = rand_graph(rng, n, m, self_loops=True)
        nc = None if i % 2 == 0 else n + int(rng.integers(0, 5))
        g = cv.from_edge_array(e, node_count=nc)
        st = cv.degree_stats(g)
        d[f"g{i}_in"] = e
        d[f"g{i}_nc"] = np.array([-1 if nc is None else nc])
        d[f"g{i}_edges"] = g.edges
        d[f"g{i}_degree"] = g.degree
        d[f"g{i}_n"] = np.array([g.node_count])
        d[f"g{i}_stats"] = np.array([st.mode_degree, st.average_degree, st.max_degree])
    return d


def community_cases():
    rng = np.random.default_rng(2)
    d = {}
    # single passes with random counters/labels, all tie rules, orders
    for i in range(24):
        n = int(rng.integers(2, 300))
        m = int(rng.integers(1, 2000))
        e = rand_graph(rng, n, m, self_loops=(i % 5 == 4))
        thr = int(rng.integers(1, 12))
        tie = i % 3
        deg = rng.integers(0, thr + 3, size=n).astype(np.int64)
        if i % 4 == 0:
            deg[:] = 0
        lab = rng.integers(0, n, size=n).astype(np.int64)
        if i % 3 == 0:
            lab = np.arange(n, dtype=np.int64)
        order = (np.arange(len(e), dtype=np.int64) if i % 2 == 0
                 else rng.permutation(len(e)).astype(np.int64))
        d[f"p{i}_edges"], d[f"p{i}_order"] = e, order
        d[f"p{i}_args"] = np.array([n, thr, tie])
        d[f"p{i}_deg0"], d[f"p{i}_lab0"] = deg.copy(), lab.copy()
        _scoda_pass(e, order, np.int64(thr), tie, deg, lab)
        d[f"p{i}_deg"], d[f"p{i}_lab"] = deg, lab
    # resolve on random functional graphs
    for i in range(12):
        n = int(rng.integers(1, 500))
        lab = rng.integers(0, n, size=n).astype(np.int64)
        if i % 2:
            lab = np.where(rng.random(n) < 0.5, np.arange(n), lab)
        d[f"r{i}_in"] = lab
        d[f"r{i}_out"] = _resolve_labels(lab)
    # schedules
    for i, (m, w, s, mode) in enumerate([(37, 4, 5, "random"), (1000, 3, 9, "random"),
                                         (50, 7, 1, "roundrobin"), (999, 4, 11, "random"),
                                         (2, 4, 0, "random"), (10, 1, 0, "random")]):
        d[f"s{i}_args"] = np.array([m, w, s, 0 if mode == "random" else 1])
        d[f"s{i}_out"] = cv.make_schedule(m, w, s, mode)
    # full detection
    graphs = [planted(0, 8, 16, 8), planted(3, 40, 12, 60), sbm(5, 3000, 30, 20000, 0.1),
              sbm(6, 800, 10, 5000, 0.3), rand_graph(np.random.default_rng(7), 500, 3000)]
    cfgs = [dict(workers=1, interleave="random", round_stream="contract", tie_rule="src-joins-dst"),
            dict(workers=4, interleave="random", round_stream="contract", tie_rule="src-joins-dst"),
            dict(workers=3, interleave="roundrobin", round_stream="contract", tie_rule="dst-joins-src"),
            dict(workers=1, interleave="random", round_stream="restream", tie_rule="skip")]
    c = 0
    for gi, e in enumerate(graphs):
        g = cv.from_edge_array(e)
        for ci, cfg in enumerate(cfgs):
            base = [2, 0][ci % 2] or cv.degree_stats(g).mode_degree
            a = cv.detect_communities(g, cv.ThresholdSchedule(base=base, rounds=10),
                                      seed=3 + gi, **cfg)
            d[f"d{c}_edges"] = g.edges
            d[f"d{c}_args"] = np.array([g.node_count, base, 10, 3 + gi, cfg["workers"],
                                        0 if cfg["interleave"] == "random" else 1,
                                        0 if cfg["round_stream"] == "contract" else 1,
                                        {"src-joins-dst": 0, "dst-joins-src": 1, "skip": 2}[cfg["tie_rule"]]])
            d[f"d{c}_label"] = a.label
            d[f"d{c}_counter"] = a.counter_degree
            d[f"d{c}_history"] = np.stack(a.round_history)
            c += 1
    return d


def sketch_cases():
    d = {}
    for i, (rows, seed) in enumerate([(4, 0), (1, 3), (6, 11), (2, 5)]):
        s = cv.sketch_new(rows, 97, seed)
        d[f"h{i}_args"] = np.array([rows, seed])
        d[f"h{i}_a"], d[f"h{i}_b"] = s.hash_a, s.hash_b
    rng = np.random.default_rng(3)
    for i in range(10):
        rows = int(rng.integers(1, 6))
        cols = int(rng.integers(4, 7000))
        k = int(rng.integers(1, 20000))
        keys = rng.integers(-2**40, 2**40, size=k) if i % 3 == 0 else rng.integers(0, 5000, size=k)
        amounts = rng.integers(0, 10**6, size=k)
        s = cv.sketch_new(rows, cols, seed=i)
        cv.sketch_add_many(s, keys, amounts)
        probe = np.concatenate([keys[:500], rng.integers(0, 2**35, size=100)])
        d[f"a{i}_args"] = np.array([rows, cols, i])
        d[f"a{i}_keys"], d[f"a{i}_amounts"] = keys.astype(np.int64), amounts.astype(np.int64)
        d[f"a{i}_table"] = s.table
        d[f"a{i}_probe"] = probe.astype(np.int64)
        d[f"a{i}_est"] = cv.sketch_estimate_many(s, probe)
        d[f"a{i}_idx"] = s._indices(probe)
    # saturation
    s = cv.sketch_new(2, 8, seed=0)
    big = np.iinfo(np.int64).max - 5
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        cv.sketch_add_many(s, np.array([0, 1, 0]), np.array([big, 3, big]))
    d["sat_table"] = s.table
    d["default_cols"] = np.array([cv.default_cols(x) for x in (0, 100, 10**8, 65_000_001, 2**30)])
    return d


def contract_cases():
    rng = np.random.default_rng(4)
    d = {}
    for i in range(10):
        n = int(rng.integers(3, 3000))
        e = rand_graph(rng, n, int(rng.integers(2, 20000)))
        g = cv.from_edge_array(e, node_count=n)
        if i % 3 == 0:
            labels = rng.integers(0, max(2, n // 10), size=n)
        elif i % 3 == 1:
            labels = rng.integers(-10**12, 10**12, size=max(2, n // 7))[rng.integers(0, max(2, n // 7), size=n)]
        else:
            a = cv.detect_communities(g, cv.ThresholdSchedule(base=3), seed=i, workers=1)
            labels = a.label
        labels = labels.astype(np.int64)
        s = cv.sketch_new(4, int(rng.integers(16, 7000)), seed=i)
        cv.accumulate_sizes(s, labels, g.degree)
        sg = cv.contract(g, labels, s)
        d[f"c{i}_edges"], d[f"c{i}_n"] = g.edges, np.array([n])
        d[f"c{i}_labels"] = labels
        d[f"c{i}_sk"] = np.array([s.rows, s.cols, i])
        d[f"c{i}_table"] = s.table
        d[f"c{i}_se"], d[f"c{i}_w"] = sg.edges, sg.weight
        d[f"c{i}_mult"], d[f"c{i}_comm"] = sg.multiplicity, sg.community_id
    return d


def layout_cases():
    rng = np.random.default_rng(5)
    d = {}
    # repulsion (BH + exact), including coincident and clustered points
    for i in range(10):
        n = int(rng.integers(2, 2000))
        pos = rng.uniform(-50, 50, (n, 2))
        if i == 3:
            pos = np.zeros((n, 2))
        if i == 4:
            pos[: n // 2] = pos[0]
        if i == 5:
            pos = rng.normal(0, 1e-3, (n, 2))
        mass = rng.uniform(1, 20, n)
        theta = [0.5, 0.0, 0.9, 0.5, 0.5, 0.3, 0.05, 1.2, 0.5, 0.7][i]
        d[f"f{i}_pos"], d[f"f{i}_mass"] = pos, mass
        d[f"f{i}_theta"] = np.array([theta])
        d[f"f{i}_out"] = cv.repulsion_forces(pos, mass, 80.0, theta)
    # attraction
    pos = rng.uniform(-5, 5, (50, 2))
    e = rand_graph(rng, 50, 300)
    w = rng.uniform(0.5, 3, len(e))
    out = rng.normal(size=(50, 2))
    d["att_pos"], d["att_edges"], d["att_w"], d["att_in"] = pos, e, w, out.copy()
    _attraction(pos, e, w, -1.0, out)
    d["att_out"] = out
    # full layouts on small supergraphs / graphs
    cases = []
    for gi, e in enumerate([planted(0, 8, 16, 8), planted(3, 40, 12, 60)]):
        g = cv.from_edge_array(e)
        a = cv.detect_communities(g, cv.ThresholdSchedule(base=2, rounds=10), seed=11, workers=1)
        sk = cv.sketch_new(4, cv.default_cols(g.edge_count), seed=0)
        cv.accumulate_sizes(sk, a.label, g.degree)
        cases.append(("sg", cv.contract(g, a.label, sk)))
    cases.append(("g", cv.from_edge_array(planted(1, 6, 10, 12))))
    for li, (kind, obj) in enumerate(cases):
        for pi, params in enumerate([dict(iterations=1), dict(iterations=30),
                                     dict(iterations=20, theta=0.0, speed_form="sum"),
                                     dict(iterations=15, gravity=0.0, attraction_form="reversed", theta=0.8)]):
            res = cv.layout(obj, cv.LayoutParams(seed=li, **params))
            key = f"l{li}_{pi}"
            d[key + "_kind"] = np.array([0 if kind == "sg" else 1])
            if kind == "sg":
                d[key + "_edges"], d[key + "_weight"], d[key + "_mult"] = obj.edges, obj.weight, obj.multiplicity
            else:
                d[key + "_edges"], d[key + "_degree"] = obj.edges, obj.degree
            d[key + "_params"] = np.array([params.get("iterations"), params.get("gravity", 1.0),
                                           params.get("theta", 0.5),
                                           0 if params.get("speed_form", "product") == "product" else 1,
                                           0 if params.get("attraction_form", "canonical") == "canonical" else 1,
                                           li])
            d[key + "_pos"], d[key + "_disp"] = res.positions, res.displacement
    return d


def _text(s):
    return np.frombuffer(s.encode("utf-8"), dtype=np.uint8)


def writers_cases():
    """Output formats (C/render.py, C/supergraph.py:79-91,
    C/community.py:284-294, C/graph.py:100-111, C/sketch.py:101-102,
    C/cli.py:200-215): the reference's exact text for small inputs."""
    import io
    import tempfile

    from commviz.cli import _export_nodes_tsv
    from commviz.render import ColorAssignment
    d = {}
    rng = np.random.default_rng(11)
    tmp = tempfile.mkdtemp()
    for i, n in enumerate([1, 7, 40, 300]):
        pos = rng.normal(size=(n, 2)) * (10.0 ** rng.integers(-4, 4))
        if n >= 7:
            pos[0] = [-0.0, -1e-4]          # "-0.000"
            pos[1] = [0.0005, -0.0005]       # exact ties of the decimal grid
            pos[2] = [1.0005, 2.5e-3]
        w = rng.integers(0, 50, size=n).astype(np.int64)
        alpha = [1.0, 0.5, 2.0, 1.3][i]
        col = cv.assign_colors(w, alpha=alpha)
        rad = cv.node_radii(pos, w)
        ne = 3 * n
        e = rng.integers(0, n, size=(ne, 2))
        mult = rng.integers(1, 9, size=ne)
        k = f"s{i}"
        d[k + "_pos"], d[k + "_w"], d[k + "_alpha"] = pos, w, np.float64(alpha)
        d[k + "_classes"], d[k + "_radii"] = col.classes, rad
        d[k + "_edges"], d[k + "_mult"] = e, mult
        for tag, kw in (("plain", {}), ("edges", dict(edges=e, multiplicity=mult)),
                        ("edges1", dict(edges=e))):
            buf = io.StringIO()
            cv.export_svg(buf, pos, rad, col, **kw)
            d[f"{k}_svg_{tag}"] = _text(buf.getvalue())
    # TSVs over a real pipeline result
    e = sbm(3, 300, 12, 2000, 0.1)
    g = cv.from_edge_array(e)
    a = cv.detect_communities(g, cv.ThresholdSchedule(base=cv.degree_stats(g).mode_degree),
                              seed=0, workers=4)
    s = cv.sketch_new(4, 97, seed=0)
    cv.accumulate_sizes(s, a.label, g.degree)
    sg = cv.contract(g, a.label, s)
    res = cv.layout(sg, cv.LayoutParams(iterations=5))
    col = cv.assign_colors(sg.weight)
    d["t_edges"] = e
    d["t_label"], d["t_hist"] = a.label, np.stack(a.round_history)
    d["t_table"], d["t_hash_a"], d["t_hash_b"] = s.table, s.hash_a, s.hash_b
    d["t_sg_edges"], d["t_sg_weight"] = sg.edges, sg.weight
    d["t_sg_mult"], d["t_sg_comm"] = sg.multiplicity, sg.community_id
    d["t_pos"] = res.positions
    d["t_full_pos"] = rng.normal(size=(g.node_count, 2))
    d["t_full_classes"] = cv.color_full_graph(a.label, sg.community_id, col)
    files = {
        "supernodes": lambda p: cv.export_supernodes_tsv(sg, p),
        "superedges": lambda p: cv.export_superedges_tsv(sg, p),
        "hierarchy": lambda p: cv.export_hierarchy_tsv(a, p),
        "edgelist": lambda p: cv.write_edge_list(g, p),
        "sketch": lambda p: cv.dump_tsv(s, p),
        "nodes": lambda p: _export_nodes_tsv(p, g, a, sg, col, res),
        "nodes_full": lambda p: _export_nodes_tsv(
            p, g, a, sg, col, cv.LayoutResult(d["t_full_pos"], np.zeros(1), 1), full=True),
    }
    for name, fn in files.items():
        path = os.path.join(tmp, name)
        fn(path)
        with open(path, encoding="utf-8") as fh:
            d["f_" + name] = _text(fh.read())
    full = ColorAssignment(classes=d["t_full_classes"])
    buf = io.StringIO()
    cv.export_svg(buf, d["t_full_pos"], np.full(g.node_count, 0.5), full, edges=g.edges)
    d["f_svg_full"] = _text(buf.getvalue())
    return d


def main():
    only = sys.argv[1:]
    for name, fn in [("graph", graph_cases), ("community", community_cases),
                     ("sketch", sketch_cases), ("contract", contract_cases),
                     ("layout", layout_cases), ("writers", writers_cases)]:
        if only and name not in only:
            continue
        d = fn()
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **d)
        print(name, len(d), os.path.getsize(path))


if __name__ == "__main__":
    main()
