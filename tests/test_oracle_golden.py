"""Pin the CPU oracle against golden vectors produced by the real reference
(tests/golden/make_golden.py).  Everything bit-exact, floats included: the
C restatement performs the same fp64 operations in the same order."""

import numpy as np
import pytest

from conftest import cases, golden
from oracle import oracle as orc

TIES = ["src-joins-dst", "dst-joins-src", "skip"]


def test_graph_golden():
    d = golden("graph")
    for i in cases(d, "g"):
        nc = int(d[f"g{i}_nc"][0])
        n, e, deg = orc.from_edge_array(d[f"g{i}_in"], None if nc < 0 else nc)
        assert n == d[f"g{i}_n"][0]
        assert np.array_equal(e, d[f"g{i}_edges"])
        assert np.array_equal(deg, d[f"g{i}_degree"])
        mode, mean, mx = orc.degree_stats(deg)
        assert [mode, mx] == [d[f"g{i}_stats"][0], d[f"g{i}_stats"][2]]
        assert mean == d[f"g{i}_stats"][1]


def test_scoda_pass_golden():
    d = golden("community")
    for i in cases(d, "p"):
        n, thr, tie = d[f"p{i}_args"]
        deg, lab = d[f"p{i}_deg0"].copy(), d[f"p{i}_lab0"].copy()
        orc.scoda_pass(d[f"p{i}_edges"], d[f"p{i}_order"], thr, tie, deg, lab)
        assert np.array_equal(deg, d[f"p{i}_deg"]), i
        assert np.array_equal(lab, d[f"p{i}_lab"]), i


def test_resolve_golden_and_kats():
    d = golden("community")
    for i in cases(d, "r"):
        assert np.array_equal(orc.resolve_labels(d[f"r{i}_in"]), d[f"r{i}_out"])
    # reference KATs, /root/reference/pkg/tests/test_community.py:30-40
    assert orc.resolve_labels([1, 2, 3, 3, 0]).tolist() == [3, 3, 3, 3, 3]
    assert orc.resolve_labels([1, 2, 0, 1, 4]).tolist() == [0, 0, 0, 0, 4]


def test_schedule_golden():
    d = golden("community")
    for i in cases(d, "s"):
        m, w, s, mode = d[f"s{i}_args"]
        out = orc.make_schedule(int(m), int(w), int(s), ["random", "roundrobin"][mode])
        assert np.array_equal(out, d[f"s{i}_out"])
    assert orc.make_schedule(8, 4, 0, "roundrobin").tolist() == [0, 2, 4, 6, 1, 3, 5, 7]


def test_detect_golden():
    d = golden("community")
    for i in cases(d, "d"):
        n, base, rounds, seed, workers, inter, rs, tie = d[f"d{i}_args"]
        e = d[f"d{i}_edges"]
        deg = np.bincount(e.ravel(), minlength=n).astype(np.int64)
        lab, cnt, hist = orc.detect_communities(
            int(n), e, deg, int(base), int(rounds), int(seed), TIES[tie], int(workers),
            ["random", "roundrobin"][inter], ["contract", "restream"][rs])
        assert np.array_equal(lab, d[f"d{i}_label"]), i
        assert np.array_equal(cnt, d[f"d{i}_counter"]), i
        assert np.array_equal(np.stack(hist), d[f"d{i}_history"]), i


def test_sketch_golden():
    d = golden("sketch")
    for i in cases(d, "h"):
        rows, seed = d[f"h{i}_args"]
        a, b = orc.sketch_params(int(rows), int(seed))
        assert np.array_equal(a, d[f"h{i}_a"]) and np.array_equal(b, d[f"h{i}_b"])
    # survey KAT
    a, b = orc.sketch_params(4, 0)
    assert a.tolist() == [1826701614, 1367864807, 1097657232, 579362556]
    assert b.tolist() == [661058651, 87989972, 161576974, 35492826]
    for i in cases(d, "a"):
        rows, cols, seed = (int(x) for x in d[f"a{i}_args"])
        a, b = orc.sketch_params(rows, seed)
        t = np.zeros((rows, cols), np.int64)
        orc.sketch_add_many(t, a, b, d[f"a{i}_keys"], d[f"a{i}_amounts"])
        assert np.array_equal(t, d[f"a{i}_table"])
        assert np.array_equal(orc.sketch_indices(a, b, cols, d[f"a{i}_probe"]), d[f"a{i}_idx"])
        assert np.array_equal(orc.sketch_estimate_many(t, a, b, d[f"a{i}_probe"]), d[f"a{i}_est"])
    a, b = orc.sketch_params(2, 0)
    t = np.zeros((2, 8), np.int64)
    big = np.iinfo(np.int64).max - 5
    assert orc.sketch_add_many(t, a, b, np.array([0, 1, 0]), np.array([big, 3, big]))
    assert np.array_equal(t, d["sat_table"])
    assert [orc.default_cols(x) for x in (0, 100, 10**8, 65_000_001, 2**30)] == d["default_cols"].tolist()


def test_contract_golden():
    d = golden("contract")
    for i in cases(d, "c"):
        rows, cols, seed = (int(x) for x in d[f"c{i}_sk"])
        a, b = orc.sketch_params(rows, seed)
        n = int(d[f"c{i}_n"][0])
        e = d[f"c{i}_edges"]
        deg = np.bincount(e.ravel(), minlength=n).astype(np.int64)
        t = np.zeros((rows, cols), np.int64)
        orc.sketch_add_many(t, a, b, d[f"c{i}_labels"], deg)
        assert np.array_equal(t, d[f"c{i}_table"])
        k, se, w, mult, comm = orc.contract(e, d[f"c{i}_labels"], t, a, b)
        assert np.array_equal(se, d[f"c{i}_se"]) and np.array_equal(w, d[f"c{i}_w"])
        assert np.array_equal(mult, d[f"c{i}_mult"]) and np.array_equal(comm, d[f"c{i}_comm"])


def test_repulsion_golden():
    d = golden("layout")
    for i in cases(d, "f"):
        out = orc.repulsion_forces(d[f"f{i}_pos"], d[f"f{i}_mass"], 80.0, float(d[f"f{i}_theta"][0]))
        assert np.array_equal(out, d[f"f{i}_out"]), i  # bit-exact restatement


def test_attraction_golden():
    d = golden("layout")
    out = d["att_in"].copy()
    orc.attraction(d["att_pos"], d["att_edges"], d["att_w"], -1.0, out)
    assert np.array_equal(out, d["att_out"])


def test_layout_golden():
    d = golden("layout")
    keys = sorted({k.rsplit("_", 1)[0] for k in d.files if k.startswith("l") and k.endswith("_pos")})
    for key in keys:
        it, g, theta, sf, af, seed = d[key + "_params"]
        e = d[key + "_edges"]
        if d[key + "_kind"][0] == 0:
            mass, ew = orc.masses_supergraph(d[key + "_weight"], d[key + "_mult"])
        else:
            mass, ew = orc.masses_graph(d[key + "_degree"], len(e))
        pos, disp = orc.layout(len(mass), mass, e, ew, iterations=int(it), seed=int(seed),
                               gravity=float(g), theta=float(theta),
                               speed_form=["product", "sum"][int(sf)],
                               attraction_form=["canonical", "reversed"][int(af)])
        assert np.array_equal(pos, d[key + "_pos"]), key  # bit-exact restatement
        assert np.array_equal(disp, d[key + "_disp"]), key
