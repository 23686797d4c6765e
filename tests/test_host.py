"""Host-side logic of the drop-in package that needs no GPU: validation,
schedules, seeded RNG parameters (checked against the reference goldens)."""

import numpy as np
import pytest

import paper_2108_00529_b200 as cv
from conftest import cases, golden
from oracle import oracle as orc


def test_schedule_matches_golden():
    d = golden("community")
    for i in cases(d, "s"):
        m, w, s, mode = (int(x) for x in d[f"s{i}_args"])
        out = cv.make_schedule(m, w, s, ["random", "roundrobin"][mode])
        assert np.array_equal(out, d[f"s{i}_out"])


def test_schedule_properties():
    # /root/reference/pkg/tests/test_community.py:43-77
    assert cv.make_schedule(7, 1, 0).tolist() == list(range(7))
    for mode in ("random", "roundrobin"):
        assert sorted(cv.make_schedule(13, 4, 5, mode).tolist()) == list(range(13))
    order = cv.make_schedule(40, 4, 9, "random")
    for w in range(4):
        sub = [e for e in order if 10 * w <= e < 10 * (w + 1)]
        assert sub == list(range(10 * w, 10 * (w + 1)))
    assert not np.array_equal(cv.make_schedule(30, 3, 7), cv.make_schedule(30, 3, 8))
    with pytest.raises(ValueError):
        cv.make_schedule(4, 2, 0, "zigzag")
    rng = np.random.default_rng(0)
    for _ in range(200):
        m, w, s = int(rng.integers(1, 60)), int(rng.integers(1, 7)), int(rng.integers(0, 500))
        for mode in ("random", "roundrobin"):
            assert np.array_equal(cv.make_schedule(m, w, s, mode), orc.make_schedule(m, w, s, mode))


def test_threshold_schedule():
    s = cv.ThresholdSchedule(base=3, rounds=5)
    assert [s.threshold(i) for i in (1, 2, 3)] == [3, 9, 27]
    assert cv.ThresholdSchedule(base=1).base == 2
    with pytest.raises(ValueError):
        cv.ThresholdSchedule(base=0)
    with pytest.raises(ValueError):
        cv.ThresholdSchedule(base=2, rounds=0)


def test_default_workers_env(monkeypatch):
    monkeypatch.setenv("COMMVIZ_WORKERS", "2")
    assert cv.default_workers() == 2
    monkeypatch.setenv("COMMVIZ_WORKERS", "junk")
    assert cv.default_workers() == 4
    monkeypatch.delenv("COMMVIZ_WORKERS")
    assert cv.default_workers() == 4


def test_default_cols_and_params():
    assert [cv.default_cols(x) for x in (0, 100, 10**8, 65_000_001, 2**30)] == \
        golden("sketch")["default_cols"].tolist()
    with pytest.raises(ValueError):
        cv.LayoutParams(iterations=0)
    with pytest.raises(ValueError):
        cv.LayoutParams(gravity=-1)
    with pytest.raises(ValueError):
        cv.LayoutParams(repulsion=0)
    with pytest.raises(ValueError):
        cv.LayoutParams(theta=-0.1)
    with pytest.raises(ValueError):
        cv.LayoutParams(speed_form="cubic")
    with pytest.raises(ValueError):
        cv.LayoutParams(attraction_form="log")
    cv.LayoutParams(gravity=0.0)


def test_init_positions_and_masses():
    pos = cv.init_positions(400, seed=1)
    assert np.array_equal(pos, orc.init_positions(400, 1))
    assert np.all(np.abs(pos) <= 10.0)
    sg = cv.SuperGraph(node_count=2, edges=np.empty((0, 2), np.int64),
                       weight=np.array([0, 5]), multiplicity=np.empty(0, np.int64),
                       community_id=np.arange(2))
    from paper_2108_00529_b200.layout import _masses_and_edges
    assert _masses_and_edges(sg)[0].tolist() == [1.0, 5.0]


def test_graph_and_supergraph_validate():
    with pytest.raises(ValueError):
        cv.Graph(node_count=2, edges=np.zeros((2, 3), np.int64), degree=np.zeros(2, np.int64))
    with pytest.raises(ValueError):
        cv.Graph(node_count=2, edges=np.array([[0, 1]]), degree=np.array([2, 2]))
    with pytest.raises(ValueError):
        cv.SuperGraph(node_count=2, edges=np.zeros((1, 3), np.int64), weight=np.ones(2),
                      multiplicity=np.ones(1), community_id=np.arange(2))
    with pytest.raises(ValueError):
        cv.SuperGraph(node_count=2, edges=np.zeros((0, 2), np.int64), weight=np.ones(3),
                      multiplicity=np.zeros(0), community_id=np.arange(2))


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="CUDA device"):
        cv.from_edge_array(np.array([[0, 1]]))


def test_reference_arm_runs_the_shipped_package_on_c1():
    """bench.py's reference arm times oracle/_ref (the unmodified commviz
    package); on the CPU-runnable C1 shape its community count and
    supergraph size must equal the oracle restatement's."""
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import build_ref
    if not os.path.exists(build_ref.ZIP):
        pytest.skip("oracle/_ref not built here")
    pytest.importorskip("numba")
    import bench
    from paper_2108_00529_b200 import synth
    step = bench.reference_package_runner()
    m, secs, st = step("C1")
    e = synth.config_graph("C1", seed=0)
    n, ee, deg = orc.from_edge_array(e)
    lab, _, _ = orc.detect_communities(n, ee, deg, orc.degree_stats(deg)[0], 10, 0, workers=1)
    assert m == len(e) and secs > 0
    assert st["communities"] == len(np.unique(lab)) == st["supernodes"]
