"""Native edge-list loader: the C++ tokenizer
(cvz_parse_begin/take, host code -- runs here without a GPU) against a
restatement of C/graph.py:50-92's line loop, and the whole
parse_edge_list / load_edge_list (tokenizer + GPU first-seen remap) against
the oracle on the B200."""

import ctypes

import numpy as np
import pytest

from conftest import has_gpu
from oracle import oracle as orc
from paper_2108_00529_b200 import _native


def ref_tokens(text: str):
    """C/graph.py:65-86 up to the remap: (ext pairs, error) where error is
    (line, kind, tokens) with kind 1 = token count, 2 = non-integer."""
    out = []
    for no, line in enumerate(text.splitlines(), start=1):
        s = line.strip()
        if not s or s[0] in "#%":
            continue
        parts = s.split()
        if len(parts) != 2:
            return out, (no, 1, len(parts))
        try:
            u, v = int(parts[0]), int(parts[1])
        except ValueError:
            return out, (no, 2, 0)
        if u != v:
            out += [u, v]
    return out, None


def native_tokens(data: bytes, threads: int):
    lib = _native.load()
    h = ctypes.c_void_p()
    m, el = ctypes.c_int64(0), ctypes.c_int64(0)
    ec, et = ctypes.c_int(0), ctypes.c_int(0)
    rc = lib.cvz_parse_begin(data, len(data), threads, ctypes.byref(h), ctypes.byref(m),
                             ctypes.byref(el), ctypes.byref(ec), ctypes.byref(et))
    assert rc == 0
    if ec.value:
        return None, (el.value, ec.value, et.value if ec.value == 1 else 0)
    buf = np.empty(2 * m.value, np.int64)
    assert lib.cvz_parse_take(h, buf.ctypes.data_as(ctypes.c_void_p)) == 0
    return buf.tolist(), None


BREAKS = ["\n", "\r\n", "\r", "\v", "\f", "\x1c", "\x1d", "\x1e"]
SPACES = [" ", "\t", "  ", "\x1f", " \t "]


def random_text(rng, lines=200, bad=0.0):
    out = []
    for _ in range(lines):
        r = rng.random()
        if r < 0.08:
            line = rng.choice(["", "   ", "# comment 1 2", "% x", "  #c", "\t"])
        else:
            toks = []
            for _ in range(2):
                x = int(rng.integers(-50, 5000))
                t = str(x)
                q = rng.random()
                if q < 0.05 and x >= 10:
                    t = t[:1] + "_" + t[1:]
                elif q < 0.08:
                    t = "+" + t if x >= 0 else t
                elif q < 0.10:
                    t = "00" + t if x >= 0 else t
                toks.append(t)
            if rng.random() < 0.05:
                toks[1] = toks[0]                      # self-loop
            if rng.random() < bad:
                k = rng.integers(4)
                if k == 0:
                    toks.append("7")
                elif k == 1:
                    toks = toks[:1]
                elif k == 2:
                    toks[0] = rng.choice(["1.5", "x", "1__2", "_1", "1_", "--3", "0x10", "+"])
                else:
                    toks[1] = "1e3"
            sp = SPACES[rng.integers(len(SPACES))]
            line = SPACES[rng.integers(len(SPACES))] * int(rng.integers(2)) + sp.join(toks)
        out.append(line + BREAKS[rng.integers(len(BREAKS))])
    return "".join(out)


@pytest.mark.parametrize("threads", [1, 3, 16])
def test_tokenizer_matches_reference_loop(threads):
    rng = np.random.default_rng(threads)
    for trial in range(60):
        text = random_text(rng, lines=int(rng.integers(1, 300)), bad=0.0 if trial % 2 else 0.01)
        ref, err = ref_tokens(text)
        got, gerr = native_tokens(text.encode(), threads)
        assert gerr == err, (trial, gerr, err)
        if err is None:
            assert got == ref


def test_tokenizer_edge_cases():
    cases = {
        "1 2": ([1, 2], None),
        "1 2\n\n3 3\n4 5\r\n": ([1, 2, 4, 5], None),
        "\r\n\r\n1 x\n": ([], (3, 2, 0)),
        "1 2 3": ([], (1, 1, 3)),
        "a\rb c": ([], (1, 1, 1)),
        "1_000 -2": ([1000, -2], None),
        "9223372036854775807 -9223372036854775808": ([2**63 - 1, -2**63], None),
        "# only comments\n% here\n": ([], None),
        "1\x1f2 3": ([], (1, 1, 3)),     # \x1f is whitespace, not a line break
        "1 2\x1c3 4": ([1, 2, 3, 4], None),
    }
    for text, (pairs, err) in cases.items():
        got, gerr = native_tokens(text.encode(), 2)
        assert gerr == err, text
        if err is None:
            assert got == pairs, text
        assert ref_tokens(text) == (pairs if err is None else ref_tokens(text)[0], err), text
    # outside the native subset -> code 3 (caller falls back to the Python loop)
    for text in ("1 2\n3 99999999999999999999", "# café\n1 2", "1 2 3 4"):
        _, gerr = native_tokens(text.encode(), 1)
        assert gerr[1] == 3, text


def test_edge_cache_format_round_trip(tmp_path):
    """Binary edge cache: header + array round trip, int64
    widening for ids >= 2^31, and the ParseErrors of a bad file (host only)."""
    from paper_2108_00529_b200 import graph as G
    rng = np.random.default_rng(3)
    e = rng.integers(0, 1000, size=(5000, 2))
    p = tmp_path / "g.cvzb"
    G._write_cache_arrays(p, 1200, e)
    n, back = G._read_cache_arrays(p)
    assert n == 1200 and back.dtype == np.dtype("<i4") and np.array_equal(back, e)
    assert p.stat().st_size == G._CACHE_HDR + e.size * 4
    wide = np.array([[0, 2**33], [5, 7]])
    G._write_cache_arrays(p, 2**33 + 1, wide)
    n, back = G._read_cache_arrays(p)
    assert n == 2**33 + 1 and back.dtype == np.dtype("<i8") and np.array_equal(back, wide)
    raw = p.read_bytes()
    for bad, msg in ((b"NOTCACHE" + raw[8:], "not a commviz edge cache"),
                     (raw[:-8], "truncated"),
                     (raw[:8] + b"\x02" + raw[9:], "version 2"),
                     (raw[:8], "not a commviz edge cache")):
        p.write_bytes(bad)
        with pytest.raises(G.ParseError, match=msg):
            G._read_cache_arrays(p)
    G._write_cache_arrays(p, 3, np.array([[0, 5]]))
    with pytest.raises(G.ParseError, match="outside"):
        G._read_cache_arrays(p)


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_edge_cache_load_matches_text(tmp_path):
    import paper_2108_00529_b200 as cv
    rng = np.random.default_rng(11)
    text = random_text(rng, lines=4000)
    g = cv.parse_edge_list(text)
    p = tmp_path / "g.cvzb"
    cv.write_edge_cache(g, p)
    for h in (cv.load_edge_list(str(p)), cv.read_edge_cache(p)):
        assert h.node_count == g.node_count
        assert np.array_equal(h.edges, g.edges) and np.array_equal(h.degree, g.degree)
    # isolated trailing ids survive (node_count comes from the header)
    g2 = cv.from_edge_array(np.array([[0, 1], [1, 2]]), node_count=10)
    cv.write_edge_cache(g2, p)
    h = cv.load_edge_list(str(p))
    assert h.node_count == 10 and h.degree.tolist() == [1, 2, 1] + [0] * 7


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_parse_edge_list_matches_oracle(tmp_path):
    import paper_2108_00529_b200 as cv
    rng = np.random.default_rng(7)
    for trial in range(8):
        text = random_text(rng, lines=int(rng.integers(5, 3000)))
        g = cv.parse_edge_list(text)
        n, e, deg = orc.parse_edge_list(text)
        assert g.node_count == n and np.array_equal(g.edges, e) and np.array_equal(g.degree, deg)
        gb = cv.parse_edge_list(text.encode())
        assert np.array_equal(gb.edges, e)
    # large random external ids (sparse 64-bit range) and a file
    ids = rng.integers(-2**62, 2**62, size=5000)
    pairs = ids[rng.integers(0, 5000, size=(40000, 2))]
    text = "\n".join(f"{a} {b}" for a, b in pairs) + "\n"
    p = tmp_path / "g.txt"
    p.write_text("# header\n" + text)
    g = cv.load_edge_list(str(p))
    n, e, deg = orc.parse_edge_list("# header\n" + text)
    assert g.node_count == n and np.array_equal(g.edges, e) and np.array_equal(g.degree, deg)
    # reference errors
    for bad, msg in (("1 2\n3\n", "line 2: expected two tokens, got 1"),
                     ("1 2\nx y\n", "line 2: non-integer token"),
                     ("# c\n\n", "no edges"), ("5 5\n", "no edges")):
        with pytest.raises(cv.ParseError, match=msg):
            cv.parse_edge_list(bad)
    # non-ASCII goes through the reference loop with the same result
    g = cv.parse_edge_list("# café\n10 20\n20 30\n")
    assert g.edges.tolist() == [[0, 1], [1, 2]]


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_run_pipeline_end_to_end(tmp_path):
    """C/cli.py:120-170 through the drop-in API: file -> artifacts, checked
    against the oracle run on the same edge list."""
    import json

    import paper_2108_00529_b200 as cv
    from paper_2108_00529_b200 import synth
    e = synth.planted_partition(3000, 30000, 30, seed=2)
    path = tmp_path / "g.txt"
    path.write_text("# planted\n" + "\n".join(f"{a + 1000}\t{b + 1000}" for a, b in e) + "\n")
    cv.warmup_jit()
    rep, sg, res = cv.run_pipeline(cv.PipelineConfig(input=str(path), outdir=str(tmp_path / "o"),
                                                     workers=1, iterations=20))
    n, ee, deg = orc.parse_edge_list(path.read_text())
    lab, _, hist = orc.detect_communities(n, ee, deg, orc.degree_stats(deg)[0], 10, 0, workers=1)
    A, B = orc.sketch_params(4, 0)
    t = np.zeros((4, orc.default_cols(len(ee))), np.int64)
    orc.sketch_add_many(t, A, B, lab, deg)
    k, se, w, mult, comm = orc.contract(ee, lab, t, A, B)
    assert (rep.node_count, rep.edge_count, rep.supernode_count, rep.superedge_count) == (
        n, len(ee), k, len(se))
    assert rep.rounds_run == len(hist)
    assert abs(rep.modularity - orc.modularity(ee, deg, lab)) <= 1e-9
    out = tmp_path / "o"
    for f in ("layout.svg", "nodes.tsv", "supernodes.tsv", "superedges.tsv", "hierarchy.tsv",
              "report.json"):
        assert (out / f).exists(), f
    se_f = np.loadtxt(out / "superedges.tsv", dtype=np.int64, skiprows=1).reshape(-1, 3)
    assert np.array_equal(se_f[:, :2], se) and np.array_equal(se_f[:, 2], mult)
    sn = np.loadtxt(out / "supernodes.tsv", dtype=np.int64, skiprows=1).reshape(-1, 3)
    assert np.array_equal(sn[:, 1], comm) and np.array_equal(sn[:, 2], w)
    assert json.loads((out / "report.json").read_text())["supernode_count"] == k
    with pytest.raises(cv.PipelineStageError, match="parse"):
        cv.run_pipeline(cv.PipelineConfig(input=str(tmp_path / "missing.txt"),
                                          outdir=str(out)))


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_run_ablation_rows(tmp_path):
    """C/cli.py:221-269 sweep: one row per setting, detection bit-exact vs the
    oracle at every threshold, TSV written with the reference's columns."""
    import paper_2108_00529_b200 as cv
    from paper_2108_00529_b200 import synth
    e = synth.planted_partition(2000, 20000, 20, seed=8)
    path = tmp_path / "g.txt"
    path.write_text("\n".join(f"{a} {b}" for a, b in e) + "\n")
    cfg = cv.PipelineConfig(input=str(path), outdir=str(tmp_path), workers=1)
    rows = cv.run_ablation(cfg, "threshold", str(tmp_path / "abl.tsv"))
    n, ee, deg = orc.parse_edge_list(path.read_text())
    for r in rows:
        lab, _, _ = orc.detect_communities(n, ee, deg, r["value"], 10, 0, workers=1)
        assert r["communities"] == len(np.unique(lab))
        assert abs(r["modularity"] - orc.modularity(ee, deg, lab)) <= 1e-9
        assert r["mean_weight_overshoot"] >= 0  # count-min never undercounts
    head = (tmp_path / "abl.tsv").read_text().splitlines()[0].split("\t")
    assert head == ["axis", "value", "communities", "supernodes", "superedges", "modularity",
                    "mean_weight_overshoot", "detect_ms"]
    with pytest.raises(ValueError):
        cv.run_ablation(cfg, "zoom")
