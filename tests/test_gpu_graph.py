"""GPU parity: device graph builders vs the reference golden vectors and the
oracle — bit-exact (offsets, targets, CSC, edge ids, degrees)."""

import io
import json
import os

import numpy as np
import pytest

from oracle import graph as og

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def gb(cuda):
    import paper_2605_29346_b200 as gb

    return gb


def eq(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b))


def test_known_answers(gb):
    g = gb.load_edge_list(io.StringIO("0 1\n0 2\n1 2\n"))
    assert g.offsets.tolist() == [0, 2, 3, 3] and g.targets.tolist() == [1, 2, 2]
    g = gb.load_edge_list(io.StringIO("n=3\n"))
    assert g.num_vertices == 3 and g.offsets.tolist() == [0, 0, 0, 0] and g.targets.size == 0
    g = gb.load_edge_list(io.StringIO("0 5\n1 2\n0 3\n0 5\n"))
    assert g.neighbors(0).tolist() == [5, 3, 5]
    g = gb.load_edge_list(io.StringIO("0 1\n"), symmetrize=True)
    assert g.num_edges == 2 and g.neighbors(0).tolist() == [1] and g.neighbors(1).tolist() == [0]
    g = gb.load_edge_list(io.StringIO("5 1000\n1000 7\n"), compact_ids=True)
    assert g.num_vertices == 3 and g.neighbors(0).tolist() == [2] and g.neighbors(2).tolist() == [1]
    g = gb.csr_from_edges(3, np.array([0, 0, 0]), np.array([1, 1, 2]))
    assert g.neighbors(0).tolist() == [1, 1, 2]
    assert gb.total_degree(gb.load_edge_list(io.StringIO("n=4\n"))) == 0


def test_closed_form_generators(gb, golden):
    g = gb.generate(gb.GraphGenSpec("star", 5), 0)
    assert g.degree(0) == 4 and all(g.degree(v) == 0 for v in range(1, 5))
    g = gb.generate(gb.GraphGenSpec("complete", 3), 0)
    assert g.num_edges == 6 and g.degrees.tolist() == [2, 2, 2] and gb.total_degree(g) == 6
    g = gb.generate(gb.GraphGenSpec("ring", 4), 0)
    assert g.neighbors(3).tolist() == [0] and g.degrees.tolist() == [1, 1, 1, 1]
    for name, spec in (("star_5", ("star", 5)), ("ring_4", ("ring", 4)),
                       ("complete_3", ("complete", 3)), ("complete_17", ("complete", 17))):
        g = gb.generate(gb.GraphGenSpec(*spec), 0)
        assert eq(g.offsets, golden[f"{name}/offsets"]) and eq(g.targets, golden[f"{name}/targets"])


@pytest.mark.parametrize("name,n,m,ex,seed", [
    ("pl_1000_20000_s42", 1000, 20000, 2.1, 42),
    ("pl_10000_200000_s7", 10_000, 200_000, 2.1, 7),
    ("pl_2708_10556_s42", 2708, 10556, 2.1, 42),
    ("pl_3000_30000_e25_s5", 3000, 30000, 2.5, 5),
])
def test_powerlaw_generate_bit_exact(gb, golden, name, n, m, ex, seed):
    g = gb.generate(gb.GraphGenSpec("power-law", n, m, exponent=ex), seed)
    assert eq(g.offsets, golden[f"{name}/offsets"])
    assert eq(g.targets, golden[f"{name}/targets"])
    assert eq(g.degrees, np.diff(golden[f"{name}/offsets"]))


def test_powerlaw_draws_match_numpy_stream(gb):
    from paper_2605_29346_b200.graph import powerlaw_edges_device

    for n, m, seed in ((50, 3001, 1), (100_000, 1_000_003, 99)):
        s, d = powerlaw_edges_device(n, m, 2.1, seed)
        rs, rd = og.powerlaw_edges(n, m, 2.1, seed)
        assert eq(s.cpu().numpy(), rs) and eq(d.cpu().numpy(), rd)


def test_uniform_generate(gb, golden):
    g = gb.generate(gb.GraphGenSpec("uniform-random", 500, 5000), 43)
    assert eq(g.offsets, golden["ur_500_5000_s43/offsets"])
    assert eq(g.targets, golden["ur_500_5000_s43/targets"])
    g = gb.generate(gb.GraphGenSpec("uniform-random", 100, 0.02), 5)
    assert g.num_edges == 200
    assert eq(g.targets, golden["ur_100_p002_s5/targets"])


@pytest.mark.parametrize("name", ["edges_64_4000", "edges_70000_300000"])
def test_csr_from_edges_stable(gb, golden, name):
    n = int(golden[f"{name}/offsets"].size - 1)
    g = gb.csr_from_edges(n, golden[f"{name}/src"], golden[f"{name}/dst"])
    assert eq(g.offsets, golden[f"{name}/offsets"]) and eq(g.targets, golden[f"{name}/targets"])


@pytest.mark.parametrize("n", [1, 2, 15, 16, 17, 2047, 2048, 2049, 70_000, 5_000_000])
def test_csr_from_edges_key_widths(gb, n):
    # exercises every radix width / pass count, including V=1 and tail tiles
    rng = np.random.default_rng(n)
    m = 50_000 + (n % 7)
    src = rng.integers(0, n, m)
    dst = rng.integers(0, n, m)
    g = gb.csr_from_edges(n, src, dst)
    off, tgt = og.csr_from_edges(n, src, dst)
    assert eq(g.offsets, off) and eq(g.targets, tgt)


def test_csr_from_edges_empty_and_skewed(gb):
    g = gb.csr_from_edges(4, np.array([], dtype=np.int64), np.array([], dtype=np.int64))
    assert g.offsets.tolist() == [0, 0, 0, 0, 0] and g.targets.size == 0
    src = np.zeros(100_000, dtype=np.int64)  # every edge in row 0
    dst = np.arange(100_000, dtype=np.int64) % 7
    g = gb.csr_from_edges(7, src, dst)
    assert eq(g.targets, dst) and g.offsets.tolist() == [0] + [100_000] * 7


def test_builder_errors(gb):
    with pytest.raises(gb.RangeError):
        gb.csr_from_edges(3, np.array([0, 1]), np.array([1, 3]))
    with pytest.raises(ValueError):
        gb.csr_from_edges(3, np.array([0, 3]), np.array([1, 1]))
    with pytest.raises(ValueError):
        gb.csr_from_edges(3, np.array([-1, 0]), np.array([1, 1]))
    with pytest.raises(ValueError):
        gb.make_csr(2, np.array([0, 2, 1]), np.array([0, 1]))
    with pytest.raises(ValueError):
        gb.make_csr(2, np.array([0, 1]), np.array([0]))
    with pytest.raises(ValueError):
        gb.make_csr(2, np.array([1, 1, 2]), np.array([0, 1]))
    with pytest.raises(gb.RangeError):
        gb.make_csr(2, np.array([0, 1, 2]), np.array([0, 5]))
    with pytest.raises(gb.ConfigError):
        gb.generate(gb.GraphGenSpec("uniform-random", 10, 101), 0)


def test_subgraph_csr(gb, golden):
    off, tgt = gb.build_subgraph_csr(np.array([0, 0, 2]), np.array([1, 2, 1]), 3)
    assert off.tolist() == [0, 2, 2, 3] and tgt.tolist() == [1, 2, 1]
    off, tgt = gb.build_subgraph_csr(np.array([]), np.array([]), 2)
    assert off.tolist() == [0, 0, 0] and tgt.size == 0
    with pytest.raises(IndexError):
        gb.build_subgraph_csr(np.array([3]), np.array([0]), 3)
    for h in range(2):
        k = f"subgraph_hop{h}"
        off, tgt = gb.build_subgraph_csr(golden[f"{k}/edge_src"], golden[f"{k}/edge_dst"],
                                         int(golden[f"{k}/num_local"][0]))
        assert eq(off, golden[f"{k}/offsets"]) and eq(tgt, golden[f"{k}/targets"])
        assert off[-1] == tgt.size == golden[f"{k}/edge_src"].size


def test_csc_and_eid(gb, golden):
    off, tgt = golden["pl_1000_20000_s42/offsets"], golden["pl_1000_20000_s42/targets"]
    g = gb.make_csr(1000, off, tgt)
    csc = g.csc(with_eid=True)
    assert eq(csc.offsets.cpu(), golden["pl_1000_20000_s42/csc_offsets"])
    assert eq(csc.cols.cpu(), golden["pl_1000_20000_s42/csc_rows"])
    _, _, eid = og.transpose(1000, 1000, off, tgt)
    assert eq(csc.eid.cpu(), eid)


def test_coalesced(gb, golden):
    off, tgt = golden["pl_10000_200000_s7/offsets"], golden["pl_10000_200000_s7/targets"]
    g = gb.make_csr(10_000, off, tgt)
    co = g.csr_coalesced()
    c_off, c_cols, mult = og.coalesce(10_000, off, tgt)
    assert eq(co.offsets.cpu(), c_off) and eq(co.cols.cpu(), c_cols)
    assert eq(co.vals.cpu().numpy().astype(np.float64), mult)
    t_off, t_rows, _ = og.transpose(10_000, 10_000, off, tgt)
    cc = g.csc_coalesced()
    c2_off, c2_cols, mult2 = og.coalesce(10_000, t_off, t_rows)
    assert eq(cc.offsets.cpu(), c2_off) and eq(cc.cols.cpu(), c2_cols)
    assert eq(cc.vals.cpu().numpy().astype(np.float64), mult2)


def test_csr1_roundtrip_bytes(gb, tmp_path):
    ref = os.path.join(GOLDEN, "csr1_small.bin")
    g = gb.load_csr(ref)
    out = tmp_path / "x.csr"
    gb.save_csr(g, out)
    assert out.read_bytes() == open(ref, "rb").read()
    bad = tmp_path / "bogus.csr"
    bad.write_bytes(b"NOPE" + b"\0" * 16)
    with pytest.raises(gb.ParseError):
        gb.load_csr(bad)


def test_edge_list_golden(gb, golden):
    g = gb.load_edge_list(io.StringIO("# c\n0 5\n1 2\n0 3\n0 5\n7 1\nn=9\n"))
    assert eq(g.offsets, golden["edgelist_a/offsets"]) and eq(g.targets, golden["edgelist_a/targets"])
    g = gb.load_edge_list(io.StringIO("5 1000\n1000 7\n7 5\n"), symmetrize=True, compact_ids=True)
    assert eq(g.offsets, golden["edgelist_b/offsets"]) and eq(g.targets, golden["edgelist_b/targets"])


@pytest.mark.slow
@pytest.mark.parametrize("name", ["reddit_s42", "products_s42"])
def test_full_size_generate_digest(gb, name):
    """Reddit/products-shape graphs generated + CSR/CSC-built on device must
    hash-match the reference's own generate() + transposed build."""
    import hashlib

    path = os.path.join(GOLDEN, "digests.json")
    if not os.path.exists(path):
        pytest.skip("digests.json not generated")
    d = json.load(open(path))[name]
    g = gb.generate(gb.GraphGenSpec("power-law", d["num_vertices"], d["num_edges"],
                                    exponent=d["exponent"]), d["seed"])
    h = lambda t: hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest()  # noqa: E731
    assert h(g.d_offsets) == d["offsets_sha256"]
    assert h(g.d_targets) == d["targets_sha256"]
    csc = g.csc()
    assert h(csc.offsets) == d["csc_offsets_sha256"]
    assert h(csc.cols) == d["csc_rows_sha256"]


def test_csr1_streamed_ingest_chunks(gb, tmp_path):
    """load_csr streams the arrays through pinned staging buffers straight to
    device: a file spanning many (tiny) chunks round-trips bit-exactly."""
    import torch

    from paper_2605_29346_b200.graph import _stream_to_device

    g = gb.generate(gb.GraphGenSpec("power-law", 20_000, 300_000, exponent=2.1), 3)
    path = tmp_path / "g.csr1"
    gb.save_csr(g, path)
    h = gb.load_csr(path)
    assert np.array_equal(h.offsets, g.offsets) and np.array_equal(h.targets, g.targets)
    raw = np.arange(10_007, dtype=np.int32)
    dst = torch.empty(raw.size, dtype=torch.int32, device="cuda")
    _stream_to_device(io.BytesIO(raw.tobytes()), dst, raw.nbytes, chunk=1000)
    assert np.array_equal(dst.cpu().numpy(), raw)


@pytest.mark.parametrize("case", ["uniform", "gaps", "one_key", "skew"])
def test_sort_pairs_and_offsets_match_numpy(gb, case):
    """gnn_sort_pairs (stable LSD radix: ballot-ranked, shared-memory staged
    scatter) and gnn_offsets_from_keys (run boundaries + binary-searched long
    gaps) vs numpy's stable argsort and bincount -> cumsum (graph.py:110-114),
    bit-exact, including empty keys at the head, in long interior gaps and at
    the tail, and key ranges needing 1, 2 and 3 radix passes."""
    import torch
    from paper_2605_29346_b200.graph import _offsets_from_keys, _sort_pairs

    rng = np.random.default_rng(7)
    n = 300_001
    if case == "uniform":
        R = 3_000_000  # 22 bits: two 11-bit passes
        k = rng.integers(0, R, n)
    elif case == "gaps":
        R = 1 << 27  # three 9-bit passes; keys in a few clusters, huge empty gaps
        k = np.concatenate([rng.integers(1000, 1100, n // 3), rng.integers(5_000_000, 5_000_050, n // 3),
                            rng.integers(R - 300, R - 200, n - 2 * (n // 3))])
        rng.shuffle(k)
    elif case == "one_key":
        R = 100_000
        k = np.full(n, 777)
    else:
        R = 232_965  # Reddit rows: 2 passes of 9 bits, power-law skew
        k = np.minimum((rng.pareto(1.1, n) * 10).astype(np.int64), R - 1)
    v = rng.integers(-2**31, 2**31 - 1, n)
    kt = torch.from_numpy(k.astype(np.int32)).cuda()
    vt = torch.from_numpy(v.astype(np.int32)).cuda()
    ko, vo = _sort_pairs(kt, vt, R)
    order = np.argsort(k, kind="stable")
    assert eq(ko.cpu().numpy(), k[order])
    assert eq(vo.cpu().numpy(), v.astype(np.int32)[order])
    off = _offsets_from_keys(ko, R).cpu().numpy()
    ref = np.concatenate([[0], np.cumsum(np.bincount(k, minlength=R))])
    assert eq(off, ref)
