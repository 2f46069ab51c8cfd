"""GPU parity of the device sampled-block pipeline
against the reference sampler's own outputs (tests/golden/sampling.json,
made by tests/golden/make_golden_sampling.py from the unmodified gsbench) and
against the pinned oracle restatement at larger sizes: bit-exact."""

import json
import os

import numpy as np
import pytest
import torch

from oracle import graph as og
from oracle import sampler as osm

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "sampling.json")


@pytest.fixture(scope="module")
def gb(cuda):
    import paper_2605_29346_b200 as gb

    return gb


def _graph(gb, spec):
    kind, n, m, ex, gseed = spec
    if kind == "power-law":
        return gb.generate(gb.GraphGenSpec(kind, n, m, exponent=ex), gseed)
    return gb.generate(gb.GraphGenSpec(kind, n, m), gseed)


def test_device_sampler_matches_reference_golden(gb):
    from paper_2605_29346_b200.sampling import SampleConfig, sample_minibatch

    for case in json.load(open(GOLDEN)):
        g = _graph(gb, case["graph"])
        cfg = SampleConfig(batch_size=len(case["seeds"]), fanouts=tuple(case["fanouts"]))
        sg, meta = sample_minibatch(g, cfg, np.array(case["seeds"]), case["sample_seed"])
        ref = case["result"]
        assert sg.local_to_global.tolist() == ref["local_to_global"], case["graph"]
        assert list(meta.per_hop_vertex_counts) == ref["per_hop_vertex_counts"]
        assert list(meta.per_hop_edge_counts) == ref["per_hop_edge_counts"]
        assert meta.total_unique_vertices == ref["total_unique_vertices"]
        assert meta.total_edges == ref["total_edges"]
        for b, rb in zip(sg.hops, ref["hops"]):
            assert b.hop_index == rb["hop"]
            assert b.src_local.tolist() == rb["frontier_local"]
            assert b.dst_unique_local.tolist() == rb["new_unique_local"]
            assert b.edge_src.tolist() == rb["edge_src"]
            assert b.edge_dst.tolist() == rb["edge_dst"]


@pytest.mark.parametrize("batch,fanouts", [(1024, (25, 10)), (4096, (15, 10, 5)), (7, (0, 40))])
def test_device_sampler_matches_oracle_large(gb, batch, fanouts):
    """Reddit-scale base graph (100k vertices, 5M edges, power-law) — many
    thousands of draws per hop, skewed degrees, repeated destinations."""
    from paper_2605_29346_b200.sampling import SampleConfig, build_subgraph_csr, sample_minibatch

    g = gb.generate(gb.GraphGenSpec("power-law", 100_000, 5_000_000, exponent=2.1), 11)
    seeds = np.random.default_rng(batch).choice(100_000, size=batch, replace=False)
    sg, meta = sample_minibatch(g, SampleConfig(batch, fanouts), seeds, 2024)
    l2g, hops, vc, ec = osm.sample_minibatch(g.offsets, g.targets, seeds, fanouts, 2024)
    assert np.array_equal(sg.local_to_global, l2g)
    assert list(meta.per_hop_vertex_counts) == vc and list(meta.per_hop_edge_counts) == ec
    for b, h in zip(sg.hops, hops):
        for got, key in ((b.src_local, "frontier_local"), (b.dst_unique_local, "new_unique_local"),
                         (b.edge_src, "edge_src"), (b.edge_dst, "edge_dst")):
            assert np.array_equal(got, h[key]), key
        # the sampled block's CSR (device build) equals the reference recipe
        off, tgt = build_subgraph_csr(torch.from_numpy(b.edge_src.astype(np.int64)).cuda(),
                                      torch.from_numpy(b.edge_dst.astype(np.int64)).cuda(),
                                      sg.num_local_vertices)
        r_off, r_tgt = og.build_subgraph_csr(b.edge_src, b.edge_dst, sg.num_local_vertices)
        assert np.array_equal(off.cpu().numpy(), r_off) and np.array_equal(tgt.cpu().numpy(), r_tgt)


def test_device_sampler_errors(gb):
    from paper_2605_29346_b200.errors import ConfigError
    from paper_2605_29346_b200.sampling import (SampleConfig, SubgraphBuilder, dedup_relabel,
                                                sample_minibatch)

    g = gb.generate(gb.GraphGenSpec("power-law", 1000, 20000, exponent=2.1), 42)
    with pytest.raises(ConfigError):
        SampleConfig(0, (5,))
    with pytest.raises(ConfigError):
        SampleConfig(4, ())
    with pytest.raises(ConfigError):
        sample_minibatch(g, SampleConfig(4, (3,)), np.array([1, 2, 3]), 0)
    with pytest.raises(ConfigError):
        SubgraphBuilder(1000, np.array([1, 1, 2]))
    with pytest.raises(ConfigError):
        SubgraphBuilder(1000, np.array([5, 1000]))
    b = SubgraphBuilder(1000, np.array([1, 2]))
    with pytest.raises(ValueError):
        dedup_relabel(np.array([7]), np.array([3]), b, 1)


def test_device_sampler_on_device_and_deterministic(gb):
    from paper_2605_29346_b200.sampling import SampleConfig, gather_indices, sample_minibatch

    g = gb.generate(gb.GraphGenSpec("power-law", 20_000, 400_000, exponent=2.1), 3)
    seeds = np.arange(0, 20_000, 97)[:128]
    a, ma = sample_minibatch(g, SampleConfig(128, (10, 10)), seeds, 5, on_device=True)
    b, mb = sample_minibatch(g, SampleConfig(128, (10, 10)), seeds, 5)
    assert a.local_to_global.is_cuda
    assert np.array_equal(a.local_to_global.cpu().numpy(), b.local_to_global)
    assert ma == mb
    feat, lab = gather_indices(b)
    assert np.array_equal(lab, seeds)


@pytest.mark.parametrize("fanouts", [(10, 10), (25, 10, 5), (0, 7)])
def test_replayed_device_sampler_matches_oracle(gb, fanouts):
    """DeviceSampler (device-resident counts, capacity buffers, one CUDA-graph
    replay per mini-batch) reproduces the reference sampler bit-exactly over
    several replays with different seeds and RNG streams."""
    from paper_2605_29346_b200.sampling import DeviceSampler, SampleConfig

    g = gb.generate(gb.GraphGenSpec("power-law", 50_000, 2_000_000, exponent=2.1), 4)
    cfg = SampleConfig(256, fanouts)
    ds = DeviceSampler(g, cfg)
    ds.capture()
    off, tgt = g.offsets, g.targets
    for it in range(4):
        seeds = np.random.default_rng(it).choice(50_000, 256, replace=False)
        ds.run(seeds, 100 + it)
        sg, meta = ds.result()
        l2g, hops, vc, ec = osm.sample_minibatch(off, tgt, seeds, fanouts, 100 + it)
        assert np.array_equal(sg.local_to_global, l2g), it
        assert list(meta.per_hop_vertex_counts) == vc and list(meta.per_hop_edge_counts) == ec
        for b, h in zip(sg.hops, hops):
            for got, key in ((b.src_local, "frontier_local"), (b.dst_unique_local, "new_unique_local"),
                             (b.edge_src, "edge_src"), (b.edge_dst, "edge_dst")):
                assert np.array_equal(got, h[key]), (it, key)


@pytest.mark.parametrize("K", [100, 602, 3])
def test_gather_features(gb, K):
    from paper_2605_29346_b200.sampling import gather_features

    X = torch.rand(5000, K, device="cuda")
    ids = torch.from_numpy(np.random.default_rng(K).integers(0, 5000, 777)).cuda()
    out = gather_features(X, ids)
    assert torch.equal(out, X[ids])


def test_sampled_gcn_step_matches_oracle(cuda):
    """Mini-batch GCN on a sampled subgraph (SampledGCNTrainer): loss over the
    B seeds and every parameter gradient equal the float64 oracle run on the
    same local subgraph (A_s from the sampled hop edges, X rows of the
    sampled vertices, labels of the seeds)."""
    import paper_2605_29346_b200 as gb
    from oracle import graph as og
    from oracle import ops as oo
    from paper_2605_29346_b200.models import SampledGCNTrainer
    from paper_2605_29346_b200.sampling import SampleConfig

    g = gb.generate(gb.GraphGenSpec("power-law", 5000, 100_000, exponent=2.1), 11)
    rng = np.random.default_rng(4)
    F, Hd, C, B = 48, 16, 9, 64
    X = torch.from_numpy(rng.uniform(-1, 1, (5000, F)).astype(np.float32)).cuda()
    y = torch.from_numpy(rng.integers(0, C, 5000)).cuda()
    tr = SampledGCNTrainer(g, X, y, F, Hd, C, SampleConfig(batch_size=B, fanouts=(5, 4)), seed=0)
    seeds = rng.choice(5000, B, replace=False)
    A, l2g, B_ = tr.subgraph(seeds, rng=7)
    tr.forward_backward(A, l2g, B_)
    torch.cuda.synchronize()
    off, tgt = A.offsets, A.targets
    n = A.num_vertices
    t_off, t_rows, _ = og.transpose(n, n, off, tgt)
    ids = l2g.cpu().numpy()
    assert np.array_equal(ids[:B], seeds)  # seeds are locals 0..B-1
    p = {k: v.double().cpu().numpy() for k, v in tr.params().items()}
    ref = oo.gcn2_step(off, tgt, t_off, t_rows, X.cpu().numpy()[ids], p["W1"], p["b1"], p["W2"],
                       p["b2"], y.cpu().numpy()[ids], loss_rows=B)
    assert abs(tr.loss.item() - ref["loss"]) <= 1e-5 * abs(ref["loss"])
    for k, gv in tr.grads().items():
        ok, worst = oo.close(gv.cpu().numpy(), ref[k], ref["abs"][k])
        assert ok, (k, worst)


def test_sampled_gcn_replay_matches_eager_and_oracle(cuda):
    """the replayed mini-batch step (capture + run: one CUDA
    graph per batch, envelope-sized buffers, device counts) builds exactly the
    eager step's local subgraph (CSR offsets / targets / local->global ids) and
    its loss and gradients equal the float64 oracle on that subgraph; replaying
    the same batch twice is bit-identical."""
    import paper_2605_29346_b200 as gb
    from oracle import graph as og
    from oracle import ops as oo
    from paper_2605_29346_b200.models import SampledGCNTrainer
    from paper_2605_29346_b200.sampling import SampleConfig

    g = gb.generate(gb.GraphGenSpec("power-law", 6000, 150_000, exponent=2.1), 12)
    rng = np.random.default_rng(5)
    F, Hd, C, B = 50, 16, 7, 128
    X = torch.from_numpy(rng.uniform(-1, 1, (6000, F)).astype(np.float32)).cuda()
    y = torch.from_numpy(rng.integers(0, C, 6000)).cuda()
    cfg = SampleConfig(batch_size=B, fanouts=(6, 4))
    tr = SampledGCNTrainer(g, X, y, F, Hd, C, cfg, seed=0)
    ref_tr = SampledGCNTrainer(g, X, y, F, Hd, C, cfg, seed=0)
    tr.capture(adam=False)
    Xh, yh = X.cpu().numpy(), y.cpu().numpy()
    for it in range(3):
        seeds = rng.choice(6000, B, replace=False)
        tr.run(seeds, rng=100 + it)
        off, tgt, ids, B_ = tr.replay_subgraph()
        A, l2g, _ = ref_tr.subgraph(seeds, rng=100 + it)
        assert np.array_equal(off, A.offsets) and np.array_equal(tgt, A.targets)
        assert np.array_equal(ids, l2g.cpu().numpy())
        n = off.size - 1
        t_off, t_rows, _ = og.transpose(n, n, off, tgt)
        p = {k: v.double().cpu().numpy() for k, v in tr.params().items()}
        ref = oo.gcn2_step(off, tgt, t_off, t_rows, Xh[ids], p["W1"], p["b1"], p["W2"], p["b2"],
                           yh[ids], loss_rows=B)
        assert abs(tr.loss.item() - ref["loss"]) <= 1e-5 * abs(ref["loss"])
        got = {k: v.clone() for k, v in tr.grads().items()}
        for k, gv in got.items():
            ok, worst = oo.close(gv.cpu().numpy(), ref[k], ref["abs"][k])
            assert ok, (it, k, worst)
        loss0 = tr.loss.item()
        tr.run(seeds, rng=100 + it)  # same batch again: bit-identical
        torch.cuda.synchronize()
        assert tr.loss.item() == loss0
        for k, gv in tr.grads().items():
            assert torch.equal(gv, got[k]), k


def test_sampled_gcn_replay_trains(cuda):
    import paper_2605_29346_b200 as gb
    from paper_2605_29346_b200.models import SampledGCNTrainer
    from paper_2605_29346_b200.sampling import SampleConfig

    g = gb.generate(gb.GraphGenSpec("power-law", 3000, 60_000, exponent=2.1), 5)
    rng = np.random.default_rng(1)
    yy = np.where(rng.random(3000) < 0.85, 0, rng.integers(0, 4, 3000))
    y = torch.from_numpy(yy).cuda()
    X = torch.randn(3000, 16, device="cuda")
    tr = SampledGCNTrainer(g, X, y, 16, 16, 4, SampleConfig(batch_size=128, fanouts=(5, 5)),
                           lr=0.05, seed=0)
    tr.capture()
    losses = [tr.run(rng.choice(3000, 128, replace=False), rng=it).item() for it in range(40)]
    assert np.mean(losses[-5:]) < np.mean(losses[:5]) - 0.1, losses


def test_sampled_gcn_training_lowers_the_loss(cuda):
    import paper_2605_29346_b200 as gb
    from paper_2605_29346_b200.models import SampledGCNTrainer
    from paper_2605_29346_b200.sampling import SampleConfig

    g = gb.generate(gb.GraphGenSpec("power-law", 3000, 60_000, exponent=2.1), 5)
    rng = np.random.default_rng(1)
    # skewed labels (85% class 0): learnable through the output bias even though
    # a seed's own features are not aggregated (no self loops in A_s)
    yy = np.where(rng.random(3000) < 0.85, 0, rng.integers(0, 4, 3000))
    y = torch.from_numpy(yy).cuda()
    X = torch.randn(3000, 16, device="cuda")
    tr = SampledGCNTrainer(g, X, y, 16, 16, 4, SampleConfig(batch_size=128, fanouts=(5, 5)),
                           lr=0.05, seed=0)
    losses = []
    for it in range(40):
        seeds = rng.choice(3000, 128, replace=False)
        losses.append(tr.step(seeds, rng=it).item())
    assert np.mean(losses[-5:]) < np.mean(losses[:5]) - 0.1, losses


def test_sample_hop_takes_reference_generator(gb):
    """sample_hop(graph, frontier, fanout, rng) with the reference's own
    np.random.Generator (sampler.py:118-123): same draws as gsbench's
    sample_hop (oracle restatement), and the generator ends at the same
    stream position, so consecutive calls keep matching."""
    from paper_2605_29346_b200.sampling import sample_hop

    g = gb.generate(gb.GraphGenSpec("power-law", 20_000, 400_000, exponent=2.1), 3)
    off, tgt = g.offsets, g.targets
    frontier = np.random.default_rng(0).choice(20_000, 300, replace=False)
    r_dev = np.random.default_rng(77)
    r_ref = np.random.default_rng(77)
    for fan in (5, 3):
        s, d = sample_hop(g, frontier, fan, r_dev)
        rs, rd = osm.sample_hop(off, tgt, frontier, fan, r_ref)
        assert np.array_equal(s.cpu().numpy(), rs) and np.array_equal(d.cpu().numpy(), rd)
        assert r_dev.bit_generator.state == r_ref.bit_generator.state


def test_device_sampler_rejects_bad_seeds(gb):
    """ConfigError (as SubgraphBuilder / the reference) for duplicate or
    out-of-range seeds — never an out-of-bounds device access; a replay after
    a rejected batch still matches the oracle."""
    from paper_2605_29346_b200.errors import ConfigError
    from paper_2605_29346_b200.sampling import DeviceSampler, SampleConfig

    g = gb.generate(gb.GraphGenSpec("power-law", 5_000, 100_000, exponent=2.1), 9)
    ds = DeviceSampler(g, SampleConfig(8, (4,)))
    ds.capture()
    with pytest.raises(ConfigError):
        ds.run(np.array([1, 2, 3, 4, 5, 6, 7, 7]))
    with pytest.raises(ConfigError):
        ds.run(np.array([1, 2, 3, 4, 5, 6, 7, 5_000]))
    with pytest.raises(ConfigError):
        ds.run(np.array([-1, 2, 3, 4, 5, 6, 7, 8]))
    seeds = np.arange(10, 18)
    for it in range(3):  # back-to-back replays without a sync in between
        ds.run(seeds + it, 5 + it)
    sg, _ = ds.result()
    l2g, *_ = osm.sample_minibatch(g.offsets, g.targets, seeds + 2, (4,), 7)
    assert np.array_equal(sg.local_to_global, l2g)
