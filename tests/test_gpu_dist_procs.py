"""GPU, two real processes: the row-partitioned GCN epoch driven through
DistGCNTrainer + TorchDistExchange (torch.distributed, gloo backend so both
ranks can share the one GPU a test box has) on per-rank RowBlocks, against
the single-GPU GCNTrainer and the float64 oracle.  The same code path runs
over NCCL one process per GPU in bench.py --gpus N."""

import json
import os
import socket
import tempfile

import numpy as np
import pytest
import torch

from oracle import graph as og
from oracle import ops as oo

pytestmark = pytest.mark.gpu

V, E, F, HD, C, GSEED, XSEED = 5000, 80_000, 64, 16, 41, 3, 21


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist

    import paper_2605_29346_b200 as gb
    from paper_2605_29346_b200.dist import (DistGCNTrainer, RowPartition, TorchDistExchange,
                                            expected_bounds)

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    spec = gb.GraphGenSpec("power-law", V, E, exponent=2.1)
    bounds = expected_bounds(spec, world, 170.0)
    blk = gb.graph.powerlaw_row_block(spec, GSEED, int(bounds[rank]), int(bounds[rank + 1]),
                                      pack=False)
    part = RowPartition.from_block(blk, world, rank, bounds)
    tr = DistGCNTrainer(part, F, HD, C, seed=0)
    X = torch.empty(part.rows, F, device="cuda")
    gb.graph.fill_uniform(X, part.lo, XSEED)
    y = torch.empty(part.rows, dtype=torch.int64, device="cuda")
    gb.graph.fill_labels(y, part.lo, C, XSEED)
    tr.set_inputs(X, y)
    ex = TorchDistExchange()
    losses = []
    for _ in range(3):
        tr.step(ex)
        losses.append(tr.loss.item())
    res = {"losses": losses, "lo": part.lo, "hi": part.hi,
           "params": {k: v.cpu().tolist() for k, v in tr.params().items()},
           "grads": {k: v.cpu().tolist() for k, v in tr.grads().items()}}
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump(res, f)
    dist.barrier()
    dist.destroy_process_group()


def test_two_process_dist_trainer_matches_single_gpu_and_oracle(cuda):
    import torch.multiprocessing as mp

    import paper_2605_29346_b200 as gb
    from paper_2605_29346_b200.models import GCNTrainer, glorot

    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(2, _free_port(), d), nprocs=2, start_method="spawn",
                           join=True)
        res = [json.load(open(os.path.join(d, f"rank{r}.json"))) for r in range(2)]
    # single-GPU trainer on the whole graph, same synthetic inputs
    g = gb.generate(gb.GraphGenSpec("power-law", V, E, exponent=2.1), GSEED)
    Xf = torch.empty(V, F, device="cuda")
    gb.graph.fill_uniform(Xf, 0, XSEED)
    yf = torch.empty(V, dtype=torch.int64, device="cuda")
    gb.graph.fill_labels(yf, 0, C, XSEED)
    single = GCNTrainer(g, F, HD, C, seed=0, coalesced=True)
    single.set_inputs(Xf, yf)
    ls = []
    for i in range(3):
        if i == 0:  # the first step's gradients against the float64 oracle
            single.forward_backward()
            torch.cuda.synchronize()
            off, tgt = g.offsets, g.targets
            t_off, t_rows, _ = og.transpose(V, V, off, tgt)
            ref = oo.gcn2_step(off, tgt, t_off, t_rows, Xf.cpu().numpy(),
                               glorot(F, HD, 0, 0).astype(np.float64), np.zeros(HD),
                               glorot(HD, C, 0, 2).astype(np.float64), np.zeros(C),
                               yf.cpu().numpy())
            for r in res:
                assert abs(r["losses"][0] - ref["loss"]) <= 1e-5 * abs(ref["loss"])
            single.k_adam()
            ls.append(single.loss.item())
        else:
            ls.append(single.step().item())
    for r in res:
        assert np.allclose(r["losses"], ls, rtol=1e-4), (r["losses"], ls)
        for k, v in single.params().items():
            assert np.allclose(np.array(r["params"][k]), v.cpu().numpy(), rtol=1e-4, atol=1e-6), k
    # replicas stay identical (one all-reduce of the gradients per step)
    for k in res[0]["params"]:
        assert res[0]["params"][k] == res[1]["params"][k]
    assert res[0]["hi"] == res[1]["lo"] and res[0]["lo"] == 0 and res[1]["hi"] == V
