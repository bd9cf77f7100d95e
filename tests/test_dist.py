"""Multi-process (world_size 2, gloo, CPU) coverage of the data-parallel host
logic: batch sharding, gradient all-reduce, identical replicas, and the
equivalence of 2-rank training with single-process training on the full batch.
The attention operator is swapped for a plain fp32 torch attention here (the
B200 kernels need the GPU; they are covered by the -m gpu suites)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_00040_b200 import train as T


def ref_attn(q, k, v, causal, variant):
    s = (q.float() @ k.float().transpose(-1, -2)) / q.shape[-1] ** 0.5
    if causal:
        n = s.shape[-1]
        s = s.masked_fill(torch.ones(n, n, dtype=torch.bool).triu(1), float("-inf"))
    return (torch.softmax(s, -1) @ v.float()).to(q.dtype)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        layer, log = T.train(cfg, device="cpu", attn_fn=ref_attn)
        params = torch.cat([p.detach().flatten() for p in layer.parameters()])
        out[rank] = (params.numpy(), np.array(log.losses))
    finally:
        dist.destroy_process_group()


CFG = T.TrainConfig(steps=3, seq_len=16, batch=4, d_model=32, n_heads=2, head_dim=64, lr=1e-2,
                    compute_dtype="fp32")


def test_two_rank_training_matches_single_process():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, CFG, out), nprocs=world, join=True)
    p0, l0 = out[0]
    p1, l1 = out[1]
    np.testing.assert_array_equal(p0, p1)      # replicas stay identical
    np.testing.assert_array_equal(l0, l1)      # all-reduced loss
    layer, log = T.train(CFG, device="cpu", attn_fn=ref_attn)
    ps = torch.cat([p.detach().flatten() for p in layer.parameters()]).numpy()
    # fp32: shard-vs-full-batch reductions differ only in summation order
    np.testing.assert_allclose(l0, np.array(log.losses), rtol=1e-5)
    np.testing.assert_allclose(p0, ps, rtol=0, atol=1e-4)


def test_shard_is_contiguous_and_complete():
    a = np.arange(8 * 3).reshape(8, 3)
    parts = [T.shard((a,), r, 4)[0] for r in range(4)]
    np.testing.assert_array_equal(np.concatenate(parts), a)


def test_config_validation_lists_problems():
    bad = T.TrainConfig(steps=0, lr=0, batch=3, head_dim=96, attn_mode="nope")
    probs = bad.validate(world=2)
    assert len(probs) >= 5


def test_divergence_raises_stability_error():
    def exploding(q, k, v, causal, variant):
        return ref_attn(q, k, v, causal, variant) * float("inf")
    with pytest.raises(T.StabilityError) as ei:
        T.train(T.TrainConfig(steps=2, seq_len=8, batch=2, d_model=16, n_heads=1, head_dim=64),
                device="cpu", attn_fn=exploding)
    assert ei.value.step == 0


def test_make_task_copy_solution():
    X, t = T.make_task(3, 16, 32, 4)
    assert X.shape == (4, 16, 32) and t.shape == (4, 32)
    np.testing.assert_array_equal(X[:, -1], t)
