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
    bad = T.TrainConfig(steps=0, lr=0, batch=3, head_dim=40, attn_mode="nope")
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


def _shard_worker(rank, world, port, out):
    import importlib.util
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        spec = importlib.util.spec_from_file_location(
            "bench_mod", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "bench.py"))
        bench = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(bench)
        owned = {}
        for units in (128, 40, 7, 3, 1):   # C2 B*H, C3 B*H, ragged splits
            h0, h1 = bench.shard_units(units, rank, world)
            mine = torch.zeros(units, dtype=torch.int64)
            mine[h0:h1] = 1
            dist.all_reduce(mine)          # every head owned by exactly one rank
            owned[units] = mine.numpy()
        out[rank] = owned
    finally:
        dist.destroy_process_group()


def test_bench_shard_plan_covers_every_head_once_gloo():
    """bench.py's multi-GPU plan: the named config's B*H heads split contiguously over
    the ranks, each (b, h) exactly once; world_size 2 over gloo."""
    world = 2
    out = mp.Manager().dict()
    mp.spawn(_shard_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for rank in range(world):
        for units, owned in out[rank].items():
            assert np.all(owned == 1), (units, owned)


def test_bench_shard_plan_all_world_sizes():
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "bench_mod", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    for world in (1, 2, 4, 8):
        for units in (128, 40, 32, 256, 5):
            spans = [bench.shard_units(units, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == units
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    assert [bench.shard_units(128, r, 8) for r in range(8)][3] == (48, 64)   # C2: 16 heads per GPU
    assert bench.shard_units(40, 7, 8) == (35, 40)                             # C3: 5 heads per GPU
    # both arms print the same workload description
    cfg = bench.parse_config("c2")
    assert bench.config_dict("c2", cfg, 8) == bench.config_dict("c2", cfg, 8)
    assert bench.config_dict("c2", cfg, 1)["parallelism"].startswith("dp1")
