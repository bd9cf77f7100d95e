"""Benchmark of the B200 NVFP4 Attn-QAT path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c4|c5-<N>] [--impl ours|reference]

Default workload = BASELINE.json configs[1]: Llama-3-8B-shaped causal
inference forward, B=4 H=32 N=8192 d=128 (FP4). One step = one call of the
public operator (``attn_forward``: NVFP4 quantizers for Q/K/V + the fused
two-pass tcgen05 attention kernel) on inputs already resident in HBM.

Multi-GPU (torchrun, one process per GPU): every rank runs the full per-GPU
workload on its own batch (B x H heads are independent units; no
communication on the attention path) -> "scaling": "weak"; the timed region
is bracketed by barriers and the max over ranks is reported.

``--impl reference`` times the reference algorithm on the host CPU cores (the
oracle port in oracle/ -- the reference is pure NumPy), rank 0
only, on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FP4 attention fwd / fwd+bwd TFLOPS per B200 (d=128) and 1/2/4/8-GPU tokens/s"

CONFIGS = {
    # name: (B, H, N, d, causal, mode)
    "c1": (1, 2, 256, 64, False, "train"),
    "c2": (4, 32, 8192, 128, True, "fwd"),
    "c3": (1, 40, 32760, 128, False, "fwd"),
    "c4": (8, 32, 4096, 128, True, "train"),
    # C4 as a full data-parallel QAT layer step: projections + attention fwd/bwd +
    # NCCL gradient all-reduce + AdamW; global batch 8 sharded over ranks
    "c4-layer": (8, 32, 4096, 128, True, "layer"),
}


def parse_config(name):
    if name.startswith("c5-"):
        # sweep point: H=32 d=128, B = 65536/N, fwd+bwd, causal unless suffixed -nc
        parts = name.split("-")
        n = int(parts[1])
        causal = not (len(parts) > 2 and parts[2] == "nc")
        return (max(1, 65536 // n), 32, n, 128, causal, "train")
    return CONFIGS[name]


def alg_flops(B, H, N, d, causal, mode):
    """Algorithmic FLOPs: fwd = 4 B H N^2 d (x (N+1)/2N causal);
    fwd+bwd = 3.5 x fwd. QAT overheads (pass-1 QK^T, O' MMA) are not counted."""
    f = 4.0 * B * H * N * N * d
    if causal:
        f *= (N + 1) / (2.0 * N)
    return f * (3.5 if mode == "train" else 1.0)


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 7:
                    continue
                try:
                    sm.append(float(f[0]))
                    mx.append(float(f[1]))
                except ValueError:
                    continue
                for nm, v in zip(names, f[3:7]):
                    if v.lower() == "active":
                        reasons.add(nm)
        finally:
            os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU reference

def _cpu_head(args):
    # one BLAS thread per worker: the pool already runs one head per core, and
    # nested BLAS threads oversubscribe the host (100x slower backward)
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):
        return _cpu_head_body(*args)


def _cpu_head_body(n, d, causal, mode, seed):
    from oracle import nvfp4_attn_oracle as orc
    rng = np.random.default_rng(seed)
    Q, K, V = (rng.standard_normal((n, d)).astype(np.float32).astype(np.float64) for _ in range(3))
    t0 = time.perf_counter()
    if mode == "fwd":
        orc.forward_inference(Q, K, V, causal, 128, 128 if n % 128 == 0 else n, 32)
    else:
        dO = rng.standard_normal((n, d))
        bk = 128 if n % 128 == 0 else n
        O, L, Op = orc.forward_training(Q, K, V, causal, 128 if n % 128 == 0 else n, bk, 32, ordered=False)
        orc.backward(Q, K, V, dO, O, L, Op, causal, 128 if n % 128 == 0 else n, bk, 32, ordered=False)
    return time.perf_counter() - t0


class CpuReference:
    """Reference algorithm (oracle port) on all host cores: one head per process."""

    def __init__(self, cfg, max_n=8192):
        B, H, N, d, causal, mode = cfg
        self.cores = os.cpu_count() or 1
        self.n = min(N, max_n)   # heads at N > 8192 are sampled at 8192 and scaled by N^2
        self.N, self.d, self.causal, self.mode = N, d, causal, mode
        self.pool = ProcessPoolExecutor(max_workers=self.cores)
        list(self.pool.map(_cpu_head, [(256, d, causal, mode, i) for i in range(self.cores)]))  # warm

    def step(self, seed=0):
        t0 = time.perf_counter()
        list(self.pool.map(_cpu_head, [(self.n, self.d, self.causal, self.mode, seed * 1000 + i)
                                       for i in range(self.cores)]))
        dt = time.perf_counter() - t0
        flops = self.cores * alg_flops(1, 1, self.n, self.d, self.causal, self.mode)
        return flops / dt / 1e12, dt

    def sample(self):
        s = f"{self.cores} heads (one per process, 1 BLAS thread each) of N={self.n} d={self.d} {'causal' if self.causal else 'non-causal'}"
        s += " inference fwd" if self.mode == "fwd" else " training fwd+bwd"
        if self.n != self.N:
            s += f"; N={self.N} extrapolated from N={self.n} (N^2 scaling is already in the FLOP count)"
        return s + "; TFLOP/s = sample algorithmic FLOPs / wall time"

    def close(self):
        self.pool.shutdown()


def run_reference_arm(args, cfg, rank, world):
    if rank != 0:
        return
    ref = CpuReference(cfg)
    for i in range(args.warmup):
        ref.step(i)
    vals, times = [], []
    for i in range(args.steps):
        v, dt = ref.step(100 + i)
        vals.append(v)
        times.append(dt)
    ref.close()
    value = float(np.mean(vals))
    B, H, N, d, causal, mode = cfg
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(times)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64 (numpy)",
        "data": "synthetic N(0,1)",
        "config": {"workload": args.config, "B": B, "H": H, "N": N, "d": d, "causal": causal, "mode": mode},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": ref.cores, "kind": "port",
                         "sample": ref.sample()},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ----------------------------------------------------------------------------- GPU arm

def measure_mma_peaks(lib, torch):
    """Live tensor-pipe peaks (TFLOP/s) from the in-library probe: NVFP4 and bf16."""
    out = {}
    ctas = torch.cuda.get_device_properties(0).multi_processor_count
    st = torch.cuda.current_stream()
    for kind, name in ((0, "nvfp4"), (1, "bf16")):
        rounds = 20000 if kind == 0 else 5000
        lib.aq_probe_mma_peak(kind, ctas, rounds, st.cuda_stream)
        best = 0.0
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            lib.aq_probe_mma_peak(kind, ctas, rounds, st.cuda_stream)
            e1.record(st)
            e1.synchronize()
            best = max(best, lib.aq_probe_mma_flops(kind, ctas, rounds) / (e0.elapsed_time(e1) * 1e-3) / 1e12)
        out[name] = best
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = parse_config(args.config)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))

    if args.impl == "reference":
        run_reference_arm(args, cfg, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_2603_00040_b200 as aq
    from paper_2603_00040_b200 import _lib

    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    B, H, N, d, causal, mode = cfg
    if mode == "layer":
        run_layer_mode(args, cfg, rank, world, local)
        return
    dev = torch.device("cuda", local)
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    q, k, v = (torch.randn(B, H, N, d, generator=gen, device=dev).to(torch.bfloat16) for _ in range(3))
    lib = _lib.load()
    st = torch.cuda.current_stream()
    heads = B * H

    if mode == "fwd":
        ws = torch.empty(lib.aq_attn_fwd_workspace_bytes(heads, N, N, d, 0, 0), dtype=torch.uint8, device=dev)
        o = torch.empty(heads, N, d, dtype=torch.bfloat16, device=dev)
        lse = torch.empty(heads, N, dtype=torch.float32, device=dev)

        def step():
            aq.attn_forward(q, k, v, causal=causal, train=False, workspace=ws, out=o, lse_out=lse)
        launches_per_step = 4          # quantize Q, K (rows), V (cols), fused attention
    else:
        d_o = torch.randn(B, H, N, d, generator=gen, device=dev).to(torch.bfloat16)
        qg, kg, vg = (t.clone().requires_grad_() for t in (q, k, v))

        def step():
            for t_ in (qg, kg, vg):
                t_.grad = None
            out = aq.attn_qat(qg, kg, vg, causal=causal)
            out.backward(d_o)
        launches_per_step = 4 + 2      # fwd (3 quantizers + attention) + bwd pre, fused bwd (dK/dV + dQ roles)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    with ClockSampler(local) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(st)
        for _ in range(args.steps):
            step()
        e1.record(st)
        barrier()
    ms = e0.elapsed_time(e1) / args.steps
    clocks = clk.summary()
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    flops_rank = alg_flops(B, H, N, d, causal, mode)
    value = world * flops_rank / (ms_max * 1e-3) / 1e12
    tokens_s = world * B * N / (ms_max * 1e-3)

    # ---- dominant kernel alone (attention on pre-staged operands) -> roofline
    roof = None
    peaks = measure_mma_peaks(lib, torch)
    if mode == "fwd":
        aq.attn_forward(q, k, v, causal=causal, train=False, workspace=ws, out=o, lse_out=lse)
        torch.cuda.synchronize()
        reps = max(args.steps, 5)
        k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k0.record(st)
        for _ in range(reps):
            aq.attn_forward(q, k, v, causal=causal, train=False, workspace=ws, out=o, lse_out=lse,
                            operands_staged=True)
        k1.record(st)
        k1.synchronize()
        kms = k0.elapsed_time(k1) / reps
        achieved = alg_flops(B, H, N, d, causal, "fwd") / (kms * 1e-3) / 1e12
        roof = {"bound": "tensor", "kernel": "attn_fwd_infer_kernel<128>", "achieved": achieved,
                "peak": peaks["nvfp4"], "unit": "TFLOP/s", "frac": achieved / peaks["nvfp4"],
                "peak_source": "measured live: tcgen05 kind::mxf4nvf4 M128N256K64 issue-rate probe (aq_probe_mma_peak)",
                "kernel_ms": kms, "kernel_share_of_step": kms / ms,
                "path_ceiling_frac": achieved / (peaks["nvfp4"] * 2.0 / 3.0),
                # the binding unit is the SFU: 2 exponentials per score (7/8 on MUFU.EX2) plus one
                # reciprocal per 16-key block = 1.81 MUFU ops per score (ncu: 1.87 incl. merges),
                # at 16 MUFU/clk/SM; the algorithmic FLOPs per score are 4 d
                "sfu_ceiling_tflops": _sfu_ceiling(d, clocks.get("sm_mhz") or 1965.0, torch),
                "sfu_frac": achieved / _sfu_ceiling(d, clocks.get("sm_mhz") or 1965.0, torch),
                "traffic": _traffic_from_profiles(args.config)}
    else:
        roof = {"bound": "tensor", "kernel": "attn_fwd+attn_bwd", "achieved": value / world,
                "peak": peaks["nvfp4"], "unit": "TFLOP/s", "frac": value / world / peaks["nvfp4"],
                "peak_source": "measured live nvfp4 probe; mixed FP4/bf16 ceiling = 1.17 x bf16 peak",
                "mixed_ceiling_frac": value / world / (1.17 * peaks["bf16"]),
                "traffic": _traffic_from_profiles(args.config)}

    # ---- end to end through the public API with host buffers: pinned host
    # inputs in, host outputs back, every step; the host entry points stream
    # head chunks so H2D, kernels and D2H overlap (paper_2603_00040_b200/host.py)
    e2e = None
    hq, hk, hv = (x.cpu().pin_memory() for x in (q, k, v))
    if mode == "fwd":
        ho = torch.empty(B, H, N, d, dtype=torch.bfloat16).pin_memory()
        hl = torch.empty(B, H, N, dtype=torch.float32).pin_memory()

        def e2e_step():
            aq.attn_forward_host(hq, hk, hv, causal=causal, train=False, out=ho, lse_out=hl)
        h2d_b, d2h_b = 3 * q.numel() * 2, ho.numel() * 2 + hl.numel() * 4
    else:
        hdo = d_o.cpu().pin_memory()
        ho = torch.empty(B, H, N, d, dtype=torch.bfloat16).pin_memory()
        hg = [torch.empty_like(h).pin_memory() for h in (hq, hk, hv)]

        def e2e_step():
            aq.attn_qat_host(hq, hk, hv, hdo, causal=causal, out=ho, grads_out=hg)
        h2d_b, d2h_b = 4 * q.numel() * 2, 4 * q.numel() * 2
    for _ in range(2):
        e2e_step()
    barrier()
    if os.environ.get("AQ_E2E_DEBUG"):
        for i in range(4):
            b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            b0.record(st)
            e2e_step()
            t1 = time.perf_counter()
            b1.record(st)
            barrier()
            print(f"e2e debug step {i}: {b0.elapsed_time(b1):.2f} ms device, host enqueue {1e3*(t1-t0):.2f} ms",
                  file=sys.stderr)
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(11)]
        evs[0].record(st)
        for i in range(10):
            e2e_step()
            evs[i + 1].record(st)
        barrier()
        print("back-to-back:", [round(evs[i].elapsed_time(evs[i + 1]), 2) for i in range(10)], file=sys.stderr)
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(st)
    for _ in range(args.steps):
        e2e_step()
    a1.record(st)
    barrier()
    ems = a0.elapsed_time(a1) / args.steps
    et = torch.tensor([ems], device=dev)
    if world > 1:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e = {"value": world * flops_rank / (float(et.item()) * 1e-3) / 1e12, "unit": "TFLOP/s",
           "h2d_bytes_per_step": h2d_b, "d2h_bytes_per_step": d2h_b, "ms_per_step": float(et.item()),
           "api": "attn_forward_host (inference)" if mode == "fwd" else "attn_qat_host (fwd+bwd)",
           "pcie_gbs": (h2d_b + d2h_b) / (float(et.item()) * 1e-3) / 1e9}

    # ---- the same inference step serving from a stored FP4 KV cache (kvcache.py):
    # only Q (bf16) and the 4-bit K / V^T cross PCIe; the cache is built once,
    # outside the timed region, like a serving KV cache
    e2e_kv4 = None
    if mode == "fwd":
        hcache = aq.kv4_quantize(k, v).pin_memory()

        def kv4_step():
            aq.attn_forward_kv4_host(hq, hcache, causal=causal, out=ho, lse_out=hl)
        for _ in range(2):
            kv4_step()
        barrier()
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0.record(st)
        for _ in range(args.steps):
            kv4_step()
        b1.record(st)
        barrier()
        kms = b0.elapsed_time(b1) / args.steps
        kt_ = torch.tensor([kms], device=dev)
        if world > 1:
            dist.all_reduce(kt_, op=dist.ReduceOp.MAX)
        e2e_kv4 = {"value": world * flops_rank / (float(kt_.item()) * 1e-3) / 1e12, "unit": "TFLOP/s",
                   "ms_per_step": float(kt_.item()), "api": "attn_forward_kv4_host (NVFP4 KV cache)",
                   "h2d_bytes_per_step": q.numel() * 2 + hcache.nbytes(), "d2h_bytes_per_step": d2h_b}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ref = CpuReference(cfg)
        v_, dt_ = ref.step(7)
        cpu = {"value": v_, "unit": "TFLOP/s", "cores": ref.cores, "kind": "port", "sample": ref.sample(),
               "seconds": dt_}
        ref.close()

    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "nvfp4 (e2m1 + e4m3 block16) / fp32 accum",
            "data": "synthetic N(0,1) bf16, generated on device",
            "config": {"workload": args.config, "B": B, "H": H, "N": N, "d": d, "causal": causal,
                       "mode": "inference fwd" if mode == "fwd" else "training fwd+bwd",
                       "global_batch": world * B, "parallelism": f"dp{world} over B*H (no comms)",
                       "l2": "inputs larger than L2 (3 x %.0f MB bf16)" % (q.numel() * 2 / 1e6)},
            "tokens_per_s": tokens_s,
            "roofline": roof, "mma_peaks_tflops": peaks, "cpu_baseline": cpu, "e2e": e2e, "e2e_fp4_kv_cache": e2e_kv4,
            "clocks": clocks, "gpu_launches": launches_per_step * args.steps,
        }), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_layer_mode(args, cfg, rank, world, local):
    """Data-parallel QAT layer step (projections + NVFP4 attention fwd/bwd + NCCL
    gradient all-reduce + AdamW) with the global batch sharded over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2603_00040_b200 import train as T

    B, H, N, d, causal, _ = cfg
    if B % world:
        raise SystemExit(f"global batch {B} not divisible by {world} ranks")
    b = B // world
    D = H * d
    dev = torch.device("cuda", local)
    layer = T.AttnLayer(D, H, d, seed=0, device=dev)
    opt = torch.optim.AdamW(layer.parameters(), lr=1e-4)
    ar = T.GradAllReduce(list(layer.parameters()), world)
    gen = torch.Generator(device=dev).manual_seed(rank)
    x = torch.randn(b, N, D, generator=gen, device=dev).bfloat16()
    tgt = torch.randn(b, N, D, generator=gen, device=dev).bfloat16()
    st = torch.cuda.current_stream()

    def step(xb):
        opt.zero_grad(set_to_none=True)
        y = layer(xb, causal)
        loss = torch.mean((y.float() - tgt.float()) ** 2)
        loss.backward()
        ar.wait()
        opt.step()
        return loss

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step(x)
    barrier()
    with ClockSampler(local) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(st)
        for _ in range(args.steps):
            step(x)
        e1.record(st)
        barrier()
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    attn = alg_flops(b, H, N, d, causal, "train")
    proj = 24.0 * b * N * D * D        # 4 projection GEMMs, fwd + 2x bwd
    value = world * (attn + proj) / (ms_max * 1e-3) / 1e12
    # end to end: host batch in (pinned), loss out, every step
    hx = x.cpu().pin_memory()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    a0.record(st)
    for _ in range(args.steps):
        loss = step(hx.to(dev, non_blocking=True))
        loss.item()
    a1.record(st)
    barrier()
    et = torch.tensor([a0.elapsed_time(a1) / args.steps], device=dev)
    if world > 1:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "nvfp4 attention / bf16 projections / fp32 accum",
            "data": "synthetic N(0,1), generated on device",
            "config": {"workload": args.config, "B": B, "H": H, "N": N, "d": d, "causal": causal,
                       "mode": "QAT layer step (proj + attn fwd/bwd + NCCL grad all-reduce + AdamW)",
                       "global_batch": B, "parallelism": f"dp{world} batch-sharded"},
            "tokens_per_s": B * N / (ms_max * 1e-3),
            "flops_breakdown_per_rank": {"attention_alg": attn, "projections": proj},
            "e2e": {"value": world * (attn + proj) / (float(et.item()) * 1e-3) / 1e12, "unit": "TFLOP/s",
                    "h2d_bytes_per_step": hx.numel() * 2, "d2h_bytes_per_step": 4,
                    "ms_per_step": float(et.item())},
            "clocks": clk.summary(), "gpu_launches": 7 * args.steps,
        }), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _sfu_ceiling(d, sm_mhz, torch):
    """Forward TFLOP/s at which the MUFU (SFU) pipe saturates: 4 d algorithmic FLOPs per
    score over 1.87 MUFU ops per score (ncu, profiles/) at 16 MUFU results / clk / SM."""
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    mufu_per_s = 16.0 * sms * sm_mhz * 1e6
    return 4.0 * d * mufu_per_s / 1.87 / 1e12


def _traffic_from_profiles(config):
    """DRAM bytes per launch of the dominant kernel from the committed ncu summary (or None)."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(config, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


if __name__ == "__main__":
    main()
