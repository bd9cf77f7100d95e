"""Benchmark of the B200 NVFP4 Attn-QAT path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c4|c5-<N>] [--impl ours|reference]

Default workload = BASELINE.json configs[1]: Llama-3-8B-shaped causal
inference forward, B=4 H=32 N=8192 d=128 (FP4). One step = one call of the
public operator (``attn_forward``: NVFP4 quantizers for Q/K/V + the fused
two-pass tcgen05 attention kernel) on inputs already resident in HBM.

Multi-GPU (one process per GPU; ``--gpus N`` relaunches itself under torchrun
when WORLD_SIZE is unset): the NAMED config's B x H heads are split
contiguously over the ranks (C2: 128 heads -> 16 per GPU at N=8; C3: 40 -> 5;
every (b, h) pair is an independent unit, oracle.py:96-103), with no
communication on the attention path -> "scaling": "strong" (the total work is
fixed); value = the whole config's algorithmic FLOPs / the slowest rank's
time (barrier-bracketed, max over ranks via an NCCL all-reduce).

The 1-GPU C2 line also carries, nested under ``other_configs``, the tier's
largest single-GPU config C3 (Wan 2.1, N = 32760) and the fwd+bwd half of the
metric C4 (Llama training shape), each with its own roofline, and every entry
carries the same-box BF16 comparator (cuDNN SDPA) with the FP4 / BF16 ratio.

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
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32/f64 (numpy)",
        "data": "synthetic N(0,1)",
        "config": config_dict(args.config, cfg, world),
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


def shard_units(units, rank, world):
    """Contiguous block split of the flattened B*H head index over the ranks
    (SURVEY 8(e)): rank r owns heads [start, stop); every head is owned once."""
    base, rem = divmod(units, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


def config_dict(name, cfg, world):
    """The workload description both arms print (same keys, same values)."""
    B, H, N, d, causal, mode = cfg
    return {"workload": name, "B": B, "H": H, "N": N, "d": d, "causal": causal,
            "mode": {"fwd": "inference fwd", "train": "training fwd+bwd", "layer": "QAT layer step"}[mode],
            "global_batch": B, "parallelism": f"dp{world}: B*H heads sharded contiguously (no comms)"
            if mode != "layer" else f"dp{world} batch-sharded + NCCL grad all-reduce",
            "l2": "inputs larger than L2 (bf16 Q/K/V %.0f MB each)" % (B * H * N * d * 2 / 1e6)}


def _events(torch):
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def time_device(torch, fn, steps, warmup, st, barrier):
    for _ in range(warmup):
        fn()
    barrier()
    e0, e1 = _events(torch)
    e0.record(st)
    for _ in range(steps):
        fn()
    e1.record(st)
    barrier()
    return e0.elapsed_time(e1) / steps


def bf16_comparator(torch, q, k, v, causal, mode, d_o=None, steps=5):
    """Same-box BF16 FlashAttention on the same per-rank shape: cuDNN SDPA (the
    strongest local bf16 attention); flash_attn 2.8 as the fallback."""
    import torch.nn.functional as F
    from torch.nn.attention import SDPBackend, sdpa_kernel
    st = torch.cuda.current_stream()
    for name, be in (("cudnn_sdpa", SDPBackend.CUDNN_ATTENTION), ("flash_sdpa", SDPBackend.FLASH_ATTENTION)):
        try:
            with sdpa_kernel(be):
                if mode == "fwd":
                    def fn():
                        F.scaled_dot_product_attention(q, k, v, is_causal=causal)
                else:
                    qg, kg, vg = (t.detach().clone().requires_grad_() for t in (q, k, v))

                    def fn():
                        for t_ in (qg, kg, vg):
                            t_.grad = None
                        F.scaled_dot_product_attention(qg, kg, vg, is_causal=causal).backward(d_o)
                ms = time_device(torch, fn, steps, 3, st, torch.cuda.synchronize)
            return {"impl": name, "ms": ms}
        except Exception as e:  # noqa: BLE001 - try the next backend
            err = str(e)[:100]
    return {"impl": None, "error": err}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the nested C3 / C4 entries and the bf16 comparator")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = parse_config(args.config)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: relaunch under torchrun (the driver launches torchrun itself)
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))

    if args.impl == "reference":
        run_reference_arm(args, cfg, rank, world)
        return

    import torch
    import torch.distributed as dist

    local = int(os.environ.get("LOCAL_RANK", 0))
    if os.environ.get("AQ_BENCH_SHARE_DEVICE") == "1":
        # test hook: several ranks on one GPU (exercises the multi-rank path on a 1-GPU box)
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")        # the communicator is visible in the logs
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        backend = os.environ.get("AQ_BENCH_BACKEND", "nccl")  # test hook: gloo for ranks sharing a GPU
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    B, H, N, d, causal, mode = cfg
    if mode == "layer":
        run_layer_mode(args, cfg, rank, world, local)
        return
    rec = run_attention(args, args.config, cfg, rank, world, local, main_line=True)
    if rank == 0:
        print(json.dumps(rec), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_attention(args, name, cfg, rank, world, local, main_line=False):
    """Time one attention config: the named config's B*H heads sharded over the
    ranks, whole-job TFLOP/s over the slowest rank; roofline of the dominant
    kernel; e2e through the host-buffer API; same-box bf16 comparator."""
    import torch
    import torch.distributed as dist

    import paper_2603_00040_b200 as aq
    from paper_2603_00040_b200 import _lib

    B, H, N, d, causal, mode = cfg
    units = B * H
    h0, h1 = shard_units(units, rank, world)
    heads = h1 - h0
    dev = torch.device("cuda", local)
    gen = torch.Generator(device=dev).manual_seed(1000 + h0)
    q, k, v = (torch.randn(heads, N, d, generator=gen, device=dev).to(torch.bfloat16) for _ in range(3))
    lib = _lib.load()
    st = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        t = torch.tensor([x], device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    d_o = None
    if mode == "fwd":
        ws = torch.empty(lib.aq_attn_fwd_workspace_bytes(heads, N, N, d, 0, 0), dtype=torch.uint8, device=dev)
        o = torch.empty(heads, N, d, dtype=torch.bfloat16, device=dev)
        lse = torch.empty(heads, N, dtype=torch.float32, device=dev)

        def step():
            aq.attn_forward(q, k, v, causal=causal, train=False, workspace=ws, out=o, lse_out=lse)
        launches_per_step = 4          # quantize Q, K (rows), V (cols), fused attention
    else:
        d_o = torch.randn(heads, N, d, generator=gen, device=dev).to(torch.bfloat16)
        qg, kg, vg = (t.clone().requires_grad_() for t in (q, k, v))

        def step():
            for t_ in (qg, kg, vg):
                t_.grad = None
            out = aq.attn_qat(qg, kg, vg, causal=causal)
            out.backward(d_o)
        launches_per_step = 4 + 2      # fwd (3 quantizers + attention) + bwd pre, fused bwd (dK/dV + dQ roles)

    for _ in range(args.warmup):
        step()
    barrier()
    with ClockSampler(local) as clk:
        e0, e1 = _events(torch)
        barrier()
        e0.record(st)
        for _ in range(args.steps):
            step()
        e1.record(st)
        barrier()
    ms = e0.elapsed_time(e1) / args.steps
    clocks = clk.summary()
    ms_max = max_over_ranks(ms)
    flops_job = alg_flops(B, H, N, d, causal, mode)
    value = flops_job / (ms_max * 1e-3) / 1e12
    tokens_s = B * N / (ms_max * 1e-3)

    # ---- dominant kernel alone -> roofline
    peaks = measure_mma_peaks(lib, torch)
    flops_rank = flops_job * heads / units
    reps = max(args.steps, 5)
    if mode == "fwd":
        kms = time_device(torch, lambda: aq.attn_forward(q, k, v, causal=causal, train=False, workspace=ws, out=o,
                                                       lse_out=lse, operands_staged=True), reps, 2, st, barrier)
        achieved = flops_rank / (kms * 1e-3) / 1e12
        sfu = _sfu_ceiling(d, clocks.get("sm_mhz") or 1965.0, torch)
        roof = {"bound": "tensor", "kernel": f"attn_fwd_infer_kernel<{d}>", "achieved": achieved,
                "peak": peaks["nvfp4"], "unit": "TFLOP/s", "frac": achieved / peaks["nvfp4"],
                "peak_source": "live tcgen05 kind::mxf4nvf4 M128N256K64 issue-rate probe (aq_probe_mma_peak): "
                               "MEASURED_PEAKS.json has no FP4 entry; the nominal dense FP4 peak is 9 PF/s",
                "kernel_ms": kms, "kernel_share_of_step": kms / ms,
                "path_ceiling_frac": achieved / (peaks["nvfp4"] * 2.0 / 3.0),
                # the MUFU-bound ceiling: 2 exponentials per score (pass 1 7/8, pass 2 6/8 on
                # MUFU.EX2, the rest on the FMA pipe) plus one reciprocal per 16-key block,
                # 1.69 MUFU ops per score, 16 MUFU/clk/SM
                "sfu_ceiling_tflops": sfu, "sfu_frac": achieved / sfu,
                "traffic": _traffic_from_profiles(name)}
    else:
        o_f, lse_f, ohp_f, wsf = aq.attn_forward(q, k, v, causal=causal, train=True, keep_for_bwd=True)
        wsb = torch.empty(lib.aq_attn_bwd_workspace_bytes(heads, N, N, d), dtype=torch.uint8, device=dev)
        gq, gk, gv = (torch.empty_like(q) for _ in range(3))
        bms = time_device(torch, lambda: aq.attn_backward(q, k, v, d_o, o_f, ohp_f, lse_f, causal=causal,
                                                        fwd_workspace=wsf, workspace=wsb, grads_out=(gq, gk, gv)),
                          reps, 2, st, barrier)
        bflops = flops_rank * 2.5 / 3.5
        achieved = bflops / (bms * 1e-3) / 1e12
        # denominator: the driver's measured bf16 GEMM (MEASURED_PEAKS.json, burst: a kernel timed
        # alone), as B200_PROFILING.md prescribes; the live tcgen05 issue probe is reported beside it
        mp = _measured_peaks()
        bf16_peak = mp.get("bf16_tflops") or peaks["bf16"]
        roof = {"bound": "tensor", "kernel": f"attn_bwd_kernel<{d}> (+bwd_pre)", "achieved": achieved,
                "peak": bf16_peak, "unit": "TFLOP/s", "frac": achieved / bf16_peak,
                "peak_source": ("of measured: MEASURED_PEAKS.json bf16_tflops (cuBLAS bf16 GEMM, burst)"
                                if mp.get("bf16_tflops") else
                                "live tcgen05 kind::f16 bf16 M128N256K16 probe (MEASURED_PEAKS.json absent)")
                + "; the backward's dense contractions are bf16, its S recompute FP4",
                "frac_of_tcgen05_probe": achieved / peaks["bf16"],
                "kernel_ms": bms, "kernel_share_of_step": bms / ms,
                "step_frac_of_fp4_peak": value / world / peaks["nvfp4"],
                "step_frac_of_mixed_ceiling": value / world / (1.17 * peaks["bf16"]),
                "traffic": _traffic_from_profiles(name)}
        # the training forward (K11, split-pass) beside it: FP4 S / PV plus the f16 O' MMA
        fms = time_device(torch, lambda: aq.attn_forward(q, k, v, causal=causal, train=True, workspace=wsf,
                                                       operands_staged=True, keep_for_bwd=True, out=o_f,
                                                       lse_out=lse_f, o_hp_out=ohp_f),
                          reps, 2, st, barrier)
        ffl = flops_rank / 3.5
        roof["forward"] = {"kernel": f"attn_fwd_qat_kernel<{d}>", "kernel_ms": fms,
                           "achieved": ffl / (fms * 1e-3) / 1e12, "unit": "TFLOP/s",
                           "frac_of_fp4_peak": ffl / (fms * 1e-3) / 1e12 / peaks["nvfp4"],
                           "kernel_share_of_step": fms / ms,
                           "traffic": _traffic_from_profiles("train_fwd_" + name)}

    rec = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "nvfp4 (e2m1 + e4m3 block16) / fp32 accum",
           "data": "synthetic N(0,1) bf16, generated on device",
           "config": config_dict(name, cfg, world), "tokens_per_s": tokens_s, "roofline": roof,
           "mma_peaks_tflops": peaks, "heads_per_rank": heads}
    if not args.no_extras:
        cmp_ = bf16_comparator(torch, q.unsqueeze(0), k.unsqueeze(0), v.unsqueeze(0), causal, mode,
                               d_o.unsqueeze(0) if d_o is not None else None)
        if cmp_.get("ms"):
            cms = max_over_ranks(cmp_["ms"])
            cmp_.update({"ms": cms, "tflops": flops_job / (cms * 1e-3) / 1e12, "ratio": cms / ms_max,
                         "target_ratio": 1.5 if mode == "fwd" else None})
        rec["bf16_comparator"] = cmp_
    if not main_line:
        rec["clocks"] = clocks
        return rec

    # ---- end to end through the public API with host buffers: pinned host
    # inputs in, host outputs back, every step; the host entry points stream
    # head chunks so H2D, kernels and D2H overlap (paper_2603_00040_b200/host.py)
    hq, hk, hv = (x.cpu().pin_memory() for x in (q, k, v))
    if mode == "fwd":
        ho = torch.empty(heads, N, d, dtype=torch.bfloat16).pin_memory()
        hl = torch.empty(heads, N, dtype=torch.float32).pin_memory()

        def e2e_step():
            aq.attn_forward_host(hq, hk, hv, causal=causal, train=False, out=ho, lse_out=hl)
        h2d_b, d2h_b = 3 * q.numel() * 2, ho.numel() * 2 + hl.numel() * 4
    else:
        hdo = d_o.cpu().pin_memory()
        ho = torch.empty(heads, N, d, dtype=torch.bfloat16).pin_memory()
        hg = [torch.empty_like(h).pin_memory() for h in (hq, hk, hv)]

        def e2e_step():
            aq.attn_qat_host(hq, hk, hv, hdo, causal=causal, out=ho, grads_out=hg)
        h2d_b, d2h_b = 4 * q.numel() * 2, 4 * q.numel() * 2
    ems = max_over_ranks(time_device(torch, e2e_step, args.steps, 2, st, barrier))
    rec["e2e"] = {"value": flops_job / (ems * 1e-3) / 1e12, "unit": "TFLOP/s",
                  "h2d_bytes_per_step": h2d_b * world, "d2h_bytes_per_step": d2h_b * world, "ms_per_step": ems,
                  "api": "attn_forward_host (inference)" if mode == "fwd" else "attn_qat_host (fwd+bwd)",
                  "pcie_gbs_per_rank": (h2d_b + d2h_b) / (ems * 1e-3) / 1e9}

    # ---- the same inference step serving from a stored FP4 KV cache (kvcache.py):
    # only Q (bf16) and the 4-bit K / V^T cross PCIe; the cache is built once,
    # outside the timed region, like a serving KV cache
    if mode == "fwd":
        hcache = aq.kv4_quantize(k, v).pin_memory()
        kms_ = max_over_ranks(time_device(
            torch, lambda: aq.attn_forward_kv4_host(hq, hcache, causal=causal, out=ho, lse_out=hl),
            args.steps, 2, st, barrier))
        rec["e2e_fp4_kv_cache"] = {"value": flops_job / (kms_ * 1e-3) / 1e12, "unit": "TFLOP/s",
                                   "ms_per_step": kms_, "api": "attn_forward_kv4_host (NVFP4 KV cache)",
                                   "h2d_bytes_per_step": (q.numel() * 2 + hcache.nbytes()) * world,
                                   "d2h_bytes_per_step": d2h_b * world}
    del hq, hk, hv, ho

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ref = CpuReference(cfg)
        v_, dt_ = ref.step(7)
        cpu = {"value": v_, "unit": "TFLOP/s", "cores": ref.cores, "kind": "port", "sample": ref.sample(),
               "seconds": dt_}
        ref.close()
    rec["cpu_baseline"] = cpu

    # ---- the other BASELINE configs, nested (1 GPU: the tier's largest single-GPU
    # config C3 and the fwd+bwd half of the metric, C4), each with its own roofline
    if world == 1 and not args.no_extras and name == "c2":
        del q, k, v, o, lse, ws
        torch.cuda.empty_cache()
        extra = {}
        for xname in ("c3", "c4"):
            r = run_attention(args, xname, parse_config(xname), rank, world, local)
            extra[xname] = {kk: r[kk] for kk in ("value", "unit", "ms_per_step", "tokens_per_s", "config",
                                                 "roofline", "bf16_comparator", "clocks")}
            torch.cuda.empty_cache()
        rec["other_configs"] = extra
    rec["clocks"] = clocks
    rec["gpu_launches"] = launches_per_step * args.steps
    return rec


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
            "config": config_dict(args.config, cfg, world),
            "tokens_per_s": B * N / (ms_max * 1e-3),
            "flops_breakdown_per_rank": {"attention_alg": attn, "projections": proj},
            "e2e": {"value": world * (attn + proj) / (float(et.item()) * 1e-3) / 1e12, "unit": "TFLOP/s",
                    "h2d_bytes_per_step": hx.numel() * 2, "d2h_bytes_per_step": 4,
                    "ms_per_step": float(et.item())},
            "clocks": clk.summary(), "gpu_launches": 7 * args.steps,
        }), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _measured_peaks():
    """The driver-written MEASURED_PEAKS.json (roofline denominators), or {}."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return {}


def _sfu_ceiling(d, sm_mhz, torch):
    """Forward TFLOP/s at which the MUFU (SFU) pipe saturates: 4 d algorithmic FLOPs per
    score over 1.69 MUFU ops per score (7/8 + 6/8 exponentials + 1/16 reciprocal; the pipe
    rate is measured in profiles/r02_pipe_probe.txt) at 16 MUFU results / clk / SM."""
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    mufu_per_s = 16.0 * sms * sm_mhz * 1e6
    return 4.0 * d * mufu_per_s / (0.875 + 0.75 + 0.0625) / 1e12


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
