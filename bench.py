"""Benchmark: TR-ALS NE sweeps on B200 (driver contract: one JSON line from rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--variant ne]
    python bench.py --impl reference ...      # the reference's CPU path (oracle port) on the host cores

A step is one full TR-ALS sweep (all N mode updates: Gram chain, right-hand
side, Cholesky solve, Gram refresh) plus the per-sweep relative error, on the
BASELINE config (default c5: 160^4, rank 20, fp64).  X is 5.24 GB, far larger
than the 126 MB L2, so no explicit flush is needed between steps.  With
torchrun (N > 1) X is sharded along mode 0 (BASELINE's "mode 1", 1-based) and
the partial right-hand sides are all-reduced over NCCL; total work is fixed
("strong" scaling).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TR-ALS sweeps/s & contraction TFLOP/s (% of fp64 roofline), 1-8 B200"
# BASELINE.json configs: order, dim, rank_true, noise, seed_data, rank_fit, seed_init, sweeps
CONFIGS = {
    "c1": (3, 100, 5, 1e-3, 0, 5, 1, 10),
    "c2": (4, 64, 8, 1e-2, 2, 8, 3, 20),
    "c3": (3, 500, 10, 1e-3, 4, 10, 5, 10),
    "c4": (5, 40, 6, 1e-2, 6, 8, 7, 15),
    "c5": (4, 160, 20, 1e-3, 8, 20, 9, 10),
}
FP64_PEAK_TFLOPS = 37.1      # measured DMMA.8x8x4 ceiling on this pool's B200 (profiles/r01_fp64_pipes.md)
# fp32 variant: 13 int8 MMAs per fp32-equivalent multiply-add; int8 dense ~2x the measured bf16 burst
INT8_FP32_EQ_TFLOPS = 2 * 1715.0 / 13
PEAK_SOURCE = "profiles/r01_fp64_pipes.md: mma.sync m8n8k4 f64 microbenchmark, 148 SMs"
# fp64 "ozaki" environment products: 28 int8 digit-pair MMAs per fp64 multiply-add (7 balanced
# radix-254 digits per operand, pair levels s + t <= 6)
OZ64_PAIRS = 28
# int8 tcgen05 ceiling on this pool's B200: tools/micro/i8_peak.cu (M128 N256 K32 MMAs back to back,
# 148 SMs), profiles/r01_i8_peak.jsonl: 4374.8 TOPS burst (one launch), 4260.0 sustained (launches
# back to back for 3 s).  The environment GEMM runs inside a long step (sweeps back to back), so the
# sustained figure is its roofline denominator.
INT8_PEAK_TOPS = 4260.0
INT8_PEAK_BURST_TOPS = 4374.8


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for name, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows),
                "power_w_max": max((float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()),
                                   default=None)}


def dist_setup(gpus):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def flops_per_sweep(dims, ranks):
    tot = float(np.prod(dims))
    N = len(dims)
    return sum(2.0 * tot * ranks[n] * ranks[(n + 1) % N] for n in range(N))


def roofline_sweep_time(dims, ranks, peak_tf, bw_gbs, world, elem_bytes=8):
    tot = float(np.prod(dims)) / world
    N = len(dims)
    t = 0.0
    for n in range(N):
        f = 2.0 * tot * ranks[n] * ranks[(n + 1) % N]
        t += max(f / (peak_tf * 1e12), tot * elem_bytes / (bw_gbs * 1e9))
    return t


# ---------------------------------------------------------------------------
# CPU side: the reference path (oracle port) on the host cores
# ---------------------------------------------------------------------------
def cpu_mode_sample(x, cores, n, frac):
    """Time one NE block update (solvers.py:371-384) on a slab of X along mode (n+1)%N.

    The subchain, the MTTSP and the copies all scale linearly with the slab;
    returns (seconds for the slab, fraction of the full mode update it is)."""
    from oracle import tenring_oracle as O
    N = x.ndim
    m = (n + 1) % N
    k = max(1, int(round(x.shape[m] * frac)))
    idx = [slice(None)] * N
    idx[m] = slice(0, k)
    xs = np.ascontiguousarray(x[tuple(idx)])
    cs = [c.copy() for c in cores]
    cs[m] = np.ascontiguousarray(cs[m][:, :k, :])
    grams = [O.bond_gram(g) for g in cs]
    xu = O.unfold_cyclic(xs, n)  # built before the timed sweep in the reference too (solvers.py:362)
    t0 = time.perf_counter()
    s = O.chain_grams(grams[j] for j in O.gram_order(n, N))
    a = O.unfold_cyclic(O.chain_without(cs, n), 1)
    mm = xu @ a
    z, _ = O.solve_spd_right(s, mm)
    g = O.fold_classical(z, 1, (cs[n].shape[0], cs[n].shape[1], cs[n].shape[2]))
    O.bond_gram(g)
    dt = time.perf_counter() - t0
    return dt, k / x.shape[m]


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        return max((int(i.get("num_threads", 1)) for i in threadpool_info()), default=os.cpu_count())
    except Exception:
        return os.cpu_count()


def host_inputs(cfg_name):
    """X (host numpy) and init cores for the CPU leg, from the same GPU generator as our arm."""
    import torch
    from paper_2210_11362_b200.host import make_rng, random_cores
    from paper_2210_11362_b200.synthetic import make_dataset_device
    order, dim, rt, noise, sd, rf, si, sweeps = CONFIGS[cfg_name]
    xd, _ = make_dataset_device(order, dim, rt, noise, sd)
    x = xd.cpu().numpy()
    del xd
    torch.cuda.empty_cache()
    cores = random_cores(x.shape, [rf] * order, make_rng(si))
    return x, cores


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import torch
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    order, dim, rt, noise, sd, rf, si, sweeps = CONFIGS[args.config]
    x, cores = host_inputs(args.config)
    frac = args.ref_frac
    times = []
    for step in range(args.warmup + args.steps):
        n = step % order
        dt, f = cpu_mode_sample(x, cores, n, frac)
        if step >= args.warmup:
            times.append(dt / f)  # full mode-update time
    t_mode = float(np.mean(times))
    t_sweep = order * t_mode
    value = 1.0 / t_sweep
    threads = cpu_threads()
    sample = (f"one NE block update per step (mode = step mod {order}; Gram chain + subchain + MTTSP + "
              f"Cholesky solve + Gram refresh, solvers.py:371-384) on a {frac:.3g} slab of X along the next mode, "
              f"scaled to a full sweep (x{order}/{frac:.3g}); oracle port of tenring 0.1.0, numpy/OpenBLAS")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "sweeps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_sweep * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config} NE sweep", "dims": [dim] * order, "ranks": [rf] * order,
                   "variant": "ne", "l2": "X larger than L2"},
        "cpu_baseline": {"value": value, "unit": "sweeps/s", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "sweeps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "contraction_tflops": flops_per_sweep([dim] * order, [rf] * order) / t_sweep / 1e12,
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as tdist

    world, rank, local = dist_setup(args.gpus)
    from paper_2210_11362_b200 import _lib as L
    from paper_2210_11362_b200.engine import SweepEngine
    from paper_2210_11362_b200.host import make_rng, random_cores
    from paper_2210_11362_b200.solvers import AlsConfig, _slab, decompose
    from paper_2210_11362_b200.synthetic import make_dataset_device

    order, dim, rt, noise, sd, rf, si, sweeps = CONFIGS[args.config]
    dims, ranks = [dim] * order, [rf] * order
    dev = torch.device("cuda", torch.cuda.current_device())
    x_full, _ = make_dataset_device(order, dim, rt, noise, sd, device=dev)
    fp32 = args.dtype == "float32"
    if fp32:
        x_full = x_full.float()
    shard = 0
    if world > 1:
        lo, hi = _slab(dim, world, rank)
        x_local = x_full[lo:hi].contiguous()
    else:
        lo, hi = 0, dim
        x_local = x_full
    cores0 = random_cores(dims, ranks, make_rng(si))
    eng = SweepEngine(x_local, dims, ranks, args.variant, shard_mode=shard if world > 1 else None, lo=lo, hi=hi,
                      world_size=world, fp64_gemm=args.fp64_gemm)
    oz64 = eng.oz64
    eng_gemm = eng.fp64_gemm
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record(eng.stream)
    eng.prepare_x()
    p1.record(eng.stream)
    torch.cuda.synchronize()
    prep_ms = p0.elapsed_time(p1)
    eng.compute_xnorm2()
    eng.set_cores(cores0)
    errs = torch.zeros((args.warmup + args.steps, 3), dtype=torch.float64, device=dev)
    stream = eng.stream
    use_graph = (world == 1 and not args.eager)
    if use_graph:
        eng.capture(with_error=True)
    for k in range(args.warmup):
        if use_graph:
            eng.replay()
        else:
            eng.run_sweep()
            eng.error_step(errs[k])
    torch.cuda.synchronize()
    if world > 1:
        tdist.barrier()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    l0 = L.lib().trals_launch_count()
    env_events = []
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        tdist.barrier()
    e0.record(stream)
    for k in range(args.steps):
        if use_graph:
            eng.replay()
        else:
            eng.run_sweep(env_events=env_events)
            eng.error_step(errs[args.warmup + k])
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        tdist.barrier()
    launches = L.lib().trals_launch_count() - l0
    if use_graph:
        # graph replays launch no host-side calls: count the kernels of one captured sweep
        c0 = L.lib().trals_launch_count()
        eng.run_sweep(env_events=env_events)
        eng.error_step(errs[-1])
        torch.cuda.synchronize()
        launches = (L.lib().trals_launch_count() - c0) * args.steps
        for _ in range(4):
            eng.run_sweep(env_events=env_events)
        torch.cuda.synchronize()
        errs[-1].copy_(eng.err_cur)
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1) / args.steps
    env_ms = [a.elapsed_time(b) for a, b in env_events]
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    ms_max = float(t.item())
    final_err = float(errs[args.warmup + args.steps - 1, 0].item()) if not use_graph else float(eng.err_cur[0].item())

    # dominant kernel: the X-streaming environment GEMM (one per phase)
    oz64 = (not fp32) and eng_gemm == "ozaki"
    env_flops = eng.env_flops()
    per_launch = [env_flops[i % len(env_flops)] / (env_ms[i] * 1e-3) / 1e12 for i in range(len(env_ms))]
    env_avg_ms = float(np.mean(env_ms))
    env_tf = float(np.mean(per_launch))
    env_share = env_avg_ms * len(env_flops) / ms
    traffic = None
    tag = "_fp32" if fp32 else ("_oz64" if oz64 else "")
    tpath = os.path.join(ROOT, "profiles", f"{args.config}{tag}_env_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    peaks = load_peaks()
    bw = float(peaks.get("hbm_gbs", 6458.1))
    F = flops_per_sweep(dims, ranks)
    ebytes = 4 if fp32 else 8
    # P = the peak of the pipe actually used (fp64 on int8: the int8 rate / 28 pairs)
    peak_tf = (INT8_FP32_EQ_TFLOPS if fp32 else
               INT8_PEAK_TOPS / OZ64_PAIRS if oz64 else FP64_PEAK_TFLOPS)
    t_roof = roofline_sweep_time(dims, ranks, peak_tf, bw, world, ebytes)
    t_roof_dmma = roofline_sweep_time(dims, ranks, FP64_PEAK_TFLOPS, bw, world, ebytes)
    sweep_s = ms_max * 1e-3
    value = 1.0 / sweep_s

    # e2e through the public API: host (pinned) X -> decompose(max_iters=BASELINE sweeps) -> host cores
    e2e = None
    if not args.no_e2e:
        xh = torch.empty(x_full.shape, dtype=x_full.dtype, pin_memory=True)
        xh.copy_(x_full)
        del x_full, x_local
        eng = None
        torch.cuda.empty_cache()
        cfg = AlsConfig(ranks=tuple(ranks), max_iters=sweeps, seed=si, error_mode="cheap", timing_buckets=False,
                        dtype=args.dtype, fp64_gemm=args.fp64_gemm)
        decompose(xh, args.variant, cfg)  # warm-up call (allocator, plan)
        torch.cuda.synchronize()
        reps = []
        for _ in range(args.e2e_reps):
            if world > 1:
                tdist.barrier()
            t0 = time.perf_counter()
            cores, rep = decompose(xh, args.variant, cfg)
            reps.append(time.perf_counter() - t0)
        tt = torch.tensor([float(np.mean(reps))], dtype=torch.float64, device=dev)
        if world > 1:
            tdist.all_reduce(tt, op=tdist.ReduceOp.MAX)
        t_call = float(tt.item())
        core_bytes = sum(int(np.prod(c.shape)) * 8 for c in cores)
        e2e = {"value": sweeps / t_call, "unit": "sweeps/s",
               "h2d_bytes_per_step": int(np.prod(dims)) * ebytes + core_bytes,
               "d2h_bytes_per_step": core_bytes + 8 * sweeps + 16,
               "step": f"one decompose(x_host_pinned, '{args.variant}', AlsConfig(max_iters={sweeps}, "
                       f"dtype='{args.dtype}', fp64_gemm='{args.fp64_gemm}')) call (includes X's H2D copy and, "
                       f"for the tensor-core paths, its digit slicing)",
               "seconds_per_call": t_call, "final_error": float(rep.errors[-1])}
        del xh

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        x, cores = host_inputs(args.config)
        dt, f = cpu_mode_sample(x, cores, 0, args.cpu_frac)
        t_sweep_cpu = order * dt / f
        cpu = {"value": 1.0 / t_sweep_cpu, "unit": "sweeps/s", "cores": cpu_threads(), "kind": "port",
               "sample": (f"one NE block update of mode 0 (solvers.py:371-384) on a {f:.3g} slab of X along mode 1 "
                          f"({dt:.1f} s), scaled x{order}/{f:.3g} to a full sweep; oracle port of tenring 0.1.0 on "
                          f"numpy/OpenBLAS")}
        del x

    if fp32:
        # fp32 variant: the int8-tensor-core digit-sliced GEMM streams X (4 B/elem) once per launch
        xbytes = float(np.prod(dims)) / world * 4
        gbs = xbytes / (env_avg_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": gbs, "peak": bw, "unit": "GB/s", "frac": gbs / bw, "traffic": traffic,
                "kernel": "oz8_kernel (int8 tcgen05 digit-sliced X x half-chain environment product)",
                "bytes_per_launch": xbytes, "avg_launch_ms": env_avg_ms, "share_of_step": env_share,
                "flops_per_launch": env_flops, "tflops_fp32_equiv": env_tf,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)"}
    elif oz64:
        # fp64 on the int8 tensor cores: the algorithmic work of one launch is the 28 digit-pair
        # products over the real (unpadded) M x N x K; peak = int8 dense = 2x the measured bf16 burst
        i8_peak = INT8_PEAK_TOPS
        i8_tops = env_tf * OZ64_PAIRS
        roof = {"bound": "tensor", "achieved": i8_tops, "peak": i8_peak, "unit": "TFLOP/s",
                "frac": i8_tops / i8_peak, "traffic": traffic,
                "kernel": "oz8_kernel<64, OzF64> (fp64 X x half-chain environment product on the int8 tcgen05 "
                          "tensor cores: 7 balanced radix-254 digits per operand, 28 exact int32 digit-pair products)",
                "ops": "int8 tensor ops = 28 x 2 M N K per launch", "flops_per_launch": env_flops,
                "fp64_equiv_tflops": env_tf, "fp64_equiv_frac_of_dmma_peak": env_tf / FP64_PEAK_TFLOPS,
                "avg_launch_ms": env_avg_ms, "share_of_step": env_share,
                "frac_of_burst_peak": i8_tops / INT8_PEAK_BURST_TOPS,
                "peak_source": "profiles/r01_i8_peak.jsonl: tcgen05 kind::i8 M128 N256 K32 microbenchmark, 148 SMs, "
                               "sustained (launches back to back for 3 s; burst 4374.8)"}
    else:
        roof = {"bound": "tensor", "achieved": env_tf, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": env_tf / FP64_PEAK_TFLOPS, "traffic": traffic,
                "kernel": "dmma_tma_kernel (X x half-chain environment product)",
                "flops_per_launch": env_flops, "avg_launch_ms": env_avg_ms, "share_of_step": env_share,
                "peak_source": PEAK_SOURCE}
    line = {
        "metric": METRIC, "value": value, "unit": "sweeps/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32 (X) / f64" if fp32 else "f64", "data": "synthetic (BASELINE recipe; cores from the reference Philox "
                                                     "stream, X reconstructed on the GPU, device noise)",
        "config": {"workload": f"{args.config} {args.variant.upper()} sweep" + (" (fp32 variant)" if fp32 else ""),
                   "dims": dims, "ranks": ranks, "dtype": args.dtype,
                   "variant": args.variant, "parallelism": f"shard mode 0 x{world}" if world > 1 else "single",
                   "l2": "X (%.2f GB) larger than the 126 MB L2, no flush needed" % (np.prod(dims) * ebytes / 1e9),
                   "step": "one full sweep + per-sweep relative error",
                   "fp64_gemm": None if fp32 else eng_gemm,
                   "x_digits_ms": prep_ms if (fp32 or oz64) else None,
                   "launch": "CUDA graph replay" if use_graph else "eager stream launches"},
        "contraction_tflops": F / sweep_s / 1e12,
        "contraction_roofline_frac": t_roof / sweep_s,
        "roofline_sweep_ms": t_roof * 1e3,
        "roofline_pipe_tflops": peak_tf,
        "contraction_roofline_frac_vs_dmma_peak": t_roof_dmma / sweep_s,
        "x_passes_per_sweep": eng.stats.x_passes_per_sweep if eng is not None else 2,
        "roofline": roof,
        "gpu_launches": int(launches),
        "clocks": clocks,
        "final_error": final_err,
    }
    if e2e is not None:
        line["e2e"] = e2e
    if cpu is not None:
        line["cpu_baseline"] = cpu
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        tdist.barrier()
        tdist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c5")
    ap.add_argument("--variant", choices=["ne", "qr", "qrne"], default="ne")
    ap.add_argument("--dtype", choices=["float64", "float32"], default="float64",
                    help="float32 = the fp32 variant (BASELINE config 4): int8 tensor-core environment products")
    ap.add_argument("--fp64-gemm", choices=["auto", "ozaki", "dmma"], default="auto",
                    help="fp64 environment products: int8 tensor-core digit slicing, the DMMA pipe, or "
                         "auto (ozaki for products >= 4 GFLOP: c3-c5)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--eager", action="store_true", help="no CUDA graph for the small configs")
    ap.add_argument("--e2e-reps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-frac", type=float, default=0.5, help="slab fraction for the cpu_baseline sample")
    ap.add_argument("--ref-frac", type=float, default=0.125, help="slab fraction per --impl reference step")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
