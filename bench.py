"""Benchmark: TR-ALS sweeps on B200 (driver contract: one JSON line from rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--variant ne]
    python bench.py --impl reference ...      # the reference's CPU path (oracle port) on the host cores

Our arm: a step is one full TR-ALS sweep (all N mode updates: Gram chain,
right-hand side, solve, Gram/QR refresh) plus the per-sweep relative error, on
the BASELINE config (default c5: 160^4, rank 20, fp64).  X is 5.24 GB, far
larger than the 126 MB L2, so no explicit flush is needed between steps.
`--gpus N` runs one process per GPU (re-launching itself under
torch.distributed.run when WORLD_SIZE is not set): X is sharded along mode 0
(BASELINE's "mode 1", 1-based) and the partial right-hand sides are
all-reduced over NCCL; total work is fixed ("strong" scaling).

Reference arm: the reference's own CPU path (the oracle port of tenring's
solvers, faithful operation order; the pure-Python reference cannot travel to
the GPU box) on all host cores; a step is one full-size block update, N
consecutive steps are one sweep.  It imports neither torch nor this package.
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

# the CPU legs use every host core the process may run on (scipy-openblas caps at 64 threads)
os.environ.setdefault("OPENBLAS_NUM_THREADS", str(min(64, len(os.sched_getaffinity(0)))))

import numpy as np  # noqa: E402

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
# CPU side: the reference's path (the oracle port, faithful operation order) on the host cores
# ---------------------------------------------------------------------------
def cpu_info():
    """Cores the CPU legs use: affinity, physical cores, the BLAS pool actually running."""
    info = {"affinity": len(os.sched_getaffinity(0)), "logical": os.cpu_count(),
            "openblas_num_threads_env": os.environ.get("OPENBLAS_NUM_THREADS")}
    try:
        import psutil
        info["physical"] = psutil.cpu_count(logical=False)
    except Exception:
        info["physical"] = None
    try:
        from threadpoolctl import threadpool_info
        blas = [i for i in threadpool_info() if i.get("user_api") == "blas"]
        info["blas_threads"] = max((int(i.get("num_threads", 1)) for i in blas), default=None)
        info["blas"] = ",".join(sorted({f"{i.get('internal_api')} {i.get('version')} {i.get('architecture')}"
                                        for i in blas}))
    except Exception:
        info["blas_threads"] = None
    try:
        with open("/proc/cpuinfo") as f:
            info["model"] = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), None)
    except Exception:
        info["model"] = None
    try:
        with open("/proc/meminfo") as f:
            info["mem_total_gb"] = round(int(next(ln for ln in f if ln.startswith("MemTotal")).split()[1]) / 2**20, 1)
    except Exception:
        pass
    return info


def cpu_block_steps(x, variant, ranks, init, n_steps, n_warm=0):
    """Run n_warm + n_steps consecutive full-size block updates of the reference's sweep (mode = k mod N,
    solvers.py:370-384 / :420-443 / :473-493) with the oracle's faithful restatement; returns the
    per-step seconds of the last n_steps and the set-up seconds (unfoldings / initial Grams)."""
    from oracle import tenring_oracle as O
    st = O.BlockStepper(x, variant, ranks, init)
    t0 = time.perf_counter()
    st.prepare()
    prep = time.perf_counter() - t0
    times = []
    for k in range(n_warm + n_steps):
        t0 = time.perf_counter()
        st.step(k % x.ndim)
        dt = time.perf_counter() - t0
        if k >= n_warm:
            times.append(dt)
    return times, prep


def run_reference(args):
    """--impl reference: the reference's CPU solver path (oracle port; the pure-Python reference
    cannot travel to the GPU box) on the host cores.  Imports neither torch nor this package."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    from oracle import lean
    from oracle import tenring_oracle as O
    order, dim, rt, noise, sd, rf, si, sweeps = CONFIGS[args.config]
    dims, ranks = [dim] * order, [rf] * order
    t0 = time.perf_counter()
    x, _ = lean.synth(O.Recipe(order=order, dim=dim, rank=rt, noise=noise, seed=sd))
    synth_s = time.perf_counter() - t0
    init = O.gaussian_ring(dims, ranks, O.philox(si))
    times, prep = cpu_block_steps(x, args.variant, ranks, init, args.steps, args.warmup)
    t_step = float(np.mean(times))
    value = 1.0 / (order * t_step)
    ci = cpu_info()
    threads = ci.get("blas_threads") or ci["affinity"]
    sample = (f"{args.steps} consecutive full-size {args.variant.upper()} block updates (mode = step mod {order}) "
              f"after {args.warmup} warm-up updates: {args.steps / order:g} complete sweeps of the reference's "
              f"per-mode loop (materialised subchain, cyclic-unfold copies, numpy/OpenBLAS dgemm, scipy Cholesky), "
              f"oracle port of tenring 0.1.0 on X from the reference recipe (seed {sd}, host Philox noise)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "sweeps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference recipe, host)",
        "config": {"workload": f"{args.config} {args.variant.upper()} sweep", "dims": dims, "ranks": ranks,
                   "variant": args.variant, "l2": "CPU run",
                   "step": f"one full-size block update of the sweep; {order} consecutive steps = one sweep; "
                           f"value = 1 / ({order} x mean step time)"},
        "cpu_baseline": {"value": value, "unit": "sweeps/s", "cores": threads, "kind": "port", "sample": sample,
                         "cpu": ci},
        "e2e": {"value": value, "unit": "sweeps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "contraction_tflops": flops_per_sweep(dims, ranks) * value / 1e12,
        "setup_seconds": {"synth": synth_s, "unfold_and_grams": prep},
        "step_seconds": times,
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def self_launch(args):
    """--gpus N without torchrun: re-run this script under torch.distributed.run with N ranks
    (one process per GPU, rendezvous on 127.0.0.1); rank 0's JSON line passes through."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def capture_checked(eng, cores0, tdist, world):
    """Capture the sweep (+ error) as a CUDA graph.  For a sharded run the graph holds the NCCL
    all-reduces too; it is kept only if one replay reproduces an eager sweep bit for bit on every
    rank (otherwise the run stays eager and says so)."""
    import torch
    try:
        eng.capture(with_error=True)
    except Exception as e:  # pragma: no cover - hardware path
        if world > 1:
            return False, f"capture failed: {type(e).__name__}: {e}"[:200]
        raise
    if world == 1:
        return True, "CUDA graph replay"
    eng.set_cores(cores0)
    eng.run_sweep()
    torch.cuda.synchronize()
    ref = [g.clone() for g in eng.Gc]
    eng.set_cores(cores0)
    eng.replay()
    torch.cuda.synchronize()
    bad = torch.tensor([float(sum(int(not torch.equal(a, b)) for a, b in zip(ref, eng.Gc)))], device=ref[0].device,
                       dtype=torch.float64)
    tdist.all_reduce(bad)
    eng.set_cores(cores0)
    if bad.item() != 0:
        eng.graph = None
        return False, "graph replay differed from the eager sweep; eager launches"
    return True, "CUDA graph replay (NCCL all-reduces captured)"


def run_ours(args):
    import torch
    import torch.distributed as tdist

    world, rank, local = dist_setup(args.gpus)
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    from paper_2210_11362_b200 import _lib as L
    from paper_2210_11362_b200.engine import OZ64_MAX_RHO, SweepEngine
    from paper_2210_11362_b200.host import make_rng, random_cores
    from paper_2210_11362_b200.solvers import AlsConfig, _slab, decompose
    from paper_2210_11362_b200.synthetic import make_dataset_device

    order, dim, rt, noise, sd, rf, si, sweeps = CONFIGS[args.config]
    dims, ranks = [dim] * order, [rf] * order
    dev = torch.device("cuda", torch.cuda.current_device())
    # the reference recipe: true cores from the reference Philox stream, X reconstructed on the GPU,
    # the reference's host noise stream (numpy Philox) -- the same X the CPU legs time
    x_full, _ = make_dataset_device(order, dim, rt, noise, sd, device=dev, noise_source="host")
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
    # the accuracy guard of fp64_gemm="auto" (include/trals.h), as decompose() applies it
    rho = eng.x_dynamic_range()
    if args.fp64_gemm == "auto" and eng.oz64 and rho > OZ64_MAX_RHO:
        eng = SweepEngine(x_local, dims, ranks, args.variant, shard_mode=shard if world > 1 else None, lo=lo,
                          hi=hi, world_size=world, fp64_gemm="dmma")
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
    use_graph, launch_note = False, "eager stream launches"
    if not args.eager:
        use_graph, launch_note = capture_checked(eng, cores0, tdist, world)
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
    aux_events = {}
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
            eng.run_sweep(env_events=env_events, aux_events=aux_events)
            eng.error_step(errs[args.warmup + k])
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        tdist.barrier()
    clocks = sampler.stop()
    launches = L.lib().trals_launch_count() - l0
    if use_graph:
        # graph replays make no host-side library calls: count the kernels of one sweep + error
        # (eagerly, outside the timed region) and time the environment launches there
        c0 = L.lib().trals_launch_count()
        eng.run_sweep()
        eng.error_step(errs[-1])
        torch.cuda.synchronize()
        launches = (L.lib().trals_launch_count() - c0) * args.steps
        for _ in range(4):
            eng.run_sweep(env_events=env_events, aux_events=aux_events)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    env_ms = [a.elapsed_time(b) for a, b in env_events]
    aux_ms = {k: float(np.mean([a.elapsed_time(b) for a, b in v])) for k, v in aux_events.items()}
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    ms_max = float(t.item())
    final_err = float(eng.err_cur[0].item()) if use_graph else float(errs[args.warmup + args.steps - 1, 0].item())

    # dominant kernel: the X-streaming environment GEMM (one per phase)
    oz64 = (not fp32) and eng_gemm in ("ozaki", "crt")
    # form of the int8 engine behind the environment products: CRT (one int8 GEMM per modulus) for
    # long contractions, else the 28 digit-pair products
    crt = oz64 and eng.env_kinds == {"crt"}
    i8_products = L.lib().trals_crt_moduli() if crt else OZ64_PAIRS
    i8_forms = sorted(eng.env_kinds) if oz64 else None
    env_flops = eng.env_flops()
    per_launch = [env_flops[i % len(env_flops)] / (env_ms[i] * 1e-3) / 1e12 for i in range(len(env_ms))]
    env_avg_ms = float(np.mean(env_ms))
    env_tf = float(np.mean(per_launch))
    env_share = env_avg_ms * len(env_flops) / ms
    traffic = None
    tag = "_fp32" if fp32 else ("_crt" if crt else "_oz64" if oz64 else "")
    tpath = os.path.join(ROOT, "profiles", f"{args.config}{tag}_env_traffic.json")
    if os.path.exists(tpath) and world == 1:
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
               INT8_PEAK_TOPS / i8_products if oz64 else FP64_PEAK_TFLOPS)
    t_roof = roofline_sweep_time(dims, ranks, peak_tf, bw, world, ebytes)
    t_roof_dmma = roofline_sweep_time(dims, ranks, FP64_PEAK_TFLOPS, bw, world, ebytes)
    sweep_s = ms_max * 1e-3
    value = 1.0 / sweep_s

    x_host = None
    if not (args.no_e2e and args.no_cpu_baseline):
        x_host = torch.empty(x_full.shape, dtype=x_full.dtype, pin_memory=True)
        x_host.copy_(x_full)
    del x_full, x_local
    eng = None
    torch.cuda.empty_cache()

    # e2e through the public API: pinned host X -> decompose(...) -> host cores + per-sweep errors.
    # Headline: the reference's DEFAULT AlsConfig (exact error every sweep, per-bucket timing);
    # also the fast configuration (cheap error, graph replay).
    e2e, e2e_fast = None, None
    if not args.no_e2e:
        def timed_calls(cfg):
            decompose(x_host, args.variant, cfg)  # warm-up call (allocator, plan, graph)
            torch.cuda.synchronize()
            reps = []
            for _ in range(args.e2e_reps):
                if world > 1:
                    tdist.barrier()
                t0 = time.perf_counter()
                cores, rep = decompose(x_host, args.variant, cfg)
                reps.append(time.perf_counter() - t0)
            tt = torch.tensor([float(np.mean(reps))], dtype=torch.float64, device=dev)
            if world > 1:
                tdist.all_reduce(tt, op=tdist.ReduceOp.MAX)
            return float(tt.item()), cores, rep

        slab_elems = int(np.prod(dims)) // dim * (hi - lo)
        # element_budget: c5 exceeds the reference's 2^27 default budget for exact errors
        # (validation.py:8-40); the reference needs the same override for this config
        common = dict(ranks=tuple(ranks), max_iters=sweeps, seed=si, dtype=args.dtype, fp64_gemm=args.fp64_gemm,
                      element_budget=int(np.prod(dims)))
        t_call, cores, rep = timed_calls(AlsConfig(**common))
        core_bytes = sum(int(np.prod(c.shape)) * 8 for c in cores)
        e2e = {"value": sweeps / t_call, "unit": "sweeps/s",
               "h2d_bytes_per_step": slab_elems * ebytes,
               "d2h_bytes_per_step": core_bytes + 8 * sweeps,
               "step": f"one decompose(x_host_pinned, '{args.variant}', AlsConfig(ranks, max_iters={sweeps}, "
                       f"seed={si}, element_budget=|X|)) call with the reference's defaults (error_mode='exact' every sweep, "
                       f"per-bucket timing), incl. X's H2D copy and, for the tensor-core engines, its digit "
                       f"slicing; value = sweeps / call time",
               "seconds_per_call": t_call, "final_error": float(rep.errors[-1]),
               "iter_seconds_mean": float(np.mean(rep.iter_seconds))}
        t_call, cores, rep = timed_calls(AlsConfig(error_mode="cheap", timing_buckets=False, **common))
        e2e_fast = {"value": sweeps / t_call, "unit": "sweeps/s", "seconds_per_call": t_call,
                    "step": "same call with error_mode='cheap', timing_buckets=False (CUDA graph replay)",
                    "final_error": float(rep.errors[-1])}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import tenring_oracle as O
        xh = x_host.numpy() if not fp32 else x_host.double().numpy()
        init = O.gaussian_ring(dims, ranks, O.philox(si))
        times, prep = cpu_block_steps(xh, "ne", ranks, init, order)
        t_sweep_cpu = float(sum(times))
        ci = cpu_info()
        cpu = {"value": 1.0 / t_sweep_cpu, "unit": "sweeps/s", "cores": ci.get("blas_threads") or ci["affinity"],
               "kind": "port",
               "sample": (f"one complete full-size NE sweep ({order} block updates, {t_sweep_cpu:.1f} s; set-up "
                          f"{prep:.1f} s untimed as in the reference) of the oracle port of tenring 0.1.0 "
                          f"(materialised subchain, unfold copies, numpy/OpenBLAS) on this run's X"),
               "cpu": ci, "block_seconds": times}
    del x_host

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
        # fp64 on the int8 tensor cores: the algorithmic work of one launch is the int8 products
        # (28 digit pairs, or one per CRT modulus) over the real (unpadded) M x N x K
        i8_tops = env_tf * i8_products
        if crt:
            kern = ("crt8_kernel<pair> (fp64 X x half-chain environment product on the int8 tcgen05 tensor cores "
                    f"by the Chinese remainder theorem: {i8_products} u8 x u8 GEMMs modulo pairwise coprime p_i <= 256, "
                    "cta_group::2 MMAs 256 x {208,192} x 32, exact int32 sums reduced mod p_i in the epilogue; "
                    "timed alone -- the half chain's residue slicing and the exact 128-bit CRT reconstruction "
                    "are separate launches, see other_env_stages_ms)")
        else:
            kern = ("oz8_kernel<64, OzF64> (fp64 X x half-chain environment product on the int8 tcgen05 "
                    "tensor cores: 7 balanced radix-254 digits per operand, 28 exact int32 digit-pair products)")
        roof = {"bound": "tensor", "achieved": i8_tops, "peak": INT8_PEAK_TOPS, "unit": "TFLOP/s",
                "frac": i8_tops / INT8_PEAK_TOPS, "traffic": traffic,
                "kernel": kern,
                "ops": f"int8 tensor ops = {i8_products} x 2 M N K per launch", "flops_per_launch": env_flops,
                "fp64_equiv_tflops": env_tf, "fp64_equiv_frac_of_dmma_peak": env_tf / FP64_PEAK_TFLOPS,
                "avg_launch_ms": env_avg_ms, "share_of_step": env_share,
                "frac_of_burst_peak": i8_tops / INT8_PEAK_BURST_TOPS,
                "other_env_stages_ms": aux_ms or None,
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
        "vs_baseline": None, "dtype": "f32 (X) / f64" if fp32 else "f64",
        "data": "synthetic (BASELINE recipe: cores from the reference Philox stream, X reconstructed on the GPU, "
                "noise from the reference's host Philox stream)",
        "config": {"workload": f"{args.config} {args.variant.upper()} sweep" + (" (fp32 variant)" if fp32 else ""),
                   "dims": dims, "ranks": ranks, "dtype": args.dtype,
                   "variant": args.variant, "parallelism": f"X sharded along mode 0 over {world} GPUs" if world > 1
                   else "single",
                   "l2": "X (%.2f GB) larger than the 126 MB L2, no flush needed" % (np.prod(dims) * ebytes / 1e9),
                   "step": "one full sweep + per-sweep relative error (cheap identity)",
                   "fp64_gemm": None if fp32 else eng_gemm,
                   "int8_engine_forms": i8_forms,
                   "x_digits_ms": prep_ms if (fp32 or oz64) else None,
                   "x_row_range_rho": rho if not fp32 else None,
                   "launch": launch_note},
        "contraction_tflops": F / sweep_s / 1e12,
        "contraction_roofline_frac": t_roof / sweep_s,
        "roofline_sweep_ms": t_roof * 1e3,
        "roofline_pipe_tflops": peak_tf,
        "contraction_roofline_frac_vs_dmma_peak": t_roof_dmma / sweep_s,
        "x_passes_per_sweep": 2,
        "roofline": roof,
        "gpu_launches": int(launches),
        "clocks": clocks,
        "final_error": final_err,
    }
    if e2e is not None:
        line["e2e"] = e2e
        line["e2e_fast"] = e2e_fast
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
    ap.add_argument("--fp64-gemm", choices=["auto", "ozaki", "crt", "dmma"], default="auto",
                    help="fp64 environment products: int8 tensor-core digit slicing, the DMMA pipe, or "
                         "auto (ozaki for products >= 4 GFLOP: c3-c5)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--eager", action="store_true", help="no CUDA graph")
    ap.add_argument("--e2e-reps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.warmup < 3:
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
