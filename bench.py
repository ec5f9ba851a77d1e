#!/usr/bin/env python
"""bench.py -- randomized Tucker (lmra alg1/2/4/5) on B200, BASELINE.json's metric.

Default workload: cfg4 = 1000^3 fp64 (8 GB) Gaussian-core Tucker tensor + 1e-2 noise,
randomized T-HOSVD with nearly-optimal AMM sampling (alg4, rank 50, p=10, q=2, c=400),
the largest BASELINE configuration and the one sharded over 1/2/4/8 GPUs.

A step = one full decomposition (the reference's timed run_algorithm span,
bench.cpp:247-249) of the device-resident tensor.  value = algorithmic tensor bytes
(SURVEY 8d rules R1-R6) per second, whole job.  Inputs are 8 GB >> the 126 MB L2, so
no flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfgX] [--impl reference]

--gpus N > 1 without a torchrun environment relaunches itself under torch.distributed.run
(one process per GPU, NCCL); each rank generates only its slab of the last mode.

--impl reference times the CPU restatement of the reference (oracle/; the reference itself
needs Eigen3, which is absent: DESIGN.md) on all host cores, on the SAME workload and input
bits (the oracle's host generators reproduce the device generators exactly): one full
decomposition per step.  It imports baseline_configs and oracle only -- no GPU library.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L2_FLUSH_BELOW = 256 << 20   # inputs below this may stay L2-resident (126 MB L2): flush per step
L2_FLUSH_BYTES = 256 << 20
P64_MEASURED_TFLOPS = 37.0   # DMMA m16n8k4 loop, profiles/fp64_peaks_r01.json (this pool's B200)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--algorithm", default=None,
                    help="run the config's tensor and AlgoConfig through another algorithm (e.g. alg6/alg7)")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-threads", type=int, default=0, help="CPU arm threads (default: all host cores)")
    ap.add_argument("--no-single-thread", action="store_true",
                    help="reference arm: skip the extra 1-thread decomposition")
    return ap.parse_args()


def maybe_relaunch(args):
    """--gpus N > 1 outside torchrun: relaunch under torch.distributed.run, one rank per GPU."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) != args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}")
        return
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p.get("hbm_gbs", 6557.8), "MEASURED_PEAKS.json"
    except OSError:
        return 6650.0, "fallback (B200_PROFILING.md)"


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region (NVML every 5 ms from a
    host thread, so even a ~100 ms region gets samples; nvidia-smi -lms 200 as fallback)."""
    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40),
               ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4), ("hw_power_brake", 0x80))

    def __init__(self, cuda_index: int, period_s: float = 0.005):
        self.cuda_index = cuda_index
        self.period = period_s
        self.rows = []  # (sm_mhz, max_mhz, reason_bits)
        self.src = None
        self._stop = threading.Event()
        self.t = None

    def _handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:  # map the CUDA device to its NVML handle by PCI bus id
            import torch
            pr = torch.cuda.get_device_properties(self.cuda_index)
            bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:  # noqa: BLE001
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.cuda_index)

    def _sample(self):
        nv, h = self.nv, self.h
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        self.rows.append((float(sm), float(mx), int(bits)))

    def _loop(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:  # noqa: BLE001
                return
            self._stop.wait(self.period)

    def __enter__(self):
        if os.environ.get("LMRA_BENCH_CLOCK_PERIOD"):  # diagnostics: sampling period override
            self.period = float(os.environ["LMRA_BENCH_CLOCK_PERIOD"])
        try:
            self.nv, self.h = self._handle()
            self._sample()
            self.src = "nvml"
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.src = None
            self._smi_start()
        return self

    def _smi_start(self):
        fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                  "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                  "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.cuda_index), f"--query-gpu={fields}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.src = "nvidia-smi"

            def rd():
                for line in self.proc.stdout:
                    p = [x.strip() for x in line.split(",")]
                    if len(p) == 6 and p[0].replace(".", "").isdigit():
                        bits = sum(b for (_, b), v in zip(self.REASONS, p[2:]) if v == "Active")
                        self.rows.append((float(p[0]), float(p[1]), bits))
            self.t = threading.Thread(target=rd, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def __exit__(self, *a):
        if self.src == "nvml":
            self._stop.set()
            self.t.join(1.0)
            try:
                self._sample()
            except Exception:  # noqa: BLE001
                pass
        elif self.src == "nvidia-smi" and self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        reasons = sorted({n for r in self.rows for n, b in self.REASONS if r[2] & b})
        return {"sm_mhz": statistics.median(r[0] for r in self.rows),
                "sm_max_mhz": max(r[1] for r in self.rows), "reasons": reasons,
                "samples": len(self.rows), "source": self.src}


# ------------------------------------------------------------------ workload (both arms)
def workload(args):
    import copy
    from baseline_configs import CONFIGS
    bc = copy.deepcopy(CONFIGS[args.config])
    if args.algorithm:
        bc.alg = args.algorithm
        bc.name = f"{bc.name}/{args.algorithm}"
    return bc


def metric_name(bc):
    return f"tensor GB/s streamed (randomized Tucker, lmra {bc.alg} {bc.name})"


def workload_config(bc, cost):
    """`config` of the JSON line: the workload only (identical for the GPU and the CPU arm)."""
    c = bc.cfg
    return {"workload": f"{bc.name}: {bc.description}", "algorithm": bc.alg, "dims": list(bc.dims),
            "rank": list(c.rank), "oversampling": c.oversampling, "power": c.power, "regime": c.regime,
            "t_samples": c.t_samples, "alpha": c.alpha, "order": c.order, "seed": c.seed,
            "generator": {"kind": bc.generator, **bc.gen_args},
            "l2": ("input >> 126 MB L2; no flush needed" if cost["tensor_bytes"] >= L2_FLUSH_BELOW
                   else "L2 flushed between timed steps (256 MB write outside the per-step CUDA events)"),
            "timing": "per step: CUDA events around the public call (run_raw, its host work included), "
                      "summed over the timed steps; the bench's bookkeeping between steps excluded",
            "algorithmic_bytes_per_step": cost["bytes"], "algorithmic_flops_per_step": cost["flops"]}


def oracle_cfg(O, bc, threads):
    c = bc.cfg
    # LMRA_NUM_THREADS = N for the mode-parallel T-HOSVD variants (README.md:132-135)
    mt = len(bc.dims) if bc.alg in ("alg1", "alg4", "alg6") else 1
    return O.AlgoConfig(rank=list(c.rank), oversampling=c.oversampling, power=c.power, alpha=c.alpha,
                        regime=c.regime, regime_beta=c.regime_beta, t_samples=c.t_samples, order=c.order,
                        seed=c.seed, strategy=c.strategy, mode_threads=mt if threads > 1 else 1,
                        keep_trace=False)


def run_cpu(bc, x, reps: int, warm: int, threads: int):
    """The oracle (C++ restatement of the reference + OpenBLAS) on the host: seconds of the
    run_algorithm span (bench.cpp:247-249) per decomposition."""
    from oracle import oracle as O
    O.set_blas_threads(threads)
    oc = oracle_cfg(O, bc, threads)
    times = []
    for i in range(warm + reps):
        d = O.run(bc.alg, x, bc.dims, oc)
        if i >= warm:
            times.append(d.seconds)
    return times


def bench_reference(args, rank, world):
    if rank != 0:
        return 0
    from baseline_configs import algorithmic_cost, generate_host
    bc = workload(args)
    cost = algorithmic_cost(bc)
    threads = args.cpu_threads or os.cpu_count() or 1
    t0 = time.time()
    x = generate_host(bc)
    gen_s = time.time() - t0
    times = run_cpu(bc, x, max(1, args.steps), args.warmup, threads)
    total = sum(times)
    v = round(cost["bytes"] * len(times) / total / 1e9, 4)
    # BASELINE.md's second CPU row: the reference's default, one thread (LMRA_NUM_THREADS=1,
    # BLAS single-threaded; README.md:132-135), one decomposition of the same workload
    single = None
    if threads > 1 and not args.no_single_thread:
        t1 = run_cpu(bc, x, 1, 0, 1)[0]
        single = {"value": round(cost["bytes"] / t1 / 1e9, 4), "unit": "GB/s", "cores": 1,
                  "seconds_per_decomposition": round(t1, 3),
                  "sample": "one decomposition of the same workload and input bits, 1 thread"}
    sample = (f"the full workload ({'x'.join(map(str, bc.dims))}, {bc.alg}): one decomposition per step, "
              f"{len(times)} timed after {args.warmup} warm-up; oracle C++ restatement of the reference + "
              f"OpenBLAS, {threads} threads; input bits identical to the GPU arm's (host generators), "
              f"generated in {gen_s:.1f} s outside the timed region")
    line = {
        "impl": "reference", "metric": metric_name(bc),
        "value": v, "unit": "GB/s", "n_gpus": world, "steps": len(times), "warmup": args.warmup,
        "ms_per_step": round(total / len(times) * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "parallelism": f"host CPU, {threads} threads",
        "config": workload_config(bc, cost),
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": threads, "kind": "port", "sample": sample,
                         "cpu_model": cpu_model(), "per_step_s": [round(t, 3) for t in times],
                         "single_thread": single},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ roofline
def phase_cost(bc, phase: str, dims_local=None):
    """Algorithmic (flops, bytes, bound) of ONE launch of a phase.  A "_i8" suffix marks a
    contraction run on the int8 tensor cores (same algorithmic cost).  Per-mode phases of the
    latency-bound chains (sampler, orth) get their work estimate with latency_bound=True."""
    if phase.endswith("_i8"):
        phase = phase[:-3]
    dims = list(dims_local or bc.dims)
    cfg = bc.cfg
    N = len(dims)
    mu = [min(m, d) for m, d in zip(cfg.rank, dims)]
    size = float(np.prod(dims))
    sk = [min(m + cfg.oversampling, d) for m, d in zip(mu, dims)]
    qr = bc.alg in ("alg6", "alg7")
    amm = bc.alg in ("alg4", "alg5")
    if phase == "norms":
        if bc.alg == "alg4" and len(dims) == 3:  # fused all-modes pass: one read, N outputs
            return 2.0 * size * 3, (size + sum(size / d for d in dims)) * 8, False
        return 2.0 * size, size * 8 + size / dims[0] * 8, False
    if phase.startswith("core_ttm"):
        k = int(phase[len("core_ttm"):])
        cur = list(dims)
        for n in sorted(range(N), key=lambda n: mu[n])[:k]:
            cur[n] = mu[n]
        n = sorted(range(N), key=lambda n: mu[n])[k]
        if qr and k == 0:
            cur[n] = sk[n]
        inp = float(np.prod(cur))
        return 2.0 * inp * mu[n], (inp + inp / cur[n] * mu[n] + cur[n] * mu[n]) * 8, False
    if phase.startswith("shrink_ttm_m"):
        n = int(phase[len("shrink_ttm_m"):])
        order = list(cfg.order) if cfg.order else list(range(N))
        cur = list(dims)
        for m in order[:order.index(n)]:
            cur[m] = mu[m]
        if qr:
            cur[n] = sk[n]
        inp = float(np.prod(cur))
        return 2.0 * inp * mu[n], (inp + inp / cur[n] * mu[n] + cur[n] * mu[n]) * 8, False
    # per-mode phases: the first processed mode's shapes (T-HOSVD: every mode of cfg1/cfg4)
    n0 = (list(cfg.order) if cfg.order else list(range(N)))[0]
    I, J, s = dims[n0], size / dims[n0], sk[n0]
    T = ((cfg.t_samples or [None] * N)[n0] or int(np.ceil(cfg.alpha * J))) if amm else J
    if phase in ("power_half", "power_gram"):
        return 2.0 * I * T * s, (I * T + T * s + I * s) * 8, False
    if phase == "gather":
        return 0.0, 2.0 * I * T * 8, False
    if phase == "sampler":  # probabilities + Neumaier + prefix sums: ~4 passes over J doubles
        return 0.0, 4.0 * J * 8, True
    if phase == "orth":  # TSQR of I x s + s x s Jacobi (~8 sweeps of s^3)
        return 4.0 * I * s * s + 8.0 * 4.0 * s ** 3, (I * s + I * mu[n0]) * 8, True
    return None


def roofline(bc, cost, per_launch, launches_per_step, ms_per_step, config_key, dims_local=None):
    """Roofline of the dominant kernel: the phase with the longest launch (per-mode phases of
    T-HOSVD overlap on their own streams, so summed phase times would overstate a share)."""
    hbm, src = measured_peaks()
    cands = [(ms, name) for name, ms in per_launch.items() if phase_cost(bc, name, dims_local)]
    if not cands:
        return None
    ms, name = max(cands)
    flops, byts, latency = phase_cost(bc, name, dims_local)
    ridge = P64_MEASURED_TFLOPS * 1e12 / (hbm * 1e9)
    sec = ms / 1e3
    if name.endswith("_i8"):
        # fp64 contraction emulated with exact int8 digit products on tcgen05 (ttm_i8.cu): it
        # streams the tensor once, so its roofline is HBM; the fp64-equivalent rate beside it
        achieved = byts / sec / 1e9
        out = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
               "frac": round(achieved / hbm, 4), "peak_source": src,
               "fp64_equiv_tflops": round(flops / sec / 1e12, 2),
               "impl": "int8 tcgen05 digit products (ttm_i8.cu)"}
    elif byts and (flops / byts <= ridge):
        achieved = byts / sec / 1e9
        out = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
               "frac": round(achieved / hbm, 4), "peak_source": src}
    else:
        achieved = flops / sec / 1e12
        out = {"bound": "tensor", "achieved": round(achieved, 4), "peak": P64_MEASURED_TFLOPS,
               "unit": "TFLOP/s", "frac": round(achieved / P64_MEASURED_TFLOPS, 5),
               "peak_source": "measured fp64 DMMA peak (profiles/fp64_peaks_r01.json); fp64 has no "
                              "tcgen05 kind, MEASURED_PEAKS.json carries bf16 only"}
    if latency:
        out["latency_bound"] = True
        out["note"] = ("latency-bound chain (a few CTAs, dependent steps): the work estimate is far below "
                       "both rooflines by construction")
    out.update({"kernel": name, "launch_ms": round(ms, 4),
                "launches_per_step": launches_per_step.get(name),
                "share_of_step": round(ms * launches_per_step.get(name, 1) / ms_per_step, 3),
                "share_note": "launch ms x launches per step / ms per step (per-mode launches of T-HOSVD "
                              "overlap on their own streams, so a per-mode phase's share can exceed its "
                              "critical-path share)",
                "algorithmic_flops_per_launch": flops, "algorithmic_bytes_per_launch": byts,
                "traffic": traffic_from_profiles(config_key, name),
                "whole_step_frac": round(cost["bytes"] / (ms_per_step / 1e3) / 1e9 / hbm, 4)})
    return out


def traffic_from_profiles(config_key: str, kernel_phase: str):
    """dram read + write bytes per launch of the kernel (ncu --set full), keyed by (config, phase)."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        v = d.get(config_key, {})
        return v.get(kernel_phase) if isinstance(v, dict) else None
    except (OSError, ValueError, AttributeError):
        return None


# ------------------------------------------------------------------ GPU arm
def generate_rank_input(P, bc, ctx, world, rank, dist):
    """This rank's input: the whole tensor (1 GPU) or its slab of the last mode, generated on
    the device without the rest (the Tucker + noise tensor exchanges per-slice norms)."""
    from paper_2303_11612_b200 import device
    from paper_2303_11612_b200.configs import generate_device, generate_device_slab
    dims = list(bc.dims)
    if world == 1:
        return generate_device(bc, ctx=ctx), dims
    start, count = P.shard_range(dims[-1], world, rank)
    local = dims[:-1] + [count]
    if bc.generator != "tucker_noise":
        return generate_device_slab(bc, start, count, ctx=ctx), local
    g = bc.gen_args
    x, sb, se = device.gen_tucker_signal_slab(dims, g["core_dims"], g["seed"], start, count, ctx=ctx)
    allb, alle = [None] * world, [None] * world
    dist.all_gather_object(allb, sb)
    dist.all_gather_object(alle, se)
    coef = device.noise_coef(np.concatenate(allb), np.concatenate(alle), g["gamma"])
    device.gen_add_noise_slab(x, dims, g["seed"], start, count, coef, ctx=ctx)
    return x, local


def bench_gpu(args, rank, world, local_rank):
    import torch
    import paper_2303_11612_b200 as P
    from baseline_configs import algorithmic_cost
    from paper_2303_11612_b200.configs import algo_config

    torch.cuda.set_device(local_rank)
    stream = torch.cuda.current_stream()
    ctx = P.Context(local_rank, stream.cuda_stream)
    # light profiling in the timed region (events only around the mode-0 contraction, the
    # roofline's dominant launch on the streaming configs); the full per-phase
    # breakdown comes from untimed profiled runs after it (per-phase event bookkeeping of the
    # per-mode chains costs host time between runs)
    timed_prof = int(os.environ.get("LMRA_BENCH_PROFILE", "3"))  # 3: the mode-0 contraction only
    ctx.set_profiling(timed_prof)
    bc = workload(args)
    cfg = algo_config(bc)
    dist = None
    if world > 1:
        import torch.distributed as dist
        uid = P.nccl_unique_id() if rank == 0 else b"\0" * 128
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        ctx.set_comm(obj[0], world, rank)

    x, local_dims = generate_rank_input(P, bc, ctx, world, rank, dist)
    dims = list(bc.dims)
    torch.cuda.synchronize()
    t = P.DenseTensor.device(x, local_dims)
    cost = algorithmic_cost(bc)

    def barrier():
        if dist is not None:
            dist.barrier()

    for _ in range(args.warmup):
        r = P.run_raw(bc.alg, t, cfg, ctx=ctx, global_dims=dims)
        r.free()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()

    phases = {}
    launches = 0
    host_split = {"host_rng_ms": 0.0, "host_sampling_ms": 0.0, "total_ms": 0.0, "device_ms": 0.0}
    # inputs that fit the 126 MB L2 (cfg1) are timed step by step with the L2 flushed in between
    # (a 256 MB write outside the per-step events); larger inputs stream from HBM anyway
    flush = None
    if cost["tensor_bytes"] < L2_FLUSH_BELOW:
        flush = torch.empty(L2_FLUSH_BYTES // 8, dtype=torch.float64, device="cuda")
    # every step is the public call (run_raw: host preamble, device work, its closing
    # synchronisation) bracketed by CUDA events on the stream; the bench's own bookkeeping between
    # steps (reading the phase timings back through ctypes, ~50 us) stays outside
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    with ClockSampler(local_rank) as clk:
        for i in range(args.steps):
            if flush is not None:
                flush.zero_()
            evs[i][0].record(stream)
            r = P.run_raw(bc.alg, t, cfg, ctx=ctx, global_dims=dims)
            evs[i][1].record(stream)
            for k, (ms, cnt) in r.phases().items():
                a = phases.get(k, (0.0, 0))
                phases[k] = (a[0] + ms, a[1] + cnt)
            tm = r.timings()
            launches += tm["launches"]
            for k in host_split:
                host_split[k] += tm[k]
            r.free()
        torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in evs)
    barrier()
    if dist is not None:
        tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    ms_per_step = ms / args.steps
    value = cost["bytes"] * args.steps / (ms / 1e3) / 1e9
    # full per-phase breakdown (diagnostics + the per-mode phases' launch times): two untimed
    # runs with every phase profiled (CUDA events on each launch's own stream)
    ctx.set_profiling(1)
    breakdown = {}
    for _ in range(2):
        r = P.run_raw(bc.alg, t, cfg, ctx=ctx, global_dims=dims)
        for k, (pms, cnt) in r.phases().items():
            a = breakdown.get(k, (0.0, 0))
            breakdown[k] = (a[0] + pms, a[1] + cnt)
        r.free()
    ctx.set_profiling(timed_prof)

    # e2e through the public API with a pinned host tensor (H2D in the timed region) and
    # the core + factors read back to the host every step
    e2e = None
    host = None
    if args.e2e_steps > 0 or (world == 1 and not args.no_cpu_baseline):
        host = torch.empty(x.numel(), dtype=torch.float64, pin_memory=True)
        host.copy_(x)
        torch.cuda.synchronize()
    if args.e2e_steps > 0:
        th = P.DenseTensor(local_dims, host.numpy())  # host buffer (pinned): H2D inside every step
        r = P.run_raw(bc.alg, th, cfg, ctx=ctx, global_dims=dims)
        dec = r.to_host(with_trace=False)
        r.free()
        d2h = (dec.core.size + sum(f.size for f in dec.factors)) * 8
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            r = P.run_raw(bc.alg, th, cfg, ctx=ctx, global_dims=dims)
            dec = r.to_host(with_trace=False)
            r.free()
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        if dist is not None:
            tt = torch.tensor([ems], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ems = float(tt.item())
        # whole job: every rank copies its slab in (together the full tensor) and reads back
        # the (replicated) core + factors
        e2e = {"value": round(cost["bytes"] * args.e2e_steps / (ems / 1e3) / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": int(np.prod(dims)) * 8, "d2h_bytes_per_step": int(d2h) * world,
               "ms_per_step": round(ems / args.e2e_steps, 3), "steps": args.e2e_steps}

    if rank != 0:
        return 0
    # per-launch device times: main-stream phases from the timed region, the per-mode chains
    # (their own streams) from the profiled runs
    per_launch = {k: v[0] / v[1] for k, v in breakdown.items() if v[1]}
    per_launch.update({k: v[0] / v[1] for k, v in phases.items() if v[1]})
    per_step = {k: v[1] / 2 for k, v in breakdown.items()}
    roof = roofline(bc, cost, per_launch, per_step, ms_per_step, bc.name,
                    local_dims if world > 1 else None)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        threads = args.cpu_threads or os.cpu_count() or 1
        reps = 1 if cost["tensor_bytes"] > 1e9 else 3
        xt = host.numpy()  # the same bits the GPU decomposed
        ctimes = run_cpu(bc, xt, reps, 0, threads)
        med = statistics.median(ctimes)
        cpu = {"value": round(cost["bytes"] / med / 1e9, 4), "unit": "GB/s", "cores": threads, "kind": "port",
               "sample": f"the full workload, {reps} decomposition(s) (median {med:.2f} s): oracle C++ "
                         f"restatement of the reference + OpenBLAS on {threads} host threads, same input bits",
               "cpu_model": cpu_model()}
    line = {
        "metric": metric_name(bc),
        "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "parallelism": f"shard-last-mode x{world} (NCCL)" if world > 1 else "single GPU",
        "config": workload_config(bc, cost),
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "host_ms_per_step": {k: round(v / args.steps, 3) for k, v in host_split.items()},
        # device time per phase and decomposition, from two untimed fully profiled runs (the
        # per-mode phases of T-HOSVD overlap on their own streams)
        "phases_ms_per_step": {k: round(v[0] / 2, 4) for k, v in sorted(breakdown.items())},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    maybe_relaunch(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return bench_reference(args, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # the communicator log shows the rank count
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        return bench_gpu(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
