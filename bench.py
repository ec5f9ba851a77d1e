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

--impl reference times the CPU restatement of the reference (oracle/, the reference
itself needs Eigen3 which is absent: DESIGN.md) on the host cores, on a bounded sample
of the same workload (cfg4's 1000x1000x125 slab = one 8-GPU rank's share).
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

P64_MEASURED_TFLOPS = 37.0   # DMMA m16n8k4 loop, profiles/fp64_peaks_r01.json (this pool's B200)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--algorithm", default=None,
                    help="run the config's tensor and AlgoConfig through another algorithm (e.g. alg6/alg7)")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p.get("hbm_gbs", 6557.8), "MEASURED_PEAKS.json"
    except OSError:
        return 6650.0, "fallback (B200_PROFILING.md)"


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


def phase_cost(bc, phase: str, dims_local=None):
    """Algorithmic (flops, bytes) of ONE launch of a phase, for the roofline.  A "_i8" suffix
    marks a contraction run on the int8 tensor cores (same algorithmic cost)."""
    if phase.endswith("_i8"):
        phase = phase[:-3]
    dims = list(dims_local or bc.dims)
    cfg = bc.cfg
    N = len(dims)
    mu = [min(m, d) for m, d in zip(cfg.rank, dims)]
    size = float(np.prod(dims))
    if phase == "norms":
        if bc.alg == "alg4" and len(dims) == 3:  # fused all-modes pass: one read, N outputs
            return 2.0 * size * 3, (size + sum(size / d for d in dims)) * 8
        return 2.0 * size, size * 8 + size / dims[0] * 8
    qr = bc.alg in ("alg6", "alg7")  # the first core / every shrink contraction reads P (s rows)
    sk = [min(m + cfg.oversampling, d) for m, d in zip(mu, dims)]
    if phase.startswith("core_ttm"):
        k = int(phase[len("core_ttm"):])
        cur = list(dims)
        for n in sorted(range(N), key=lambda n: mu[n])[:k]:
            cur[n] = mu[n]
        n = sorted(range(N), key=lambda n: mu[n])[k]
        if qr and k == 0:
            cur[n] = sk[n]
        inp = float(np.prod(cur))
        return 2.0 * inp * mu[n], (inp + inp / cur[n] * mu[n] + cur[n] * mu[n]) * 8
    if phase.startswith("shrink_ttm_m"):
        n = int(phase[len("shrink_ttm_m"):])
        order = list(cfg.order) if cfg.order else list(range(N))
        cur = list(dims)
        for m in order[:order.index(n)]:
            cur[m] = mu[m]
        if qr:
            cur[n] = sk[n]
        inp = float(np.prod(cur))
        return 2.0 * inp * mu[n], (inp + inp / cur[n] * mu[n] + cur[n] * mu[n]) * 8
    return None


def roofline(bc, phases, steps, dims_local=None, ms_per_step=None):
    hbm, src = measured_peaks()
    # dominant kernel = the phase with the largest device time among the launches that run
    # alone on the main stream (core / shrink contractions, the fused norms pass); the
    # per-mode phases of T-HOSVD overlap on their own streams, so their event times
    # include contention and are not a per-kernel duration
    # ("norms" only as the single fused 3-mode pass: ST-HOSVD's per-mode norms read shrinking
    # tensors of different sizes under one phase name)
    cands = [(ms, name, cnt) for name, (ms, cnt) in phases.items()
             if phase_cost(bc, name, dims_local) and (name != "norms" or cnt == steps)]
    if not cands:
        return None
    ms, name, cnt = max(cands)
    flops, byts = phase_cost(bc, name, dims_local)
    per_launch_ms = ms / cnt
    ridge = P64_MEASURED_TFLOPS * 1e12 / (hbm * 1e9)
    if name.endswith("_i8"):
        # fp64 contraction emulated with exact int8 digit products on tcgen05 (ttm_i8.cu): it
        # streams the tensor once, so its roofline is HBM; the fp64-equivalent rate is reported
        # beside it (above the 37 TF DMMA peak by construction)
        achieved = byts / (per_launch_ms / 1e3) / 1e9
        out = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
               "frac": round(achieved / hbm, 4), "peak_source": src,
               "fp64_equiv_tflops": round(flops / (per_launch_ms / 1e3) / 1e12, 2),
               "impl": "int8 tcgen05 digit products (ttm_i8.cu)"}
    elif flops / byts > ridge:
        achieved = flops / (per_launch_ms / 1e3) / 1e12
        out = {"bound": "tensor", "achieved": round(achieved, 3), "peak": P64_MEASURED_TFLOPS,
               "unit": "TFLOP/s", "frac": round(achieved / P64_MEASURED_TFLOPS, 4),
               "peak_source": "measured fp64 DMMA peak (profiles/fp64_peaks_r01.json); fp64 has no "
                              "tcgen05 kind, MEASURED_PEAKS.json carries bf16 only"}
    else:
        achieved = byts / (per_launch_ms / 1e3) / 1e9
        out = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
               "frac": round(achieved / hbm, 4), "peak_source": src}
    out.update({"kernel": name, "launch_ms": round(per_launch_ms, 4),
                # per-launch device time over the step's device time (the per-mode phases run
                # concurrently, so a sum of phase times would overstate the step)
                "share_of_step": round(per_launch_ms * cnt / steps / ms_per_step, 3) if ms_per_step
                else None,
                "algorithmic_flops_per_launch": flops, "algorithmic_bytes_per_launch": byts,
                "traffic": traffic_from_profiles(name)})
    return out


def traffic_from_profiles(kernel_phase: str):
    """dram bytes per launch of the dominant kernel from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(kernel_phase)
    except (OSError, ValueError):
        return None


def cpu_sample_workload():
    """Bounded CPU sample: cfg4's structure on the 1000x1000x125 slab (one 8-GPU rank's share)."""
    from paper_2303_11612_b200.configs import scaled
    return scaled("cfg4", [1000, 1000, 125])


def run_cpu(bc, reps: int, warm: int):
    from oracle import oracle as O
    from paper_2303_11612_b200.configs import algorithmic_cost
    cores = os.cpu_count() or 1
    O.set_blas_threads(cores)
    x = O.gen_tucker_noise(bc.dims, bc.gen_args["core_dims"], bc.gen_args["gamma"], bc.gen_args["seed"])
    c = bc.cfg
    oc = O.AlgoConfig(rank=list(c.rank), oversampling=c.oversampling, power=c.power, alpha=c.alpha,
                      regime=c.regime, regime_beta=c.regime_beta, t_samples=c.t_samples, order=c.order,
                      seed=c.seed, strategy=c.strategy, mode_threads=len(bc.dims), keep_trace=False)
    times = []
    for i in range(warm + reps):
        d = O.run(bc.alg, x, bc.dims, oc)
        if i >= warm:
            times.append(d.seconds)
    B = algorithmic_cost(bc)["bytes"]
    return {"per_step_s": times, "value": B / statistics.median(times) / 1e9, "cores": cores,
            "bytes": B}


def bench_reference(args, rank, world):
    if rank != 0:
        return 0
    bc = cpu_sample_workload()
    res = run_cpu(bc, max(1, args.steps), args.warmup)
    total = sum(res["per_step_s"])
    v = round(res["value"], 4)
    sample = (f"{bc.alg} on {'x'.join(map(str, bc.dims))} (cfg4 structure, 1/8 slab), oracle C++ "
              f"restatement + OpenBLAS, {res['cores']} threads, median of {len(res['per_step_s'])}")
    line = {
        "impl": "reference", "metric": "tensor GB/s streamed (randomized Tucker, lmra alg4 cfg4)",
        "value": v, "unit": "GB/s", "n_gpus": world, "steps": len(res["per_step_s"]), "warmup": args.warmup,
        "ms_per_step": round(total / len(res["per_step_s"]) * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg4 sample: " + bc.name, "algorithm": bc.alg, "dims": bc.dims},
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": res["cores"], "kind": "port",
                         "sample": sample},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def bench_gpu(args, rank, world, local_rank):
    import torch
    import paper_2303_11612_b200 as P
    from paper_2303_11612_b200.configs import CONFIGS, algorithmic_cost, generate_device

    torch.cuda.set_device(local_rank)
    stream = torch.cuda.current_stream()
    ctx = P.Context(local_rank, stream.cuda_stream)
    # light profiling in the timed region (events only around the launches on the main stream:
    # the norm pass and the contractions, what the roofline needs); the full per-phase
    # breakdown comes from untimed profiled runs after it (per-phase event bookkeeping of the
    # per-mode chains costs host time between runs)
    timed_prof = int(os.environ.get("LMRA_BENCH_PROFILE", "2"))
    ctx.set_profiling(timed_prof)
    bc = CONFIGS[args.config]
    if args.algorithm:
        import copy
        bc = copy.deepcopy(bc)
        bc.alg = args.algorithm
        bc.name = f"{bc.name}/{args.algorithm}"
    dist = None
    if world > 1:
        import torch.distributed as dist
        uid = P.nccl_unique_id() if rank == 0 else b"\0" * 128
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        ctx.set_comm(obj[0], world, rank)

    x = generate_device(bc, ctx=ctx)
    dims = list(bc.dims)
    local_dims = list(dims)
    if world > 1:  # this rank's slab of the last mode (lmra_shard_range)
        start, count = P.shard_range(dims[-1], world, rank)
        slab = int(np.prod(dims[:-1]))
        x = x[start * slab:(start + count) * slab].clone()
        local_dims[-1] = count
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
    t = P.DenseTensor.device(x, local_dims)
    cost = algorithmic_cost(bc)

    def barrier():
        if dist is not None:
            dist.barrier()

    for _ in range(args.warmup):
        r = P.run_raw(bc.alg, t, bc.cfg, ctx=ctx, global_dims=dims)
        r.free()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()

    phases = {}
    launches = 0
    host_split = {"host_rng_ms": 0.0, "host_sampling_ms": 0.0, "total_ms": 0.0, "device_ms": 0.0}
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            r = P.run_raw(bc.alg, t, bc.cfg, ctx=ctx, global_dims=dims)
            for k, (ms, cnt) in r.phases().items():
                a = phases.get(k, (0.0, 0))
                phases[k] = (a[0] + ms, a[1] + cnt)
            tm = r.timings()
            launches += tm["launches"]
            for k in host_split:
                host_split[k] += tm[k]
            r.free()
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    barrier()
    if dist is not None:
        tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    ms_per_step = ms / args.steps
    value = cost["bytes"] * args.steps / (ms / 1e3) / 1e9
    # full per-phase breakdown (diagnostics): two untimed runs with every phase profiled
    ctx.set_profiling(1)
    breakdown = {}
    for _ in range(2):
        r = P.run_raw(bc.alg, t, bc.cfg, ctx=ctx, global_dims=dims)
        for k, (pms, cnt) in r.phases().items():
            a = breakdown.get(k, (0.0, 0))
            breakdown[k] = (a[0] + pms, a[1] + cnt)
        r.free()
    ctx.set_profiling(timed_prof)

    # e2e through the public API with a pinned host tensor (H2D in the timed region) and
    # the core + factors read back to the host every step
    e2e = None
    if args.e2e_steps > 0:
        host = torch.empty(x.numel(), dtype=torch.float64, pin_memory=True)
        host.copy_(x)
        th = P.DenseTensor(local_dims, host.numpy())  # host buffer (pinned): H2D inside every step
        r = P.run_raw(bc.alg, th, bc.cfg, ctx=ctx, global_dims=dims)
        dec = r.to_host(with_trace=False)
        r.free()
        d2h = (dec.core.size + sum(f.size for f in dec.factors)) * 8
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            r = P.run_raw(bc.alg, th, bc.cfg, ctx=ctx, global_dims=dims)
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
        del host

    if rank != 0:
        return 0
    roof = roofline(bc, phases, args.steps, local_dims if world > 1 else None, ms_per_step)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        sbc = cpu_sample_workload()
        cres = run_cpu(sbc, 3, 0)
        cpu = {"value": round(cres["value"], 4), "unit": "GB/s", "cores": cres["cores"], "kind": "port",
               "sample": f"{sbc.alg} on {'x'.join(map(str, sbc.dims))} (cfg4 structure, 1/8 slab); "
                         f"oracle C++ restatement + OpenBLAS, {cres['cores']} threads, median of 3 "
                         f"({', '.join(f'{s:.2f}' for s in cres['per_step_s'])} s)"}
    line = {
        "metric": f"tensor GB/s streamed (randomized Tucker, lmra {bc.alg} {bc.name})",
        "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{bc.name}: {bc.description}", "algorithm": bc.alg, "dims": dims,
                   "rank": list(bc.cfg.rank), "oversampling": bc.cfg.oversampling,
                   "power": bc.cfg.power, "regime": bc.cfg.regime,
                   "t_samples": bc.cfg.t_samples, "alpha": bc.cfg.alpha,
                   "parallelism": f"shard-last-mode x{world}" if world > 1 else "single GPU",
                   "l2": "input 8 GB >> 126 MB L2; no flush needed" if bc.name == "cfg4"
                         else "input may be L2-resident between steps",
                   "algorithmic_bytes_per_step": cost["bytes"], "algorithmic_flops_per_step": cost["flops"]},
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
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return bench_reference(args, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist
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
