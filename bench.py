#!/usr/bin/env python
"""Benchmark of the hot path: one step = one hjmc_solve_slice over BASELINE.json configs[1]
(C2: n=3 Dubins pursuit-evasion slice, 101×101 queries, N=65,536 samples, 10 horizons × 8
Picard iterates, fp32) — all of Algorithm 1 plus the running-min tube.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

Multi-GPU (launched by torchrun, one rank per GPU, NCCL): queries are independent, so every
rank solves its own slice of the same size (global query ids offset by rank·M; weak scaling)
with no collective on the data path. Timing: barrier + synchronize around K steps, CUDA
events on the launching stream, max over ranks. --impl reference times the CPU oracle (the
reference arm for this tier) on a bounded sample of the same workload on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("query·sample evals/sec and s per 2D BRT slice at 1/2/4/8 B200; "
          "% FP32/MUFU peak")
UNIT = "evals/s"
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c2", help="c1..c5 (default c2 = BASELINE configs[1])")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=0, help="oracle sample queries (0 = auto)")
    return ap.parse_args()


def preset_for(name):
    from paper_2605_18566_b200 import inputs as I

    return I.BY_INDEX[int(name.lower().lstrip("c"))]


# Functional check of the N > 1 code path on a one-GPU box (never a timing): every rank uses
# cuda:0 and the process group is gloo. The ranks' kernels never wait on one another (the
# queries are independent), so this exercises the launch, max-over-ranks and gather logic only.
PATH_CHECK = os.environ.get("HJMC_BENCH_PATH_CHECK") == "1"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = 0 if PATH_CHECK else int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---- clocks sampled during the timed region ----------------------------------------------------
class ClockSampler:
    """SM clock, power and throttle reasons sampled by NVML in a background thread (every
    100 ms: ≥ 10 Hz) while the timed region runs — in-process, so no polling
    subprocess competes."""

    REASONS = {  # NVML clocks-event-reason bits
        "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "sw_power_cap": 0x4,
    }

    def __init__(self, index: int, period_s: float = 0.1):
        self.index, self.period = index, period_s
        self.rows, self.stop_evt, self.thread, self.h = [], threading.Event(), None, None

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        except Exception:
            self.h = None
            return
        self.thread = threading.Thread(target=self._loop, daemon=True)
        self.thread.start()

    def _loop(self):
        nv = self.nv
        while not self.stop_evt.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                pw = nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.rows.append((sm, pw, rs))
            except Exception:
                pass
            self.stop_evt.wait(self.period)

    def stop(self):
        if self.h is None:
            return None
        self.stop_evt.set()
        self.thread.join(timeout=2)
        if not self.rows:
            return None
        nv = self.nv
        smax = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        sm = [r[0] for r in self.rows]
        reasons = sorted({k for r in self.rows for k, bit in self.REASONS.items() if r[2] & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(smax), "sm_min_mhz": min(sm),
                "samples": len(self.rows), "reasons": reasons,
                "power_w_max": max(r[1] for r in self.rows), "source": "NVML, 100 ms"}


# ---- CPU oracle (cpu_baseline leg and the reference arm) --------------------------------------
def oracle_sample_run(preset, count: int, seed_offset: int = 0, nthreads: int = 0):
    """Time the oracle, as it stands, on `count` queries of the workload (full K×Kp×N each);
    nthreads = 0 uses every host core (OpenMP over queries), 1 is the paper's setting."""
    import oracle as O
    from paper_2605_18566_b200 import inputs as I

    O.build()
    P = O.Problem.from_preset(preset)
    x_all = I.queries(preset)
    ids = I.subsample_ids(x_all.shape[0], count)
    ids = (ids + seed_offset) % x_all.shape[0]
    t0 = time.perf_counter()
    r = O.solve_slice(P, x_all[ids], qids=ids.astype(np.uint32), nthreads=nthreads)
    dt = time.perf_counter() - t0
    evals = len(ids) * preset.N * preset.K * preset.Kp
    return evals / dt, dt, len(ids), (nthreads or O.max_threads()), r


def auto_sample(preset) -> int:
    """Queries of the oracle sample: ~10–30 s of host CPU work on this box's cores."""
    import oracle as O

    cores = O.max_threads()
    per_query_core_s = preset.N * preset.K * preset.Kp * preset.n * 1.0e-7  # measured: 1.56 s per C2 query-core
    return int(max(cores, min(512, round(15.0 * cores / max(per_query_core_s, 1e-9)))))


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    preset = preset_for(args.config)
    count = args.cpu_sample or max(1, auto_sample(preset) // 4)
    for w in range(args.warmup):
        oracle_sample_run(preset, max(1, count // 8), seed_offset=17 * (w + 1))
    vals, secs = [], 0.0
    for s in range(args.steps):
        v, dt, used, cores, _ = oracle_sample_run(preset, count, seed_offset=31 * s)
        vals.append(v)
        secs += dt
    value = float(np.mean(vals))
    sample = (f"{used} of {preset.M} queries of {preset.name} (deterministic spread), full "
              f"K×Kp×N = {preset.K}×{preset.Kp}×{preset.N} per query, per step")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * secs / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": preset.name, "n": preset.n, "M": preset.M,
                                        "N": preset.N, "K": preset.K, "Kp": preset.Kp},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---- our arm --------------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2605_18566_b200 import inputs as I
    from paper_2605_18566_b200 import roofline as RL
    from paper_2605_18566_b200.solver import Solver, SolverConfig

    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        if PATH_CHECK:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    preset = preset_for(args.config)
    solver = Solver(SolverConfig.from_preset(preset, device=local))
    x_host = I.queries(preset)
    M = x_host.shape[0]
    qid_base = rank * M                     # weak scaling: each rank owns its own M queries
    x = torch.from_numpy(x_host).to(dev)
    out = solver.alloc_result(M, hist=True)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        flush.zero_()                        # warm everything the timed loop launches
        solver.solve_slice(x, qid_base=qid_base, out=out)
    solver.check()
    torch.cuda.synchronize(dev)

    clocks = ClockSampler(local) if not args.no_clocks else None
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize(dev)
    if clocks:
        clocks.start()
        time.sleep(0.3)
    t_start.record(stream)
    for s in range(args.steps):
        flush.zero_()                        # L2 flush between steps (not our kernel)
        ev[s][0].record(stream)
        solver.solve_slice(x, qid_base=qid_base, out=out)
        ev[s][1].record(stream)
    t_end.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    clk = clocks.stop() if clocks else None
    solver.check()
    total_ms = t_start.elapsed_time(t_end)
    kernel_ms = [a.elapsed_time(b) for a, b in ev]
    t = torch.tensor([total_ms, sum(kernel_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, kern_sum = float(t[0]), float(t[1])
    evals_step_rank = M * preset.N * preset.K * preset.Kp
    value = evals_step_rank * world * args.steps / (total_ms / 1000.0)
    kern_avg_ms = kern_sum / args.steps

    # ---- the per-slice result gather (north_star: the only NCCL traffic), timed separately:
    # every rank's (v, dv, c, tube) all-gathered over NVLink after the solve --------------------
    gather = None
    if world > 1:
        from paper_2605_18566_b200 import shard

        res = {k: out[k] for k in ("v", "dv", "c", "tube")}
        shard.gather_results(res, M * world)              # warm the communicator
        torch.cuda.synchronize(dev)
        barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        full = shard.gather_results(res, M * world)
        g1.record(stream)
        torch.cuda.synchronize(dev)
        gt = torch.tensor([g0.elapsed_time(g1)], dtype=torch.float64, device=dev)
        dist.all_reduce(gt, op=dist.ReduceOp.MAX)
        gather = {"ms": float(gt[0]),
                  "collective": f"all_gather over {dist.get_backend()} (torch.distributed)",
                  "bytes_per_rank": int(sum(t.numel() * 4 for t in res.values())),
                  "bytes_gathered": int(sum(t.numel() * 4 for t in full.values())),
                  "share_of_step": float(gt[0]) / (total_ms / args.steps)}

    # ---- end to end: host buffers through hjmc_solve_slice_host (copies inside) ----------
    e2e = None
    if True:
        pin = lambda *s: torch.empty(s, dtype=torch.float32).pin_memory()
        xh = torch.from_numpy(x_host).pin_memory()
        hout = {"v": pin(M), "dv": pin(M, preset.n), "c": pin(M), "tube": pin(M)}
        solver.solve_slice_host(xh, qid_base=qid_base, out=hout)
        barrier()
        t0 = time.perf_counter()
        e2e_steps = max(1, min(args.steps, 3))
        for _ in range(e2e_steps):
            solver.solve_slice_host(xh, qid_base=qid_base, out=hout)
        dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e = {"value": evals_step_rank * world * e2e_steps / float(dt[0]), "unit": UNIT,
               "h2d_bytes_per_step": int(x_host.nbytes),
               "d2h_bytes_per_step": int(sum(v.numel() * 4 for v in hout.values())),
               "api": "hjmc_solve_slice_host (pageable-safe pinned host buffers, synchronous)"}

    # ---- fast path: the same solve with the exact shortcuts (bit-identical outputs): a Picard
    # iterate whose coefficient was already used — or, at a clamp, speculatively accumulated —
    # by its (query, horizon) reuses those sums instead of re-sampling ------------------------
    fast = Solver(SolverConfig.from_preset(preset, device=local, skip_stationary=True,
                                           reuse_passes=True, speculate=True))
    fast.solve_slice(x, qid_base=qid_base, out=out)
    fast.pass_count()
    fe0, fe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fsteps = max(1, min(args.steps, 3))
    barrier()
    fe0.record(stream)
    for _ in range(fsteps):
        fast.solve_slice(x, qid_base=qid_base, out=out)
    fe1.record(stream)
    torch.cuda.synchronize(dev)
    fpasses = fast.pass_count() / fsteps
    fms = torch.tensor([fe0.elapsed_time(fe1) / fsteps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(fms, op=dist.ReduceOp.MAX)
    fastpath = {"flag": "HJMC_FLAG_SKIP_STATIONARY | HJMC_FLAG_REUSE_PASSES | "
                        "HJMC_FLAG_SPECULATE_CLAMPS", "ms_per_step": float(fms[0]),
                "s_per_slice": float(fms[0]) / 1000.0,
                "passes_executed_frac": fpasses / (M * preset.K * preset.Kp),
                "evals_executed_per_s": fpasses * preset.N * world / (float(fms[0]) / 1000.0),
                "note": "outputs bit-identical to the full schedule (tests/test_gpu_parity.py); "
                        "the headline value counts the full K×Kp schedule without it"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    # ---- roofline (ALU / MUFU pipes) -----------------------------------------
    rates, rate_src = RL.load_rates()
    rl = RL.roofline(preset.n, preset.target, preset.antithetic, rates=rates)
    pipe = rl["binding_pipe"]
    ops_per_launch = rl["ops"][pipe] * evals_step_rank
    achieved = ops_per_launch / (kern_avg_ms / 1000.0) / 1e9
    peak = rl["peak_ops_per_s"] / 1e9
    roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Gop/s",
            "frac": achieved / peak, "traffic": None,
            "pipe": pipe, "ops_per_eval": rl["ops"],
            "peak_basis": f"{rl['rate']:.0f} lane-ops/clk/SM × 148 SMs × 1965 MHz (sm_max); "
                          f"rates: {rate_src}",
            "kernel": f"solve_kernel<{preset.target}, n={preset.n}, 256 threads> "
                      "(+ tube epilogue, <0.1%)",
            "kernel_ms_avg": kern_avg_ms}
    if clk and clk.get("sm_mhz"):
        roof["frac_at_measured_clock"] = roof["frac"] * 1965.0 / clk["sm_mhz"]
    # the query / coefficient / result streams (north_star: "achieved HBM GB/s"): per unit the
    # kernel reads x (n floats) and writes, per Picard iterate, vhist + chist, and per query
    # v, dv, c, tube, g0 — algorithmic bytes over the kernel time, against the measured copy peak
    hbm_bytes = 4 * (M * preset.K * preset.n + 2 * M * preset.K * preset.Kp
                     + M * (preset.n + 4))
    peaks_file = os.path.join(ROOT, "MEASURED_PEAKS.json")
    hbm_peak = None
    if os.path.exists(peaks_file):
        with open(peaks_file) as fh:
            hbm_peak = json.load(fh).get("hbm_gbs")
    hbm_gbps = hbm_bytes / (kern_avg_ms / 1000.0) / 1e9
    roof["hbm"] = {"algorithmic_bytes_per_launch": int(hbm_bytes), "achieved_gbps": hbm_gbps,
                   "peak_gbps": hbm_peak,
                   "frac": (hbm_gbps / hbm_peak) if hbm_peak else None,
                   "note": "no sample touches HBM; the streams are queries and per-iterate results"}
    # context for the fraction: the measured throughput ceiling of this kernel's own instruction
    # mix (tools/mix_ceiling.cu, C2 only)
    mix_file = os.path.join(ROOT, "profiles", "r1_mix_ceiling.json")
    if preset.name == "c2_dubins_n3" and os.path.exists(mix_file):
        with open(mix_file) as fh:
            mix = json.load(fh)["mixes"]["full_c2_mix"]["evals_per_clk_per_sm"]
        f_hz = (clk["sm_mhz"] if clk and clk.get("sm_mhz") else RL.F_MAX_MHZ) * 1e6
        per_clk = evals_step_rank / (kern_avg_ms / 1000.0) / (RL.NSM * f_hz)
        roof["mix_ceiling"] = {"evals_per_clk_per_sm": mix, "kernel_evals_per_clk_per_sm": per_clk,
                               "frac": per_clk / mix,
                               "source": "profiles/r1_mix_ceiling.json (synthetic same-mix kernel)"}
    traffic_file = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(traffic_file):
        with open(traffic_file) as fh:
            roof["traffic"] = json.load(fh).get(preset.name)

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        count = args.cpu_sample or auto_sample(preset)
        v, dt, used, cores, _ = oracle_sample_run(preset, count)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{used} of {M} queries (deterministic spread), full K×Kp×N per query; "
                         f"{dt:.1f} s wall on {cores} threads"}
        # the paper's setting: one CPU core, on a proportionally smaller sample
        n1 = max(1, count // max(cores, 1))
        v1, dt1, used1, _, _ = oracle_sample_run(preset, n1, seed_offset=7, nthreads=1)
        cpu["single_core"] = {"value": v1, "unit": UNIT, "cores": 1,
                              "sample": f"{used1} queries, {dt1:.1f} s wall on 1 thread"}

    slices = world
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": preset.name, "n": preset.n, "M_per_gpu": M, "N": preset.N,
                   "K": preset.K, "Kp": preset.Kp, "system": preset.system,
                   "target": preset.target, "delta": preset.delta, "T": preset.T,
                   "parallelism": f"query-sharded x{world} (one slice per GPU, no collective)",
                   "l2": f"flushed between steps (256 MB write); inputs {x_host.nbytes // 1024} KB"},
        "s_per_slice": (total_ms / 1000.0 / args.steps) * world / slices,
        "kernel_ms_per_step": kern_avg_ms,
        "gpu_launches": 2 * args.steps,
        "roofline": roof,
        "e2e": e2e,
        "fastpath": fastpath,
        "gather": gather,
        "cpu_baseline": cpu,
        "clocks": clk,
        "paper_context": "paper: 14–26 s per 40×40 slice (N=14,000) on one CPU core (P:474)",
    }
    if PATH_CHECK:
        line["path_check"] = "all ranks on cuda:0 over gloo: functional check, not a measurement"
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
