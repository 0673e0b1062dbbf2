#!/usr/bin/env python
"""Benchmark of the hot path: one step = one hjmc_solve_slice (all of Algorithm 1 — every
horizon × Picard iterate — plus the running-min tube) over the workload of BASELINE.json
configs[4] (C5: the n = 45 fifteen-pair Dubins game, N = 2^20 samples, 10 horizons × 10 Picard
iterates, fp32; the paper's 45-D scaling setting) on a deterministic constant-fraction
subset of its global query ids (inputs.bench_ids: 518 of every 256² θ-slice, 4,144 queries),
followed on N > 1 GPUs by the per-slice result gather.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c5]

Multi-GPU (torchrun, one rank per GPU, NCCL): STRONG scaling — the same fixed workload is split
by shard.partition into contiguous ranges of the subset; each rank solves its range with the
explicit global ids (the Philox counter carries them, so results are bit-identical for any
world size), then one NCCL all_gather of v, Dv, c, tube and vhist INSIDE the timed step
(north_star: the only collective). Timing: barrier + synchronize around K steps, CUDA events on
the launching stream, max over ranks. --impl reference times the CPU oracle (this tier's
reference arm) on a bounded sample of the same workload's Φ passes, rank 0 only.
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
    ap.add_argument("--config", default="c5", help="c1..c5 (default c5 = BASELINE configs[4])")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=0, help="oracle Φ passes per sample (0 = auto)")
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
def oracle_pass_items(preset, ids, x_all, count: int, offset: int = 0):
    """`count` Φ passes of the workload, deterministic: item t is the FIRST Picard pass of unit
    (query ids[(offset + 37 t) mod |ids|], horizon j = 1 + (offset + t) mod K) at its c^(0) =
    Γ(x, Dg(x)) (Algorithm 1 init) — exactly the pass the GPU executes for that unit."""
    import oracle as O

    P = O.Problem.from_preset(preset)
    sel = np.array([ids[(offset + 37 * t) % len(ids)] for t in range(count)], dtype=np.int64)
    js = np.array([1 + (offset + t) % preset.K for t in range(count)], dtype=np.uint32)
    c0 = np.array([O.gamma(P, x_all[q].astype(np.float64), O.dg(P, x_all[q].astype(np.float64)))
                   for q in sel])
    tau = js.astype(np.float64) * preset.T / preset.K
    return P, sel, js, c0, tau


def oracle_pass_sample(preset, ids, x_all, count: int, offset: int = 0, nthreads: int = 0):
    """Time the oracle, as it stands, on `count` of the workload's Φ passes (oracle_pass_items);
    nthreads = 0 uses every host core (OpenMP over passes), 1 the paper's setting.
    Returns (evals/s, seconds, passes, threads)."""
    import oracle as O

    O.build()
    P, sel, js, c0, tau = oracle_pass_items(preset, ids, x_all, count, offset)
    t0 = time.perf_counter()
    O.phi_items(P, x_all, sel, sel.astype(np.uint32), c0, tau, js, 0, nthreads=nthreads)
    dt = time.perf_counter() - t0
    return count * preset.N / dt, dt, count, (nthreads or O.max_threads())


def pass_seconds(preset) -> float:
    """Host-core seconds of one oracle Φ pass (two sweeps over N samples), modelled from the
    GPU box's host: 15.6 ms at C2 (n = 3, N = 2^16), 2.06 s at C5 (n = 45, N = 2^20)."""
    return preset.N * (1.0e-7 + 3.5e-8 * preset.n)


def auto_passes(preset, seconds: float) -> int:
    """Φ passes for ~`seconds` of wall time on all host cores (at least one per core)."""
    import oracle as O

    cores = O.max_threads()
    return int(max(cores, min(4096, round(seconds * cores / pass_seconds(preset)))))


def workload_config(preset, ids, world):
    sub = len(ids) < preset.M
    return {"workload": preset.name + (f" (subset: {len(ids)} of {preset.M} queries, "
                                       f"{len(ids) // len(preset.slices)} per "
                                       f"{preset.grid_pts}² slice, even spread)" if sub else ""),
            "n": preset.n, "M": int(len(ids)), "M_workload": preset.M, "N": preset.N,
            "K": preset.K, "Kp": preset.Kp, "slices": len(preset.slices),
            "system": preset.system, "target": preset.target, "delta": preset.delta,
            "T": preset.T}


def run_reference(args):
    from paper_2605_18566_b200 import inputs as I

    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    preset = preset_for(args.config)
    ids = I.bench_ids(preset)
    x_all = I.queries(preset)
    import oracle as O

    O.build()
    cores = O.max_threads()
    per_step = args.cpu_sample or cores                  # one Φ pass per host core per step
    for w in range(args.warmup):
        oracle_pass_sample(preset, ids, x_all, max(1, cores // 4), offset=1000 + w)
    vals, secs = [], 0.0
    for st in range(args.steps):
        v, dt, used, cores, = oracle_pass_sample(preset, ids, x_all, per_step, offset=st * per_step)
        vals.append(v)
        secs += dt
    value = args.steps * per_step * preset.N / secs
    sample = (f"{per_step} Φ passes per step of {preset.name} (each the first Picard pass of a "
              f"(query, horizon) unit of the benchmark's subset at its c^(0), N = {preset.N} "
              f"samples, n = {preset.n}), OpenMP over passes on {cores} host threads")
    cfg = workload_config(preset, ids, world)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * secs / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": cfg,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _measured_full_slice(preset):
    """A complete 2-D slice of the workload measured (not extrapolated) by
    tools/config_bench.py --full-slice, if profiles/ holds one for this preset (context beside
    the extrapolated s_per_slice; not re-measured by this run)."""
    import glob

    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_full_slice*.jsonl")), reverse=True):
        with open(path) as fh:
            for line in fh:
                try:
                    r = json.loads(line)
                except ValueError:
                    continue
                if r.get("config") == preset.name and r.get("measured_full_slice"):
                    return {"s": r["ms"] / 1000.0, "s_exact_shortcuts": r["fastpath"]["ms"] / 1000.0,
                            "source": os.path.relpath(path, ROOT)}
    return None


# ---- our arm --------------------------------------------------------------------------------
GATHER_KEYS = ("v", "dv", "c", "tube", "vhist")


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2605_18566_b200 import inputs as I
    from paper_2605_18566_b200 import roofline as RL
    from paper_2605_18566_b200 import shard
    from paper_2605_18566_b200.solver import Solver, SolverConfig

    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        if PATH_CHECK:
            dist.init_process_group("gloo")
        else:
            os.environ.setdefault("NCCL_DEBUG", "INFO")     # the driver reads nRanks from it
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    preset = preset_for(args.config)
    solver = Solver(SolverConfig.from_preset(preset, device=local))
    ids = I.bench_ids(preset)
    Mtot = int(len(ids))
    x_all = I.queries(preset)
    start, count = shard.partition(Mtot, world, rank)   # strong scaling: a fixed workload split
    x_host = np.ascontiguousarray(x_all[ids[start:start + count]])
    q_host = np.ascontiguousarray(ids[start:start + count].astype(np.int32))
    x = torch.from_numpy(x_host).to(dev)
    q = torch.from_numpy(q_host).to(dev)
    out = solver.alloc_result(count, hist=True)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def gather():
        if world > 1:
            return shard.gather_results({k: out[k] for k in GATHER_KEYS}, Mtot)
        return None

    for _ in range(args.warmup):
        flush.zero_()                        # warm everything the timed loop launches
        solver.solve_slice(x, qid=q, out=out)
        gather()
    solver.check()
    torch.cuda.synchronize(dev)

    clocks = ClockSampler(local) if not args.no_clocks else None
    E = lambda: torch.cuda.Event(enable_timing=True)
    ev = [(E(), E(), E()) for _ in range(args.steps)]
    t_start, t_end = E(), E()
    barrier()
    torch.cuda.synchronize(dev)
    if clocks:
        clocks.start()
        time.sleep(0.3)
    t_start.record(stream)
    for s in range(args.steps):
        flush.zero_()                        # L2 flush between steps (not our kernel)
        ev[s][0].record(stream)
        solver.solve_slice(x, qid=q, out=out)
        ev[s][1].record(stream)
        full = gather()                      # the per-slice result gather, inside the step
        ev[s][2].record(stream)
    t_end.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    clk = clocks.stop() if clocks else None
    solver.check()
    total_ms = t_start.elapsed_time(t_end)
    kernel_ms = [a.elapsed_time(b) for a, b, _ in ev]
    gather_ms = [b.elapsed_time(c) for _, b, c in ev]
    t = torch.tensor([total_ms, sum(kernel_ms), sum(gather_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, kern_sum, gath_sum = float(t[0]), float(t[1]), float(t[2])
    evals_step = Mtot * preset.N * preset.K * preset.Kp          # the whole job, all ranks
    evals_step_rank = count * preset.N * preset.K * preset.Kp
    value = evals_step * args.steps / (total_ms / 1000.0)
    kern_avg_ms = kern_sum / args.steps

    gather_info = None
    if world > 1:
        gather_info = {"ms_per_step": gath_sum / args.steps,
                       "collective": f"all_gather over {dist.get_backend()} (torch.distributed), "
                                     "inside the timed step",
                       "keys": list(GATHER_KEYS),
                       "bytes_per_rank": int(sum(out[k].numel() * 4 for k in GATHER_KEYS)),
                       "bytes_gathered": int(sum(t.numel() * 4 for t in full.values())),
                       "share_of_step": (gath_sum / args.steps) / (total_ms / args.steps)}

    # ---- end to end: host buffers through hjmc_solve_slice_host (copies inside the timing) ----
    pin = lambda *s: torch.empty(s, dtype=torch.float32).pin_memory()
    xh = torch.from_numpy(x_host).pin_memory()
    qh = torch.from_numpy(q_host).pin_memory()
    hout = {"v": pin(count), "dv": pin(count, preset.n), "c": pin(count), "tube": pin(count)}
    solver.solve_slice_host(xh, qid=qh, out=hout)
    e2e_steps = max(1, min(args.steps, 2))
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        solver.solve_slice_host(xh, qid=qh, out=hout)
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    e2e = {"value": evals_step * e2e_steps / float(dt[0]), "unit": UNIT,
           "h2d_bytes_per_step": int(x_host.nbytes + q_host.nbytes) * world,
           "d2h_bytes_per_step": int(sum(v.numel() * 4 for v in hout.values())) * world,
           "steps": e2e_steps,
           "api": "hjmc_solve_slice_host (pinned host buffers, synchronous; per rank, no gather)"}

    # ---- fast path: the same solve with the exact shortcuts (bit-identical outputs) ------------
    fast = Solver(SolverConfig.from_preset(preset, device=local, skip_stationary=True,
                                           reuse_passes=True, speculate=True))
    fast.solve_slice(x, qid=q, out=out)
    fast.pass_count()
    fe0, fe1 = E(), E()
    fsteps = max(1, min(args.steps, 3))
    barrier()
    fe0.record(stream)
    for _ in range(fsteps):
        fast.solve_slice(x, qid=q, out=out)
    fe1.record(stream)
    torch.cuda.synchronize(dev)
    fpasses = fast.pass_count() / fsteps
    fms = torch.tensor([fe0.elapsed_time(fe1) / fsteps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(fms, op=dist.ReduceOp.MAX)
    fastpath = {"flag": "HJMC_FLAG_SKIP_STATIONARY | HJMC_FLAG_REUSE_PASSES | "
                        "HJMC_FLAG_SPECULATE_CLAMPS", "ms_per_step": float(fms[0]),
                "passes_executed_frac": fpasses / max(1, count * preset.K * preset.Kp),
                "note": "outputs bit-identical to the full schedule (tests/test_gpu_parity.py); "
                        "the headline value counts the full K×Kp schedule without it"}

    if rank != 0:
        barrier()                                # rank 0 prints the line alone
        barrier()
        if world > 1:
            dist.destroy_process_group()
        return 0

    # ---- roofline (ALU / MUFU / IMAD pipes) ------------------------------------
    rates, rate_src = RL.load_rates()
    rl = RL.roofline(preset.n, preset.target, preset.antithetic, rates=rates)
    pipe = rl["binding_pipe"]
    ops_per_launch = rl["ops"][pipe] * evals_step_rank
    achieved = ops_per_launch / (kern_avg_ms / 1000.0) / 1e9
    peak = rl["peak_ops_per_s"] / 1e9
    lane = preset.n >= 37 and preset.target in ("pair_union", "pursuit_min")
    roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Gop/s",
            "frac": achieved / peak, "traffic": None,
            "pipe": pipe, "ops_per_eval": rl["ops"],
            "peak_basis": f"{rl['rate']:.1f} lane-ops/clk/SM × 148 SMs × 1965 MHz (sm_max); "
                          f"rates: {rate_src}",
            "kernel": f"solve_kernel<{preset.target}, n={preset.n}, 256 threads"
                      f"{', 4-lane groups' if lane else ''}> (+ tube epilogue, <0.1%)",
            "kernel_ms_avg": kern_avg_ms, "units_per_launch": int(count * preset.K),
            "evals_per_launch": int(evals_step_rank)}
    # every pipe's share of its own peak at the minimal per-eval counts (the metric names the
    # FP32/MUFU peak; the binding pipe above is the one with the largest demand)
    evals_per_s_kernel = evals_step_rank / (kern_avg_ms / 1000.0)
    roof["by_pipe"] = {k: rl["ops"][k] * evals_per_s_kernel / (rates[k] * RL.NSM * RL.F_MAX_MHZ * 1e6)
                       for k in ("imul", "mufu", "fp32", "alu", "issue")}
    if clk and clk.get("sm_mhz"):
        roof["frac_at_measured_clock"] = roof["frac"] * 1965.0 / clk["sm_mhz"]
    # the query / result streams (north_star: "achieved HBM GB/s"): per unit the kernel reads x
    # and writes, per Picard iterate, vhist + chist, and per query v, dv, c, tube, g0
    hbm_bytes = 4 * (count * preset.K * preset.n + 2 * count * preset.K * preset.Kp
                     + count * (preset.n + 4))
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
    # mix (a synthetic kernel with the same per-eval mix and no memory)
    f_hz = (clk["sm_mhz"] if clk and clk.get("sm_mhz") else RL.F_MAX_MHZ) * 1e6
    per_clk = evals_step_rank / (kern_avg_ms / 1000.0) / (RL.NSM * f_hz)
    mixes = {"c2_dubins_n3": ("r1_mix_ceiling.json", "full_c2_mix", "evals_per_clk_per_sm", 1.0),
             "c5_dubins15pairs_n45": ("r2_mix_ceiling_c5.json", "full_mix_2samples_2cta",
                                      "lane_samples_per_clk_per_sm", 4.0)}
    if preset.name in mixes:
        fname, key, field, lanes = mixes[preset.name]
        mix_file = os.path.join(ROOT, "profiles", fname)
        if os.path.exists(mix_file):
            with open(mix_file) as fh:
                mix = json.load(fh)["mixes"][key][field] / lanes
            roof["mix_ceiling"] = {"evals_per_clk_per_sm": mix,
                                   "kernel_evals_per_clk_per_sm": per_clk, "frac": per_clk / mix,
                                   "source": f"profiles/{fname} (synthetic same-mix kernel)"}
    traffic_file = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(traffic_file):
        with open(traffic_file) as fh:
            tr = json.load(fh).get(preset.name)
        # stored per unit ((query, horizon) CTA) of the captured launch; scale to this launch
        if isinstance(tr, dict) and "bytes_per_unit" in tr:
            roof["traffic"] = tr["bytes_per_unit"] * count * preset.K
            roof["traffic_source"] = tr.get("source")
        elif isinstance(tr, (int, float)):
            roof["traffic"] = tr

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cnt = args.cpu_sample or auto_passes(preset, 20.0)
        v, dt, used, cores = oracle_pass_sample(preset, ids, x_all, cnt)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{used} Φ passes of the workload (the first Picard pass of sampled "
                         f"(query, horizon) units at c^(0), N = {preset.N} each), OpenMP over "
                         f"passes; {dt:.1f} s wall on {cores} threads"}
        n1 = max(1, round(8.0 / pass_seconds(preset)))
        v1, dt1, used1, _ = oracle_pass_sample(preset, ids, x_all, n1, offset=7, nthreads=1)
        cpu["single_core"] = {"value": v1, "unit": UNIT, "cores": 1,
                              "sample": f"{used1} Φ passes, {dt1:.1f} s wall on 1 thread"}

    step_s = total_ms / 1000.0 / args.steps
    per_slice_q = preset.grid_pts * preset.grid_pts
    cfg = workload_config(preset, ids, world)
    cfg.update({"parallelism": f"query-sharded x{world} (strong scaling: the fixed workload split "
                              "by shard.partition; one all_gather of the results per step)",
                "l2": f"flushed between steps (256 MB write); inputs {x_host.nbytes // 1024} KB "
                      "per rank"})
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": cfg,
        "s_per_slice": step_s * per_slice_q / Mtot,
        "s_per_slice_basis": (f"extrapolated: step time × {per_slice_q} queries per slice / {Mtot} "
                              "queries per step (per-query work is fixed)"
                              if Mtot != per_slice_q else "measured: one slice per step"),
        "s_per_slice_measured": _measured_full_slice(preset),
        "kernel_ms_per_step": kern_avg_ms,
        "gpu_launches": 2 * args.steps,
        "roofline": roof,
        "e2e": e2e,
        "fastpath": fastpath,
        "gather": gather_info,
        "cpu_baseline": cpu,
        "clocks": clk,
        "paper_context": "paper: 14–26 s per 40×40 slice (N=14,000) on one CPU core (P:474); "
                         "45-D runs 27.6–30 s on a 16-core CPU (P:405–420)",
    }
    if PATH_CHECK:
        line["path_check"] = "all ranks on cuda:0 over gloo: functional check, not a measurement"
        if world > 1:
            # the gathered strong-scaling result must equal ONE rank solving the whole workload
            # bit for bit (global ids key the samples; "fully parallelizable")
            one = solver.solve_slice(torch.from_numpy(np.ascontiguousarray(x_all[ids])).to(dev),
                                     qid=torch.from_numpy(ids.astype(np.int32)).to(dev))
            line["path_check_bit_identical"] = {k: bool(torch.equal(one[k], full[k]))
                                                for k in GATHER_KEYS}
    barrier()
    print(json.dumps(line), flush=True)
    barrier()
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
