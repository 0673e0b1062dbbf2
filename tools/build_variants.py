"""Build libhjmc variants (CTA size / min blocks per SM) into variants/ for A/B timing."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_18566_b200 import build as B  # noqa: E402

# (the warp-specialised HJMC_WS variants of an earlier revision were measured and removed)
VARIANTS = {
    "w8k": ["-DHJMC_WARP_UNIT_MAX_N=8192"],
    "w32k": ["-DHJMC_WARP_UNIT_MAX_N=32768"],
    "w0": ["-DHJMC_WARP_UNIT_MAX_N=0"],
    "q0": ["-DHJMC_WARP_UNIT_MAX_N=0", "-DHJMC_QUAD_WARP_MAX_N=0"],
    "g128": ["-DHJMC_CTA_GROUP=128"],
    "lg2": ["-DHJMC_LG_LANES=2"],
    "mb3": ["-DHJMC_MINB=3"],
    "mb4": ["-DHJMC_MINB=4"],
    "mb5": ["-DHJMC_MINB=5"],
    "mb6": ["-DHJMC_MINB=6"],
    # lane-group kernel (n = 37–48): one sample per trip (the round-1 kernel) at 4 / 3 CTAs per
    # SM, two samples per trip (the default) at 4 / 3 CTAs per SM. Measured on the C5 benchmark
    # queries (1,184, full N/K/Kp): 4500 / 4451 / 4680 / 4713 ms vs the default's 4409 ms. Round 1's
    # Philox round-1 product kept by 64-bit addition (one IMAD.WIDE fewer per lane-trip) measured
    # 4478 / 4431 ms (single / dual) and was removed.
    "single4": ["-DHJMC_LG_DUAL=0", "-DHJMC_MINB=4"],
    "single3": ["-DHJMC_LG_DUAL=0", "-DHJMC_MINB=3"],
    "dual4": ["-DHJMC_LG_DUAL=1", "-DHJMC_MINB=4"],
    "dual3": ["-DHJMC_LG_DUAL=1", "-DHJMC_MINB=3"],
    "nolg2": ["-DHJMC_NO_LANE_GROUPS=1", "-DHJMC_MINB=2"],
    "du2": ["-DHJMC_LG_DUAL_UNROLL=2"],
    "du4": ["-DHJMC_LG_DUAL_UNROLL=4"],
    # generic per-thread kernel (C4, n = 15): more samples in flight at 2 CTAs/SM
    "mb2": ["-DHJMC_MINB=2"],
    "mb2u4": ["-DHJMC_MINB=2", "-DHJMC_UNROLL=4"],
    "mb3u4": ["-DHJMC_MINB=3", "-DHJMC_UNROLL=4"],
    # Philox products' high words on the FP64 pipe (DFMA.RM, hjmc_rng.cuh), by product mask.
    # Bit-identical on C2-C5 but slower everywhere (C5 1,184 queries: base 4462 ms, df5 4643,
    # dfHi 4836, dfLo 4969, dfA 5310; profiles/r2_philox_dfma_variants.jsonl)
    # lane-group speculative kernel at 2 CTAs/SM (128 registers) instead of 3
    "spec2": ["-DHJMC_LG_SPEC_MINB=2"],
    # the scheduling tie of the lane-group dual loop (default: on, at radius 0, loop unrolled x2).
    # C5, 1,184 queries: default 4326 ms; no tie (unrolled x2) 4361; tie at radius 1/2/3/5
    # 4379/4406/4412/4417; tie without unrolling 4380, with x4 4395; the tie also from each trip
    # to the next (loop-carried) 4397; a tie between every pair of consecutive Philox blocks
    # 4886 (x2: 4810); four samples per trip with one SQRT + EX2 per lane per four samples
    # (reduce-scatter of the minima; removed) 4386 ms
    "nochain": ["-DHJMC_LG_CHAIN=0"],
    "at1": ["-DHJMC_LG_CHAIN_AT=1"],
    "at2": ["-DHJMC_LG_CHAIN_AT=2"],
    "at3": ["-DHJMC_LG_CHAIN_AT=3"],
    "at5": ["-DHJMC_LG_CHAIN_AT=5"],
    # CTA size / occupancy of the lane-group dual loop (C5, 1,184 queries; default 256 threads x 2
    # CTAs at 128 registers = 16 warps/SM: 4327 ms): 128 threads x 4 CTAs at 128 registers (16
    # warps) 4404 ms; 128 threads x 5 CTAs at 96 registers (20 warps, no spill inside the loop)
    # 4488 ms; 256 threads x 1 CTA at 170 registers (8 warps) 4709 ms. 512 threads does not build
    # (the warp-per-unit instantiation's shared memory).
    "nt128mb5": ["-DHJMC_NT=128", "-DHJMC_MINB=5"],
    "nt128mb4": ["-DHJMC_NT=128", "-DHJMC_MINB=4"],
    # (-Xptxas -O2 and --allow-expensive-optimizations=false give byte-identical SASS for the
    # lane-group kernel: nothing to measure)
    # ptxas --register-usage-level 0 / 10 (default 5): C5 4388 / 4435 ms vs 4330; C4 2470 / 2418
    # vs 2415 ms — schedule-level differences move the loop by 1-2 %
    "rul0": ["-Xptxas", "--register-usage-level=0"],
    "rul10": ["-Xptxas", "--register-usage-level=10"],
    # (measured and removed: source-order permutations of the lane-group trip — Philox blocks,
    # moment pairs and partial-min triples each ascending or descending, 7 combinations, all
    # bit-identical, every one a different ptxas schedule of the same 803 instructions: 4350,
    # 4365, 4442, 4350, 4407, 4362, 4410 ms vs the default order's 4328 ms. Schedules of this
    # loop spread over ~2.6 %, and the default is the best of the sampled ones.)
    "nt512mb1": ["-DHJMC_NT=512", "-DHJMC_MINB=1"],
    "nt256mb1": ["-DHJMC_NT=256", "-DHJMC_MINB=1"],
    "dfA": ["-DHJMC_PHILOX_DFMA_MASK=0xFFFFFu"],
    "df5": ["-DHJMC_PHILOX_DFMA_MASK=0x55555u"],
    "dfA5": ["-DHJMC_PHILOX_DFMA_MASK=0xAAAAAu"],
    "dfLo": ["-DHJMC_PHILOX_DFMA_MASK=0x003FFu"],
    "dfHi": ["-DHJMC_PHILOX_DFMA_MASK=0xFFC00u"],
}
# Also measured this round and removed from the source (same queries, same box): a software-
# pipelined dual loop (the next pair's Philox words generated in the body that transforms this
# pair) 4908 ms vs 4417 ms; a prototype draw layout with 6 normals per Philox block (3 Box–Muller
# pairs from 128 bits: 30 % fewer IMAD.WIDE) 4259 ms, pipelined 4201 ms — 4–5 %, too little to
# change the frozen sampler contract (R19) and every golden fixture for: the kernel is bound by
# the MUFU/issue co-limit, not by the wide multiplies alone. Later the same day:
# Philox's three c0-only wide multiplies computed once per lane pair and exchanged by four xor-2
# shuffles (bit-identical, 4 IMAD.WIDE fewer per lane per two samples) 4531 vs 4450 ms; the
# dual loop unrolled x2 / x4 4504 / 4619 vs 4454 ms; 2-lane groups 4473 vs 4455 ms; the
# per-thread layout at 128 registers (spilling) 4873 vs 4458 ms.
# Late round 2, after the sigma-scaled lane-group pass (4370 ms on the same queries): one
# single-sample trip first in warps 4-7 so their dual trips run half a trip out of phase with
# warps 0-3 (the loop is phased: Philox-only, then MUFU-heavy, then FP32), bit-identical:
# 4478 ms (+2.5 %), removed; single-sample trips at 3 / 4 CTAs per SM 4404 / 4392 ms, the dual
# loop at 3 CTAs per SM (spilling) 4624 ms.
# Re-entry of round 2 (HEAD kernel, 4325 ms on the same queries): cos/sin of the lane-group draws
# from a 4,096-entry shared-memory (cos, sin) table at the top 12 angle bits plus a first-order
# rotation by the remaining 11 bits (error <= 2.9e-7, MUFU.SIN/COS's own size; all 127 GPU tests
# passed with it) instead of FMUL + FMUL.RZ + MUFU.COS + MUFU.SIN: 7 instructions per pair (SHF,
# LEA, LDS.64, LOP3, 3 FFMA) for 5, MUFU 100 -> 52 per eval, loop 803 -> 856 instructions per four
# lane-samples: 4520 ms (+4.5 %); the paper's 45-D preset 10.12 -> 10.48 ms. Halving the MUFU
# load does not pay for 6 % more issue slots and the FFMAs that land on the FMA-heavy pipe:
# the loop is bound by issue and the FMA-heavy pipe (IMAD.WIDE), not by the XU pipe. Removed.

if __name__ == "__main__":
    names = sys.argv[1:] or list(VARIANTS)
    def one(name):
        out = os.path.join(ROOT, "variants", f"libhjmc_{name}.so")
        B.build(force=True, extra=VARIANTS[name], out=out,
                obj_dir=os.path.join(ROOT, "variants", "_obj_" + name))
        return out
    with ThreadPoolExecutor(3) as ex:
        for o in ex.map(one, names):
            print(o)
