"""Build libhjmc variants (CTA size / min blocks per SM) into variants/ for A/B timing."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_18566_b200 import build as B  # noqa: E402

# (the warp-specialised HJMC_WS variants of an earlier revision were measured and removed)
VARIANTS = {
    "lgu1": ["-DHJMC_LG_UNROLL=1"],
    "lgu2": ["-DHJMC_LG_UNROLL=2"],
    "mb3": ["-DHJMC_MINB=3"],
    "mb4": ["-DHJMC_MINB=4"],
    "lg4": ["-DHJMC_LG_LANES=4"],
    "lg2": ["-DHJMC_LG_LANES=2"],
    "gu1": ["-DHJMC_GROUP_UNROLL=1"],
    "gu2": ["-DHJMC_GROUP_UNROLL=2"],
    "wu0": ["-DHJMC_WARP_UNIT_MAX_N=0"],
    "wu64k": ["-DHJMC_WARP_UNIT_MAX_N=65536"],
    "wuall": ["-DHJMC_WARP_UNIT_MAX_N=4294967295u"],
    "wumin0": ["-DHJMC_WARP_UNIT_MIN_WARPS_PER_SM=0"],
    "wumin16": ["-DHJMC_WARP_UNIT_MIN_WARPS_PER_SM=16"],
}

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
