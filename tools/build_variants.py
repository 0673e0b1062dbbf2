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
