"""Build libhjmc variants (CTA size / min blocks per SM) into variants/ for A/B timing."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_18566_b200 import build as B  # noqa: E402

VARIANTS = {
    "a_base": [],
    "b_swp": ["-DHJMC_SWP=1"],
    "c_unroll1": ["-DHJMC_UNROLL=1"],
    "d_unroll4": ["-DHJMC_UNROLL=4"],
    "e_mb5": ["-DHJMC_MINB=5"],
    "f_swp_mb5": ["-DHJMC_SWP=1", "-DHJMC_MINB=5"],
    "g_nt128": ["-DHJMC_NT=128", "-DHJMC_MINB=8"],
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
