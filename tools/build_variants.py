"""Build libhjmc variants (CTA size / min blocks per SM) into variants/ for A/B timing."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_18566_b200 import build as B  # noqa: E402

VARIANTS = {
    "nt256_mb1": ["-DHJMC_NT=256", "-DHJMC_MINB=1"],
    "nt256_mb3": ["-DHJMC_NT=256", "-DHJMC_MINB=3"],
    "nt256_mb4": ["-DHJMC_NT=256", "-DHJMC_MINB=4"],
    "nt128_mb8": ["-DHJMC_NT=128", "-DHJMC_MINB=8"],
    "nt512_mb2": ["-DHJMC_NT=512", "-DHJMC_MINB=2"],
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(VARIANTS)
    def one(name):
        out = os.path.join(ROOT, "variants", f"libhjmc_{name}.so")
        B.build(force=True, extra=VARIANTS[name], out=out,
                obj_dir=os.path.join(ROOT, "variants", "_obj_" + name))
        return out
    with ThreadPoolExecutor(2) as ex:
        for o in ex.map(one, names):
            print(o)
