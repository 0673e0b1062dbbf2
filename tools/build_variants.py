"""Build libhjmc variants (CTA size / min blocks per SM) into variants/ for A/B timing."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_18566_b200 import build as B  # noqa: E402

VARIANTS = {
    "a_ws0": ["-DHJMC_WS=0"],
    "b_ws_s4_p1": ["-DHJMC_WS=1", "-DHJMC_WS_STAGES=4", "-DHJMC_WS_SPT=1"],
    "c_ws_s8_p1": ["-DHJMC_WS=1", "-DHJMC_WS_STAGES=8", "-DHJMC_WS_SPT=1"],
    "d_ws_s2_p4": ["-DHJMC_WS=1", "-DHJMC_WS_STAGES=2", "-DHJMC_WS_SPT=4"],
    "e_ws_s6_p2": ["-DHJMC_WS=1", "-DHJMC_WS_STAGES=6", "-DHJMC_WS_SPT=2"],
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
