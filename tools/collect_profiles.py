"""Copy one refresh's gpurun_out/ artifacts (tools/refresh_profiles_r2c.sh) into profiles/ under
its tag: bench line, reference arm, launch list + per-kernel shares, ncu summaries/hotspots, the
config table, GPU-test and smoke summaries, and the C5 DRAM traffic per unit
(profiles/ncu_traffic.json, read by bench.py). Usage: python tools/collect_profiles.py r2c"""
import collections
import csv
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")


def cp(src, dst):
    if os.path.exists(os.path.join(G, src)):
        shutil.copy(os.path.join(G, src), os.path.join(P, dst))
        return True
    return False


def launches(tag):
    rows = list(csv.reader(open(os.path.join(G, f"{tag}_launches.csv"))))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            agg[r[ki]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out = ["ncu --metrics gpu__time_duration.sum --clock-control none  python bench.py --steps 2 "
           "--warmup 3 --no-cpu-baseline --no-clocks   (C5 subset, the benchmark workload)",
           "(cold-cache, serialised per-launch times in ns; compare shares, not absolutes)", ""]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"{k[:78]:78s} launches {len(v):3d}  avg {sum(v)/len(v):16.1f} ns  "
                   f"share {100*sum(v)/tot:7.3f}%")
    open(os.path.join(P, f"{tag}_launches_c5_summary.txt"), "w").write("\n".join(out) + "\n")


def traffic(tag):
    path = os.path.join(G, f"{tag}_c5_bench_launch_raw.csv")
    rows = list(csv.reader(open(path)))
    h, u, d = rows[0], dict(zip(rows[0], rows[1])), dict(zip(rows[0], rows[2]))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    val = lambda k: float(d[k].replace(",", "")) * scale.get(u[k], 1)
    tr = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
    units = 4144 * 10
    p = os.path.join(P, "ncu_traffic.json")
    j = json.load(open(p))
    j["c5_dubins15pairs_n45"] = {
        "bytes_per_unit": tr / units, "bytes_per_launch": int(tr),
        "source": f"profiles/{tag}_ncu_c5_bench_launch.txt: dram__bytes_read.sum + "
                  "dram__bytes_write.sum of the benchmark launch (4,144 queries x 10 horizons, "
                  "Kp = 10)",
        "note": "thread 0's double-precision v/Dv/Γ epilogue (n = 45 arrays in a local-memory "
                "stack frame that L2 later evicts) and the per-iterate results; not the sample "
                "loop, which touches no memory"}
    json.dump(j, open(p, "w"), indent=1)
    return tr


if __name__ == "__main__":
    tag = sys.argv[1] if len(sys.argv) > 1 else "r2c"
    cp(f"{tag}_bench.jsonl", f"{tag}_bench_c5.jsonl")
    cp(f"{tag}_ref.jsonl", f"{tag}_bench_reference_arm.jsonl")
    cp(f"{tag}_launches.csv", f"{tag}_launches_c5.csv")
    launches(tag)
    cp(f"{tag}_c5_summary.txt", f"{tag}_ncu_full_c5_reduced_solve_kernel.txt")
    cp(f"{tag}_c5_hotspots.txt", f"{tag}_ncu_hotspots_c5.txt")
    cp(f"{tag}_c5_bench_launch_summary.txt", f"{tag}_ncu_c5_bench_launch.txt")
    cp(f"{tag}_c5_bench_launch_raw.csv", f"{tag}_ncu_details_c5_bench_launch.csv")
    cp(f"{tag}_smoke.txt", f"{tag}_smoke.txt")
    lines = [l for l in open(os.path.join(G, f"{tag}_configs.jsonl")) if l.startswith("{")]
    open(os.path.join(P, f"{tag}_configs_all.jsonl"), "w").writelines(lines)
    log = open(os.path.join(G, f"{tag}_gpu_tests.log")).read().splitlines()
    keep = [l for l in log if ("R27" in l and " 0 of " not in l) or "passed" in l or "failed" in l
            or "pytest rc" in l or "SKIPPED" in l]
    open(os.path.join(P, f"{tag}_gpu_tests_summary.txt"), "w").write("\n".join(keep) + "\n")
    print("traffic bytes per launch", traffic(tag))
