#!/usr/bin/env bash
# Round-2 measurement evidence under profiles/ (tag $1, default r2), the headline now on C5:
#   on the GPU box (one gpurun call): the bench line (C5 subset, 1 GPU), the reference arm, the
#   ncu launch list of the bench command, `ncu --set full` of the EXACT benchmark launch (C5
#   subset, K = Kp = 10) and of reduced launches of C2–C4 and the paper's 45-D preset, the config
#   table; here: summaries, hotspots, launch shares and DRAM traffic per unit (ncu_traffic.json).
# Numbers printed under ncu are never bench values; each ncu run follows its plain run.
set -euo pipefail
tag=${1:-r2}
cd "$(dirname "$0")/.."
GPURUN=/usr/local/graft/bin/gpurun
$GPURUN --timeout 3600 -- "
mkdir -p gpurun_out
python bench.py > gpurun_out/${tag}_bench.jsonl 2> gpurun_out/${tag}_bench.err &&
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_ref.jsonl 2>/dev/null &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-clocks > /dev/null 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:solve_kernel -c 1 -f \
    -o gpurun_out/${tag}_c5 python tools/ncu_one.py c5 4144 10 10 > /dev/null 2>&1 &&
for c in 'c2 10201 10 8' 'c3 4096 1 1' 'c4 2048 1 1'; do
  set -- \$c
  ncu --set full --clock-control none --import-source on -k regex:solve_kernel -c 1 -f \
      -o gpurun_out/${tag}_\$1 python tools/ncu_one.py \$c > /dev/null 2>&1
done &&
python tools/config_bench.py c1 c2 c3 c4 c5 paper_dubins_40x40 paper_rockets3_40x40 \
    paper_double_integrator paper_multiagent45 > gpurun_out/${tag}_configs.jsonl 2>&1
"
cp gpurun_out/${tag}_bench.jsonl profiles/${tag}_bench_c5.jsonl
cp gpurun_out/${tag}_ref.jsonl profiles/${tag}_bench_reference_arm.jsonl
cp gpurun_out/${tag}_launches.csv profiles/${tag}_launches_c5.csv
grep '^{' gpurun_out/${tag}_configs.jsonl > profiles/${tag}_configs_all.jsonl
for c in c2 c3 c4 c5; do
  ncu -i gpurun_out/${tag}_$c.ncu-rep --page raw --csv > gpurun_out/${tag}_${c}_raw.csv
  python tools/ncu_summary.py gpurun_out/${tag}_${c}_raw.csv > profiles/${tag}_ncu_full_${c}_solve_kernel.txt
done
cp gpurun_out/${tag}_c5_raw.csv profiles/${tag}_ncu_details_c5.csv
ncu -i gpurun_out/${tag}_c5.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_c5_src.csv
{ echo "# C5 (bench launch) solve_kernel stall-sample hotspots by SASS opcode"; python tools/ncu_hotspots.py gpurun_out/${tag}_c5_src.csv; } \
    > profiles/${tag}_ncu_hotspots_c5.txt
python - "$tag" <<'PY'
import collections, csv, json, sys
tag = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/{tag}_launches.csv")))
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
open(f"profiles/{tag}_launches_c5_summary.txt", "w").write("\n".join(out) + "\n")
rows = list(csv.reader(open(f"gpurun_out/{tag}_c5_raw.csv")))
h, u, d = rows[0], dict(zip(rows[0], rows[1])), dict(zip(rows[0], rows[2]))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
val = lambda k: float(d[k].replace(",", "")) * scale.get(u[k], 1)
p = "profiles/ncu_traffic.json"
j = json.load(open(p))
units = 4144 * 10
tr = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
j["c5_dubins15pairs_n45"] = {"bytes_per_unit": tr / units, "bytes_per_launch": int(tr),
                             "source": f"profiles/{tag}_ncu_full_c5_solve_kernel.txt: the benchmark "
                                       "launch (4,144 queries x 10 horizons, Kp = 10), ncu --set full"}
json.dump(j, open(p, "w"), indent=1)
print("\n".join(out))
PY
echo "profiles refreshed for tag ${tag}"
