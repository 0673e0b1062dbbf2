#!/usr/bin/env bash
# Refresh the measurement evidence under profiles/ for round tag $1 (default r1):
#   1. on the GPU box (through gpurun): bench line, reference arm, ncu launch list of the bench
#      command, one `ncu --set full` capture per config kernel, the config table, the
#      instruction-mix ceiling;
#   2. here: ncu raw/source pages -> summaries (tools/ncu_summary.py, tools/ncu_hotspots.py),
#      launch shares, DRAM traffic per C2 launch (profiles/ncu_traffic.json).
# Numbers printed under ncu are never bench values; each ncu run follows its plain run.
set -euo pipefail
tag=${1:-r1}
cd "$(dirname "$0")/.."
GPURUN=/usr/local/graft/bin/gpurun
$GPURUN --timeout 2400 -- "
python bench.py > gpurun_out/${tag}_bench.jsonl 2> gpurun_out/${tag}_bench.err &&
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${tag}_ref.jsonl 2>/dev/null &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-clocks > /dev/null 2>&1 &&
for c in 'c2 10201 10 8' 'c3 4096 1 1' 'c4 2048 1 1' 'c5 1184 1 1'; do
  set -- \$c
  ncu --set full --clock-control none --import-source on -k regex:solve_kernel -c 1 -f \
      -o gpurun_out/${tag}_\$1 python tools/ncu_one.py \$c > /dev/null 2>&1
done &&
python tools/config_bench.py c1 c2 c3 c4 c5 paper_dubins_40x40 paper_rockets3_40x40 \
    paper_double_integrator paper_multiagent45 > gpurun_out/${tag}_configs.jsonl 2>&1 &&
tools/mix_ceiling > gpurun_out/${tag}_mix.json 2>&1 || nvcc -gencode arch=compute_100a,code=sm_100a \
    -O3 -o tools/mix_ceiling tools/mix_ceiling.cu && tools/mix_ceiling > gpurun_out/${tag}_mix.json
"
cp gpurun_out/${tag}_bench.jsonl profiles/${tag}_bench_c2.jsonl
cp gpurun_out/${tag}_ref.jsonl profiles/${tag}_bench_reference_arm.jsonl
cp gpurun_out/${tag}_launches.csv profiles/${tag}_launches_c2.csv
grep '^{' gpurun_out/${tag}_configs.jsonl > profiles/${tag}_configs_all.jsonl
for c in c2 c3 c4 c5; do
  ncu -i gpurun_out/${tag}_$c.ncu-rep --page raw --csv > gpurun_out/${tag}_${c}_raw.csv
  python tools/ncu_summary.py gpurun_out/${tag}_${c}_raw.csv > profiles/${tag}_ncu_full_${c}_solve_kernel.txt
done
cp gpurun_out/${tag}_c2_raw.csv profiles/${tag}_ncu_details_c2.csv
ncu -i gpurun_out/${tag}_c2.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_c2_src.csv
{ echo "# C2 solve_kernel stall-sample hotspots by SASS opcode"; python tools/ncu_hotspots.py gpurun_out/${tag}_c2_src.csv; } \
    > profiles/${tag}_ncu_hotspots_c2.txt
python - "$tag" <<'EOF'
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
       "--warmup 3 --no-cpu-baseline --no-clocks",
       "(cold-cache, serialised per-launch times in ns; compare shares, not absolutes)", ""]
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    out.append(f"{k[:78]:78s} launches {len(v):3d}  avg {sum(v)/len(v):14.1f} ns  "
               f"share {100*sum(v)/tot:7.3f}%")
open(f"profiles/{tag}_launches_c2_summary.txt", "w").write("\n".join(out) + "\n")
rows = list(csv.reader(open(f"gpurun_out/{tag}_c2_raw.csv")))
h, u, d = rows[0], dict(zip(rows[0], rows[1])), dict(zip(rows[0], rows[2]))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
val = lambda k: float(d[k].replace(",", "")) * scale.get(u[k], 1)
p = "profiles/ncu_traffic.json"
j = json.load(open(p))
j["c2_dubins_n3"] = int(val("dram__bytes_read.sum") + val("dram__bytes_write.sum"))
json.dump(j, open(p, "w"), indent=1)
print("\n".join(out))
EOF
echo "profiles refreshed for tag ${tag}"
