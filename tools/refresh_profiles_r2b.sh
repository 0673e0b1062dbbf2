#!/usr/bin/env bash
# Second half of the round-2 evidence (the first call's `--set full` of the 15.6 s benchmark
# launch ran past its one-hour limit: full-set replays with source-counter patching of a launch
# that long are impractical). Here: `--set full` of reduced launches (C2 complete, C3–C5 at
# K = Kp = 1 on the benchmark's queries) for source-level hotspots, the config table, and the
# EXACT benchmark launch (C5 subset, K = Kp = 10) with the hardware-counter sections only
# (no SASS patching) plus the DRAM byte counters — the traffic and pipe evidence of that launch.
# Reports are reduced to CSV pages and summaries ON the box (gpurun returns ≤ 64 MiB).
set -euo pipefail
tag=${1:-r2}
cd "$(dirname "$0")/.."
GPURUN=/usr/local/graft/bin/gpurun
$GPURUN --timeout 2700 -- "
mkdir -p gpurun_out
reduce() {  # \$1 = report stem: raw page CSV, summary, SASS source page, hotspots; drop the report
  ncu -i gpurun_out/\$1.ncu-rep --page raw --csv > gpurun_out/\$1_raw.csv 2>/dev/null || true
  python tools/ncu_summary.py gpurun_out/\$1_raw.csv > gpurun_out/\$1_summary.txt 2>&1 || true
  ncu -i gpurun_out/\$1.ncu-rep --page source --csv --print-source sass > gpurun_out/\$1_src.csv 2>/dev/null || true
  python tools/ncu_hotspots.py gpurun_out/\$1_src.csv > gpurun_out/\$1_hotspots.txt 2>&1 || true
  rm -f gpurun_out/\$1.ncu-rep gpurun_out/\$1_src.csv
}
for c in 'c2 10201 10 8' 'c3 4096 1 1' 'c4 2048 1 1' 'c5 4144 1 1'; do
  set -- \$c
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:solve_kernel -c 1 -f \
      -o gpurun_out/${tag}_\$1 python tools/ncu_one.py \$c > /dev/null 2>&1 || true
  reduce ${tag}_\$1
done
timeout 900 python tools/config_bench.py c1 c2 c3 c4 c5 paper_dubins_40x40 paper_rockets3_40x40 \
    paper_double_integrator paper_multiagent45 > gpurun_out/${tag}_configs.jsonl 2>&1 || true
timeout 1000 ncu --clock-control none -k regex:solve_kernel -c 1 -f \
    --section SpeedOfLight --section ComputeWorkloadAnalysis --section LaunchStats \
    --section Occupancy --section SchedulerStats --section WarpStateStats \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum \
    -o gpurun_out/${tag}_c5_bench_launch python tools/ncu_one.py c5 4144 10 10 > gpurun_out/${tag}_c5_bench_launch.log 2>&1 || true
reduce ${tag}_c5_bench_launch
du -sh gpurun_out; ls -la gpurun_out
"
