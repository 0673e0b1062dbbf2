#!/usr/bin/env bash
# Final round-2 evidence (tag $1, default r2d): the r2c set plus a complete C5 slice; ONE gpurun
# call: the whole GPU test suite, smoke(), the bench line (C5 subset, 1 GPU), the reference arm,
# the ncu launch list of the bench command, `ncu --set full` of a reduced C5 launch (K = Kp = 1
# on the benchmark's queries: source-level hotspots), the EXACT benchmark launch with the
# hardware-counter sections only (pipes, issue, stalls, DRAM bytes), and the config table.
# Numbers printed under ncu are never bench values; each ncu run follows its plain run.
# Reports are reduced to CSV pages and summaries ON the box (gpurun returns <= 64 MiB).
set -uo pipefail
tag=${1:-r2d}
cd "$(dirname "$0")/.."
GPURUN=/usr/local/graft/bin/gpurun
$GPURUN --timeout 5400 -- "
mkdir -p gpurun_out
reduce() {
  ncu -i gpurun_out/\$1.ncu-rep --page raw --csv > gpurun_out/\$1_raw.csv 2>/dev/null || true
  python tools/ncu_summary.py gpurun_out/\$1_raw.csv > gpurun_out/\$1_summary.txt 2>&1 || true
  ncu -i gpurun_out/\$1.ncu-rep --page source --csv --print-source sass > gpurun_out/\$1_src.csv 2>/dev/null || true
  python tools/ncu_hotspots.py gpurun_out/\$1_src.csv > gpurun_out/\$1_hotspots.txt 2>&1 || true
  rm -f gpurun_out/\$1.ncu-rep gpurun_out/\$1_src.csv
}
timeout 1800 python -m pytest tests -m gpu -q -rs > gpurun_out/${tag}_gpu_tests.log 2>&1; echo \"pytest rc \$?\" >> gpurun_out/${tag}_gpu_tests.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/${tag}_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/${tag}_bench.jsonl 2> gpurun_out/${tag}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_ref.jsonl 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-clocks > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:solve_kernel -c 1 -f \
    -o gpurun_out/${tag}_c5 python tools/ncu_one.py c5 4144 1 1 > /dev/null 2>&1
reduce ${tag}_c5
timeout 900 python tools/config_bench.py c1 c2 c3 c4 c5 paper_dubins_40x40 paper_rockets3_40x40 \
    paper_double_integrator paper_multiagent45 > gpurun_out/${tag}_configs.jsonl 2>&1
timeout 1200 ncu --clock-control none -k regex:solve_kernel -c 1 -f \
    --section SpeedOfLight --section ComputeWorkloadAnalysis --section LaunchStats \
    --section Occupancy --section SchedulerStats --section WarpStateStats \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum \
    -o gpurun_out/${tag}_c5_bench_launch python tools/ncu_one.py c5 4144 10 10 > gpurun_out/${tag}_c5_bench_launch.log 2>&1
reduce ${tag}_c5_bench_launch
timeout 900 python tools/config_bench.py --full-slice c5 > gpurun_out/${tag}_full_slice_c5.jsonl 2>&1
du -sh gpurun_out; ls gpurun_out | grep ${tag}
"
