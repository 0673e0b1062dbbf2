#!/bin/bash
# ncu --set full of the C5 lane-group solve kernel (reduced K = Kp = 1 launch of the benchmark's
# queries) for the in-tree library and each named variant; summaries into gpurun_out/.
# Usage (on the GPU box): bash scripts/ncu_variants.sh <queries> [variant ...]
set -u
Q=${1:-2368}; shift
mkdir -p gpurun_out
for v in base "$@"; do
  lib=paper_2605_18566_b200/libhjmc.so
  [ "$v" != base ] && lib=variants/libhjmc_$v.so
  ncu --set full --clock-control none --import-source on -k regex:solve_kernel -c 1 \
      -o gpurun_out/ncu_c5_$v -f python tools/ncu_one.py c5 $Q 1 1 --lib $lib > gpurun_out/ncu_c5_$v.log 2>&1
  ncu -i gpurun_out/ncu_c5_$v.ncu-rep --page raw --csv > gpurun_out/ncu_c5_$v.raw.csv 2>/dev/null
  python tools/ncu_summary.py gpurun_out/ncu_c5_$v.raw.csv > gpurun_out/ncu_c5_$v.summary.txt 2>&1
done
