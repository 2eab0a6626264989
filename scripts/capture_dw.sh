#!/bin/bash
# ncu --set full of the grouped dW + SGD GEMM (NP = 8) of one config-2 low-rank step.
# Outputs under gpurun_out/: the report, raw metrics, per-source-line stalls.
set -e
mkdir -p gpurun_out
ncu -f --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:\(int\)1, \(int\)8>" --launch-skip 4 --launch-count 1 \
    -o gpurun_out/r2_dw_group python scripts/lr_steps.py --steps 3 --warmup 5 > gpurun_out/r2_dw_group.log 2>&1
ncu -i gpurun_out/r2_dw_group.ncu-rep --page details --csv > gpurun_out/r2_dw_group_details.csv
ncu -i gpurun_out/r2_dw_group.ncu-rep --page raw --csv > gpurun_out/r2_dw_group_raw.csv
ncu -i gpurun_out/r2_dw_group.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_dw_group_sass.csv 2>/dev/null || true
echo done
