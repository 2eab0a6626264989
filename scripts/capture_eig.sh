#!/bin/bash
# ncu --set full of one output-layer (R = 80) background eigensolve of a config-2 low-rank run.
set -e
mkdir -p gpurun_out
ncu -f --set full --import-source on --clock-control none -k regex:lr_eig_kernel --launch-skip 27 --launch-count 1 \
    -o gpurun_out/r2_eig python scripts/lr_steps.py --steps 8 --warmup 5 --bench-data > gpurun_out/r2_eig.log 2>&1
ncu -i gpurun_out/r2_eig.ncu-rep --page details > gpurun_out/r2_eig_details.txt
ncu -i gpurun_out/r2_eig.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r2_eig_src.csv 2>/dev/null || true
echo done
