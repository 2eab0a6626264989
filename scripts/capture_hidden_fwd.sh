#!/bin/bash
# ncu --set full of one hidden-layer forward GEMM (1024 x 2048 x 2048, split-K CTA pairs) of a
# config-2 low-rank step. Outputs under gpurun_out/.
set -e
mkdir -p gpurun_out
ncu -f --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:\(int\)3, \(int\)1>" \
    --launch-skip 20 --launch-count 2 \
    -o gpurun_out/r2_hfwd python scripts/lr_steps.py --steps 3 --warmup 5 --bench-data > gpurun_out/r2_hfwd.log 2>&1
ncu -i gpurun_out/r2_hfwd.ncu-rep --page details > gpurun_out/r2_hfwd_details.txt
ncu -i gpurun_out/r2_hfwd.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r2_hfwd_src.csv 2>/dev/null || true
echo done
