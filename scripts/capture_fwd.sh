#!/bin/bash
# ncu --set full of the GEMMs of one config-2 low-rank step (the forward ones are the roofline
# kernel of bench.py), located by a launch-list pass. Outputs under gpurun_out/.
set -e
mkdir -p gpurun_out
ncu -f --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/ll.csv \
    python scripts/lr_steps.py --steps 1 --warmup 3 > /dev/null 2>&1
SKIP=$(python - <<'PY'
import csv
rows=[r for r in csv.reader(open('/tmp/ll.csv'))]
hdr=next(i for i,r in enumerate(rows) if r and r[0]=='ID')
names=[r[rows[hdr].index('Kernel Name')] for r in rows[hdr+1:] if len(r)==len(rows[hdr])]
# unique kernel launches in order (one metric row per launch)
g=[i for i,n in enumerate(names) if n.startswith('gather_kernel') or 'gather_kernel' in n]
last=g[-1]
# gemm launches before the last step's gather
print(sum(1 for n in names[:last] if 'gemm_tc_kernel' in n))
PY
)
echo "skip $SKIP gemm launches"
ncu -f --set full --import-source on --clock-control none -k regex:gemm_tc_kernel --launch-skip $SKIP --launch-count 36 \
    -o /tmp/fwd python scripts/lr_steps.py --steps 3 --warmup 3 > /dev/null 2>&1
ncu -i /tmp/fwd.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__grid_size,sm__throughput.avg.pct_of_peak_sustained_elapsed > gpurun_out/r2_fwd_raw.csv
ncu -i /tmp/fwd.ncu-rep --page details --csv > gpurun_out/r2_fwd_details.csv
echo done
