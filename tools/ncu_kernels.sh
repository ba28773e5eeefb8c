#!/bin/bash
# GPU box: ncu --set full of the kernels matching $1 (regex) in one N=$2 forward; writes the
# details page and the condensed summary to gpurun_out/ (the .ncu-rep stays in /tmp: too large).
RX=${1:-gemm}; N=${2:-256}; TAG=${3:-k}
python tools/prof_forward.py --n $N --iters 1 > gpurun_out/plain_$TAG.log 2>&1 || exit 1
ncu -f --set full --clock-control none --import-source on -k regex:"$RX" -c 6 -o /tmp/prof_$TAG \
    python tools/prof_forward.py --n $N --iters 1 > gpurun_out/ncu_$TAG.log 2>&1
ncu -i /tmp/prof_$TAG.ncu-rep --page details > gpurun_out/details_$TAG.txt 2>&1
python tools/ncu_summary.py /tmp/prof_$TAG.ncu-rep gpurun_out/summary_$TAG.csv > /dev/null
ncu -i /tmp/prof_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/source_$TAG.csv 2>/dev/null
ls -la gpurun_out/*_$TAG*
