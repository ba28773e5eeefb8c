#!/bin/bash
# GPU box: ncu --set full + SASS source page of the kernels matching $1 (regex, first $2 launches) in a
# config-4-shaped forward at batch $3; writes gpurun_out/src_$4.csv and the summary row.
RX=$1; C=${2:-1}; N=${3:-256}; TAG=${4:-k}
mkdir -p gpurun_out
python tools/prof_forward.py --n $N --iters 1 > gpurun_out/plain_$TAG.log 2>&1 || exit 1
ncu -f --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$RX" -c $C \
    -o /tmp/src_$TAG python tools/prof_forward.py --n $N --iters 1 > gpurun_out/ncu_$TAG.log 2>&1
ncu -i /tmp/src_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$TAG.csv 2>/dev/null
python tools/ncu_summary.py /tmp/src_$TAG.ncu-rep gpurun_out/sum_$TAG.csv > /dev/null
