#!/bin/bash
# GPU box: one config-4 forward (N=1024, 256ch, 56x56, Legendre 8b) under ncu --set full, every
# wl:: kernel of the forward; condensed per-kernel summary (DRAM bytes, throughput, issue, stalls)
# to gpurun_out/ncu_full_cfg4.csv.  Run only after the same command has exited 0 without ncu.
mkdir -p gpurun_out
python tools/prof_forward.py --n 1024 --iters 2 > gpurun_out/plain_cfg4.log 2>&1 || exit 1
ncu -f --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"wl::" -c 60 -o /tmp/prof_cfg4 python tools/prof_forward.py --n 1024 --iters 2 > gpurun_out/ncu_cfg4.log 2>&1
python tools/ncu_summary.py /tmp/prof_cfg4.ncu-rep gpurun_out/ncu_full_cfg4.csv > /dev/null
ncu -i /tmp/prof_cfg4.ncu-rep --page source --csv --print-source sass -k regex:sout_cw > gpurun_out/source_sout_cw.csv 2>/dev/null
ls -la gpurun_out/
