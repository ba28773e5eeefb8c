#!/bin/bash
# Round-2 profile evidence (GPU box, one gpurun call): the bench command's ncu launch list, one
# config-4 forward under ncu --set full (per-kernel summary), and SASS source pages of the two
# heaviest kernels.  Each ncu run only after the same command exited 0 without ncu.
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/p_bench.json 2> gpurun_out/p_bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/p_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/p_ncu_launch.log 2>&1
python tools/prof_forward.py --n 1024 --iters 2 > gpurun_out/p_plain_cfg4.log 2>&1 || exit 1
ncu -f --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"wl::" -c 70 -o /tmp/prof_cfg4 python tools/prof_forward.py --n 1024 --iters 2 > gpurun_out/p_ncu_cfg4.log 2>&1
python tools/ncu_summary.py /tmp/prof_cfg4.ncu-rep gpurun_out/p_ncu_full_cfg4.csv > /dev/null
ncu -i /tmp/prof_cfg4.ncu-rep --page source --csv --print-source sass -k regex:sout_ct -c 1 > gpurun_out/p_src_sout_ct.csv 2>/dev/null
ncu -i /tmp/prof_cfg4.ncu-rep --page source --csv --print-source sass -k regex:EpiHadRq -c 1 > gpurun_out/p_src_rq.csv 2>/dev/null
ncu -i /tmp/prof_cfg4.ncu-rep --page raw --csv -k regex:EpiHadRq -c 1 > gpurun_out/p_raw_rq.csv 2>/dev/null
ncu -i /tmp/prof_cfg4.ncu-rep --page raw --csv -k regex:sout_ct -c 1 > gpurun_out/p_raw_sout_ct.csv 2>/dev/null
ls -la gpurun_out/ | tail -20
