#!/bin/bash
# GPU box: the round's evidence run — GPU tests, smoke, the default bench (N=1, e2e + CPU baseline),
# the reference arm, the ncu launch list of the bench command, and one ncu --set full capture of a
# config-4 forward (per-kernel DRAM bytes / issue / tensor-pipe utilisation).
mkdir -p gpurun_out
bash tools/round_check.sh
bash tools/ncu_full_cfg4.sh > gpurun_out/ncu_full.log 2>&1
python tools/launch_table.py gpurun_out/launches.csv > gpurun_out/launch_table.txt 2>&1
tail -1 gpurun_out/launch_table.txt
