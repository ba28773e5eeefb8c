#!/bin/bash
# GPU box: the round's evidence run — GPU tests, smoke, default bench (N=1, e2e + CPU baseline), the
# reference arm, the ncu launch list of the same bench command, the config-5 training bench, and the
# ncu --set full capture of one config-4 forward (tools/ncu_full_cfg4.sh).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "tests_exit=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke_exit=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench_exit=$?" >> gpurun_out/bench_full.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python bench.py --workload train > gpurun_out/bench_train.json 2> gpurun_out/bench_train.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
bash tools/ncu_full_cfg4.sh > /dev/null 2>&1
tail -2 gpurun_out/gpu_tests.log; tail -1 gpurun_out/smoke.log; tail -1 gpurun_out/bench_full.json | cut -c1-400
