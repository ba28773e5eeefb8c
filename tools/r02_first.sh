#!/bin/bash
# Round-2 re-entry check: GPU tests, smoke, default bench line, chunk sweep (one gpurun call).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python tools/chunk_sweep.py 1024 128 64 32 16 8 > gpurun_out/chunk_sweep.log 2>&1
tail -3 gpurun_out/gpu_tests.log; tail -2 gpurun_out/smoke.log; tail -c 2500 gpurun_out/bench.json; cat gpurun_out/chunk_sweep.log
