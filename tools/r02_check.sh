#!/bin/bash
# Round-2 GPU check: GPU tests, smoke, default bench line (one gpurun call).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/gpu_tests.log; cat gpurun_out/smoke.log | tail -2; tail -c 3000 gpurun_out/bench.json
