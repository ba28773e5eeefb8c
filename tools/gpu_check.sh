#!/bin/bash
# GPU box: parity tests + a short bench (kernel split).  Usage: tools/gpu_check.sh [pytest -k expr]
mkdir -p gpurun_out
if [ -n "$1" ]; then K="-k $1"; fi
timeout 900 python -m pytest tests -m gpu -x -q $K > gpurun_out/gpu_tests.log 2>&1
echo "tests_exit=$?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench_exit=$?"
python - <<'P'
import json
try:
    d = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
    print("ms_per_step", round(d["ms_per_step"], 3), "value", round(d["value"]))
    print(json.dumps(d["kernel_ms"]))
except Exception as e:
    print("bench parse failed", e); print(open("gpurun_out/bench.err").read()[-2000:])
P
