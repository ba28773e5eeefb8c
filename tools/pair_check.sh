#!/bin/bash
# GPU box: parity tests with the two-channel (f32x2) transform kernels, then the config-4 kernel
# split with and without them (WL_NO_PAIR=1 selects the one-channel kernels).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
echo "tests_exit=$?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
for v in pair nopair; do
  if [ $v = nopair ]; then export WL_NO_PAIR=1; else unset WL_NO_PAIR; fi
  timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err
  python - $v <<'P'
import json, sys
v = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/bench_{v}.json").read().strip().splitlines()[-1])
    print(v, "ms_per_step", round(d["ms_per_step"], 3), json.dumps(d["kernel_ms"]))
except Exception as e:
    print(v, "bench parse failed", e); print(open(f"gpurun_out/bench_{v}.err").read()[-2000:])
P
done
