#!/bin/bash
# GPU box: parity tests, then the config-4 kernel split for each variant given as ENV=VALUE
# arguments ("base" = no extra environment).  Usage: tools/ab_check.sh base WL_NO_PAIR=1 ...
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
echo "tests_exit=$?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
for v in "$@"; do
  if [ "$v" = base ]; then envs=""; else envs="$v"; fi
  tag=$(echo "$v" | tr '=' '_')
  env $envs timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
  python - $tag <<'P'
import json, sys
v = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/bench_{v}.json").read().strip().splitlines()[-1])
    print(v, "ms_per_step", round(d["ms_per_step"], 3), json.dumps(d["kernel_ms"]))
except Exception as e:
    print(v, "bench parse failed", e); print(open(f"gpurun_out/bench_{v}.err").read()[-2000:])
P
done
