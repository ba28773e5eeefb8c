#!/bin/bash
# GPU box: compare the in-tree library with variants in gpurun_variants/*.so: GPU parity tests
# (tests/test_gpu_parity.py) and a short config-4 bench per library.  Usage: tools/variant_check.sh [names...]
mkdir -p gpurun_out
libs="default"
if [ $# -gt 0 ]; then libs="$libs $*"; fi
for v in $libs; do
  if [ "$v" = default ]; then unset WL_LIB_PATH; else export WL_LIB_PATH=$PWD/gpurun_variants/$v.so; fi
  if [ "$v" != default ]; then
    timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/var_$v.tests.log 2>&1
    echo "$v tests: $(tail -1 gpurun_out/var_$v.tests.log)"
  fi
  timeout 300 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
  python - "$v" <<'P'
import json, sys
v = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/var_{v}.json").read().strip().splitlines()[-1])
    print(v, "ms_per_step", round(d["ms_per_step"], 3), json.dumps(d["kernel_ms"]))
except Exception as e:
    print(v, "bench failed", e, open(f"gpurun_out/var_{v}.err").read()[-1500:])
P
done
