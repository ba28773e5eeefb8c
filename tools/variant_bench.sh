#!/bin/bash
# GPU box: bench-only A/B of gpurun_variants/<name>.so (experiments that intentionally break parity).
mkdir -p gpurun_out
LIB=paper_2004_11077_b200/libwinoleg_b200.so
cp $LIB /tmp/default_lib.so
for v in default "$@"; do
  if [ "$v" = default ]; then cp /tmp/default_lib.so $LIB; else cp gpurun_variants/$v.so $LIB; fi
  timeout 300 python bench.py --no-cpu --no-e2e --steps 20 --warmup 3 > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
  python - "$v" <<'P'
import json, sys
v = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/var_{v}.json").read().strip().splitlines()[-1])
    print(v, "ms_per_step", round(d["ms_per_step"], 3), json.dumps(d["kernel_ms"]), d.get("parity"))
except Exception as e:
    print(v, "bench failed", e, open(f"gpurun_out/var_{v}.err").read()[-1500:])
P
done
cp /tmp/default_lib.so $LIB
