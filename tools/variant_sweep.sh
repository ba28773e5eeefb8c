#!/bin/bash
mkdir -p gpurun_out
LIB=paper_2004_11077_b200/libwinoleg_b200.so
cp $LIB /tmp/default_lib.so
for v in default "$@"; do
  if [ "$v" = default ]; then cp /tmp/default_lib.so $LIB; else cp gpurun_variants/$v.so $LIB; fi
  timeout 600 python bench.py --workload sweep --steps 20 --warmup 5 > gpurun_out/vsweep_$v.jsonl 2> gpurun_out/vsweep_$v.err
  python - "$v" <<'P'
import json, sys
v = sys.argv[1]
for l in open(f"gpurun_out/vsweep_{v}.jsonl"):
    d = json.loads(l)
    if d["workload"] == "sweep": print(v, d["config"], round(d["ms"], 4))
P
done
cp /tmp/default_lib.so $LIB
