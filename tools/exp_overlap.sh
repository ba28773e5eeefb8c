#!/bin/bash
# GPU box: config-4 step time for (parts, grid-div) combinations — co-residency of two calls' kernels
# (bench.py --grid-div) — and ncu launch lists of the launch-bound shapes.
mkdir -p gpurun_out
for pg in "1 1" "2 1" "3 1" "4 1" "2 2" "3 2" "4 2" "3 3" "4 4"; do
  set -- $pg
  timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --parts $1 --grid-div $2 > gpurun_out/ov_$1_$2.json 2> gpurun_out/ov_$1_$2.err
  python - "$1" "$2" <<'P'
import json, sys
p, g = sys.argv[1:3]
try:
    d = json.loads(open(f"gpurun_out/ov_{p}_{g}.json").read().strip().splitlines()[-1])
    print(f"parts={p} grid_div={g} ms={d['ms_per_step']:.3f} parity={d.get('parity', {}).get('bit_exact')}")
except Exception as e:
    print(f"parts={p} grid_div={g} failed: {e}")
P
done | tee gpurun_out/overlap.txt
for shp in "8 64 32" "256 128 16" "256 512 4" "256 64 32"; do
  set -- $shp
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/small_$1_$2_$3.csv \
    python tools/prof_forward.py --n $1 --c $2 --hw $3 --iters 3 > gpurun_out/small_$1_$2_$3.log 2>&1
done
