#!/bin/bash
# quick GPU iteration: parity subset + config-4 bench (no e2e / cpu legs)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/q_tests.log 2>&1
tail -3 gpurun_out/q_tests.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/q_bench.json").read().strip().splitlines()[-1])
print("ms", round(d["ms_per_step"], 3), "img/s", round(d["value"]), "frac", round(d["layer_roofline"]["frac"], 4))
print({k: round(v, 3) for k, v in d["kernel_ms"].items()})
PY
tail -3 gpurun_out/q_bench.err
