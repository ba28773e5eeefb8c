#!/bin/bash
# Round-2 evidence for the non-default workloads (one gpurun call): config 1-3 sweep (fwd + bwd),
# config-3 backward, config-5 training step, config 4 with batch-wide scales.
mkdir -p gpurun_out
timeout 900 python bench.py --workload sweep --steps 20 --warmup 5 > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
timeout 600 python bench.py --workload bwd --steps 10 --warmup 3 > gpurun_out/bwd.jsonl 2> gpurun_out/bwd.err
timeout 600 python bench.py --workload train --steps 10 --warmup 3 > gpurun_out/train.jsonl 2> gpurun_out/train.err
timeout 600 python bench.py --scale-groups batch --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_batch.json 2> gpurun_out/bench_batch.err
for f in sweep bwd train; do echo "== $f"; tail -c 1500 gpurun_out/$f.err; cut -c1-600 gpurun_out/$f.jsonl; done
echo "== batch"; tail -c 1200 gpurun_out/bench_batch.json; tail -3 gpurun_out/bench_batch.err
