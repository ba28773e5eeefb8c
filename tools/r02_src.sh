#!/bin/bash
# GPU box: quick parity + bench, then ncu --set full source pages of the kernels matching $1 (regex).
RX=${1:-sout_ct}; N=${2:-512}
mkdir -p gpurun_out
bash tools/quick.sh
bash tools/ncu_source.sh "$RX" 4 $N sel
python tools/sass_mix.py gpurun_out/src_sel.csv > gpurun_out/mix_sel.txt
cat gpurun_out/sum_sel.csv | cut -c1-700
head -120 gpurun_out/mix_sel.txt
