for t in 56 28 19 14 8; do
  WL_FUSED_TEAM=$t timeout 120 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('team $t', round(d['ms_per_step'],3), d['kernel_ms']['quant_input'])"
done
WL_NO_FUSED_QUANT=1 timeout 120 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('unfused', round(d['ms_per_step'],3), d['kernel_ms']['absmax_input'], d['kernel_ms']['quant_input'])"
