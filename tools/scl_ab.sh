# A/B of stage-1 builds: stage1_scl ms per step (3 repetitions)
for i in 1 2 3; do
  timeout -k 5 200 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']; print('scl', round(k['stage1_scl'],3), 'hop', round(k['stage2_hop'],2), 'value', int(d['value']), 'clk', d['clocks']['sm_mhz'])"
done
