# int8 hop: single CTAs vs multicast CTA pairs vs cta_group::2 pairs
for i in 1 2; do
for cfg in "MPW_TC_I8_CL=1" "MPW_TC_I8_CL=2" "MPW_TC_PAIR=1"; do
  env $cfg timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --variant tensor_i8 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', round(d['value']), {k: round(v,2) for k,v in d['kernel_ms_per_step'].items()}, d['clocks']['sm_mhz'], d['clocks'].get('power_w'), 'unc', d['uncertified_frames'])"
done; done
