# int8 hop: single CTAs vs multicast CTA pairs vs cta_group::2 pairs
for i in 1 2; do
for cfg in "i8_cluster=1" "i8_cluster=2" "i8_pair=1"; do
  timeout 300 python bench.py --hop-option $cfg --steps 3 --warmup 3 --no-e2e --no-cpu --variant tensor_i8 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', round(d['value']), {k: round(v,2) for k,v in d['kernel_ms_per_step'].items()}, d['clocks']['sm_mhz'], d['clocks'].get('power_w'), 'unc', d['uncertified_frames'])"
done; done
