# A/B of the CTA-pair (multicast) hop against the single-CTA hop, same build
for i in ${REPS:-1 2}; do
  for c in 0 1; do
    timeout 300 python bench.py --hop-option f16_cluster=$c --steps 5 --warmup 3 --frames ${FRAMES:-131072} --no-e2e --no-cpu | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('cluster=$c', round(d['value']), {k: round(v,2) for k,v in d['kernel_ms_per_step'].items()}, d['clocks']['sm_mhz'], d['clocks'].get('power_w'), d['uncertified_frames'], d['fer'])"
  done
done
