# hop variants per config: frames/s and hop ms (one bench line each, no CPU/e2e legs)
for c in ${CFGS:-cfg2 cfg3 cfg1}; do
  for v in ${VARS:-tensor tensor_i8}; do
    timeout 300 python bench.py --no-cpu --no-e2e --config $c --variant $v --frames ${FRAMES:-131072} 2>/dev/null | tail -1 | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read()); print('$c', '$v', round(d['value']), {k: round(x,2) for k,x in d['kernel_ms_per_step'].items()}, 'unc', d['uncertified_frames'], 'fer', d['fer'], 'clk', d['clocks'].get('sm_mhz'))
except Exception as e: print('$c', '$v', 'failed', e)"
  done
done
