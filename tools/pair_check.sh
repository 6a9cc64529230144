# int8 pair-MMA kernel: quick parity, then bench (single-CTA kernel for comparison)
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg4 and (i8 or int8)" 2>&1 | tail -3
timeout 200 python bench.py --no-cpu --no-e2e --variant tensor_i8 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('pair', round(d['value']), {k: round(x,2) for k,x in d['kernel_ms_per_step'].items()}, d['clocks'], 'unc', d['uncertified_frames'], 'fer', d['fer'], 'ntie', d['near_tie_frames'])"
timeout 200 python bench.py --hop-option i8_cluster=1 --no-cpu --no-e2e --variant tensor_i8 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('single', round(d['value']), {k: round(x,2) for k,x in d['kernel_ms_per_step'].items()}, d['clocks'], 'unc', d['uncertified_frames'])"
