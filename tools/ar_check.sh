# async-row int8 hop: parity tests, statistics lines, bench A/B against the synchronous int8 hop
# (short hard timeouts: a deadlocked kernel must not hold the box)
set -o pipefail
timeout -k 5 240 python -m pytest tests/test_gpu_parity.py -x -q -k "tensor_i8a" 2>&1 | tail -4
timeout -k 5 120 python bench.py --variant tensor_i8a --hop-option hop_experiment=1 --steps 1 --warmup 1 --frames 32768 --no-e2e --no-cpu 2>&1 | grep -E "hop_ar\]|Error|error" | tail -4
for v in ${VARS:-tensor_i8a tensor_i8}; do
timeout -k 5 180 python bench.py --variant $v --no-cpu --no-e2e ${BENCH_ARGS:-} | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v value',d['value'],'kms',d['kernel_ms_per_step'],'frac',d['roofline']['frac'],'clk',d['clocks'],'uncert',d['uncertified_frames'],'fer',d['fer'], 'iters', d['avg_iters'], 'neartie', d['near_tie_frames'])"
done
