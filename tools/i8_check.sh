# int8 screen: parity tests, one bench line, per-tile trace
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "i8" > gpurun_out/i8_tests.log 2>&1; echo tests rc=$?; tail -4 gpurun_out/i8_tests.log
for v in ${BVARS:-tensor_i8}; do
  timeout 400 python bench.py --no-cpu --no-e2e --variant $v 2>gpurun_out/i8_bench_$v.err | tail -1 > gpurun_out/i8_bench_$v.json
  python -c "
import json,sys; d=json.load(open('gpurun_out/i8_bench_$v.json')); print('$v', round(d['value']), {k: round(x,2) for k,x in d['kernel_ms_per_step'].items()}, round(d['roofline']['achieved']), round(d['roofline']['frac'],3), d['clocks'], 'unc', d['uncertified_frames'], 'fer', d['fer'], 'ntie', d['near_tie_frames'], d['avg_iters'])"
  tail -2 gpurun_out/i8_bench_$v.err
done
VARS=tensor_i8 bash tools/trace_i8.sh
