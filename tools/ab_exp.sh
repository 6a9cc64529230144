# hop kernel ms per step under hop_experiment values (A/B of kernel variants in one build)
for i in 1 2; do
  for e in ${EXPS:-0 64}; do
    MPW_LIB=$PWD/paper_2602_08501_b200/libmpwsd_prof.so timeout 300 python bench.py --hop-option hop_experiment=$e --steps 3 --warmup 3 --frames 65536 --no-e2e --no-cpu ${BENCH_ARGS:-} | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('exp $e', round(d['value']), {k: round(v,2) for k,v in d['kernel_ms_per_step'].items()}, d['clocks']['sm_mhz'], d['clocks'].get('power_w'))"
  done
done
