# A/B: hop kernel ms per step for the committed build (tools/ab/libmpwsd_orig.so) vs the working tree
for i in ${REPS:-1 2}; do
  for v in orig new; do
    if [ $v = orig ]; then export MPW_LIB=$PWD/tools/ab/libmpwsd_orig.so; else unset MPW_LIB; fi
    timeout 300 python bench.py --steps 3 --warmup 3 --frames ${FRAMES:-65536} --no-e2e --no-cpu ${BENCH_ARGS:-} | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), {k: round(v,2) for k,v in d['kernel_ms_per_step'].items()}, d['clocks']['sm_mhz'])"
  done
done
