# repeated bench lines of one hop variant (hop ms, clock, power): noise estimate for A/B runs
for i in 1 2 3; do
timeout -k 5 180 python bench.py --variant ${V:-tensor_i8a} --no-cpu --no-e2e ${BENCH_ARGS:-} | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('${V:-tensor_i8a} value %.0f hop %.2f scl %.2f frac %.3f clk %s power %s' % (d['value'], d['kernel_ms_per_step']['stage2_hop'], d['kernel_ms_per_step']['stage1_scl'], d['roofline']['frac'], d['clocks'].get('sm_mhz'), d['clocks'].get('power_w')))"
done
