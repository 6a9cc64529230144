# two bench repetitions: frames/s, hop ms, SM clock, cycles per tile, live share, M cycles per launch, scans
for i in 1 2; do timeout -k 5 200 python bench.py --no-cpu --no-e2e | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); h=d['roofline']['hop_detail']
print(int(d['value']), round(d['kernel_ms_per_step']['stage2_hop'],2), d['clocks']['sm_mhz'], round(h['cycles_per_tile'],1), round(h['rows_live'],4), round(h['cycles_per_tile']*h['tiles_per_cta_per_step']/5e6,2), d['counters']['iterations'])"; done
