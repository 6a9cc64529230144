# per-round cycle breakdown of the tensor hop (CTA 0), hop_experiment bits: see hop_tc.cuh Params
for e in ${EXPS:-8 12 13 28}; do
  echo "== EXP $e"; MPW_LIB=$PWD/paper_2602_08501_b200/libmpwsd_prof.so timeout 300 python bench.py --hop-option hop_experiment=$e --steps 1 --warmup 3 --frames 32768 --no-e2e --no-cpu 2>&1 | grep -E "hop_tc dbg|hop_tc seg|hop_tc mma" | tail -10
done
