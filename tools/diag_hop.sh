# per-round cycle breakdown of the tensor hop (CTA 0), MPW_TC_EXPERIMENT bits: see hop_tc.cuh Params
for e in ${EXPS:-8 12 13 28}; do
  echo "== EXP $e"; MPW_TC_EXPERIMENT=$e timeout 300 python bench.py --steps 1 --warmup 3 --frames 32768 --no-e2e --no-cpu 2>&1 | grep -E "hop_tc dbg|hop_tc seg|hop_tc mma" | tail -10
done
