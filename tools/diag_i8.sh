# per-round cycle report (CTA 0) of the int8 and f16 tensor hops: hop_experiment=8
for v in ${VARS:-tensor_i8 tensor}; do
  echo "== $v"; timeout 300 python bench.py --hop-option hop_experiment=${EXP:-8} --steps 1 --warmup 3 --frames 32768 --no-e2e --no-cpu --variant $v 2>&1 | grep -E "hop_tc dbg|hop_tc mma|warp [45]:" | tail -4
done
