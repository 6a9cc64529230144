# per-tile clock trace (CTA 0, MODE 1 build) of the int8 and f16 tensor hops
for v in ${VARS:-tensor_i8 tensor}; do
  echo "== $v"
  MPW_LIB=$PWD/paper_2602_08501_b200/libmpwsd_prof.so MPW_TC_TRACE=gpurun_out/trace_$v.bin timeout 300 python bench.py --hop-option hop_experiment=128 --steps 1 --warmup 3 --frames 32768 --no-e2e --no-cpu --variant $v > /dev/null 2>&1
  python tools/hop_trace.py gpurun_out/trace_$v.bin 244
done
