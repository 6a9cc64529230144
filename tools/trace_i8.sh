# per-tile clock trace (CTA 0, MODE 1 build) of the int8 and f16 tensor hops
for v in ${VARS:-tensor_i8 tensor}; do
  echo "== $v"
  MPW_TC_EXPERIMENT=128 MPW_TC_TRACE=gpurun_out/trace_$v.bin timeout 300 python bench.py --steps 1 --warmup 3 --frames 32768 --no-e2e --no-cpu --variant $v > /dev/null 2>&1
  python tools/hop_trace.py gpurun_out/trace_$v.bin 244
done
