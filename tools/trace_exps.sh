# per-tile trace summaries of the tensor hop under several hop_experiment knobs
for e in ${EXPS:-128 144 129}; do
  echo "== EXP $e"
  MPW_LIB=$PWD/paper_2602_08501_b200/libmpwsd_prof.so timeout 300 python bench.py --hop-option hop_experiment=$e --steps 1 --warmup 3 --frames 32768 --no-e2e --no-cpu 2>&1 | grep -E "hop_tc" | tail -10
  python tools/hop_trace.py gpurun_out/hop_trace.bin 244 | grep -E "period|span|per-warp|issuer|hop_tc"
done
