# timing probes of the async-row hop (STATS build; results of probes 2/4/8 are wrong by construction)
for e in ${EXPS:-1 3 7 9}; do
  echo "== hop_experiment=$e"
  timeout -k 5 120 python bench.py --variant tensor_i8a --hop-option hop_experiment=$e --steps 1 --warmup 1 --frames 32768 --no-e2e --no-cpu 2>&1 | grep -E "hop_ar\]|Error|error|stage2_hop" | tail -4 | cut -c1-400
done
