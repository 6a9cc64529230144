# ncu full capture (with source) of the async-row hop on a 32,768-frame cfg4 step
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hop_ar -s 2 -c 1 -o gpurun_out/${PFX:-r02b}_hop_ar \
  python bench.py --variant tensor_i8a --steps 1 --warmup 2 --frames ${FRAMES:-32768} --no-e2e --no-cpu > gpurun_out/${PFX:-r02b}_ncu_hop_ar.log 2>&1; echo ncu rc=$?
