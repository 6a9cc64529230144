# Round measurement: bench line (ours + reference arm), ncu launch list, ncu full captures of the hop and SCL kernels.
P=${PFX:-r02d}
timeout -k 5 900 python bench.py > gpurun_out/${P}_bench.jsonl 2> gpurun_out/${P}_bench.err; echo bench rc=$?
timeout -k 5 600 python bench.py --impl reference --steps 2 --warmup 3 >> gpurun_out/${P}_bench.jsonl 2>> gpurun_out/${P}_bench.err; echo ref rc=$?
timeout -k 5 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${P}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/${P}_ncu_launch.log 2>&1; echo launches rc=$?
timeout -k 5 1200 ncu --set full --clock-control none --import-source on -k regex:'hop_ar|hop_tc' -s 3 -c 1 -o gpurun_out/${P}_hop \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/${P}_ncu_hop.log 2>&1; echo hop rc=$?
timeout -k 5 900 ncu --set full --clock-control none --import-source on -k regex:scl_lane -s 3 -c 1 -o gpurun_out/${P}_scl \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/${P}_ncu_scl.log 2>&1; echo scl rc=$?
