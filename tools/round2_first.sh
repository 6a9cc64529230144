# Round-2 first GPU pass: parity tests, bench + ncu (measure_round), cfg4 oracle subsample, gather ncu capture at cfg2, 2-rank spawn bench on one GPU is NOT done (ranks need separate GPUs).
set -o pipefail
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r02a_pytest.log; echo pytest rc=$?; tail -3 gpurun_out/r02a_pytest.log
PFX=r02a bash tools/measure_round.sh
timeout 900 python tools/cfg4_oracle_subsample.py --frames 8192 --out gpurun_out/r02_cfg4_oracle_subsample.json > gpurun_out/r02a_subsample.log 2>&1; echo subsample rc=$?
timeout 600 python bench.py --config cfg2 --variant gather --no-cpu --no-e2e --steps 2 --warmup 3 > gpurun_out/r02a_gather_cfg2.jsonl 2>gpurun_out/r02a_gather_cfg2.err; echo gather rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hop_gather -s 3 -c 1 -o gpurun_out/r02a_gather_cfg2 \
  python bench.py --config cfg2 --variant gather --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/r02a_ncu_gather.log 2>&1; echo gather-ncu rc=$?
