# full GPU pass: all gpu tests, round measurement, cfg4 oracle subsample (all int8/f16 hops)
set -o pipefail
timeout -k 5 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/${PFX:-r02d}_pytest.log; echo pytest rc=$?; tail -3 gpurun_out/${PFX:-r02d}_pytest.log
bash tools/measure_round.sh
timeout -k 5 900 python tools/cfg4_oracle_subsample.py --frames 8192 --out gpurun_out/r02_cfg4_oracle_subsample.json > gpurun_out/${PFX:-r02d}_subsample.log 2>&1; echo subsample rc=$?
