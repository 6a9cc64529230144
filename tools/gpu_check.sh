# quick GPU check: parity tests, hop cycle probes, one bench line
set -o pipefail
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
EXPS="${EXPS:-8}" timeout 300 bash tools/diag_hop.sh
timeout 600 python bench.py --no-cpu ${BENCH_ARGS:-} | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'kms',d['kernel_ms_per_step'],'frac',d['roofline']['frac'],'e2e',d['e2e']['value'] if d['e2e'] else None,'clk',d['clocks'],'uncert',d['uncertified_frames'],'fer',d['fer'])"
