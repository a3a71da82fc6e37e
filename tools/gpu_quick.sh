# quick GPU check: gpu tests (optionally filtered) + selected bench configs
# usage: bash tools/gpu_quick.sh TAG "pytest -k expr or empty" cfg...
set -u
TAG=$1; K=$2; shift 2
O=gpurun_out/$TAG; mkdir -p $O
if [ -n "$K" ]; then timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > $O/pytest.log 2>&1
else timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; fi
tail -4 $O/pytest.log
for c in "$@"; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --e2e-steps 0 > $O/bench_$c.json 2> $O/bench_$c.err
  tail -1 $O/bench_$c.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['parity']; print('$c', round(d['ms_per_step'],4), 'ms', round(d['value'],2), 'Gb/s frac', round(d['roofline']['frac'],4), 'err', '%.2e'%p['xhat_normwise_max'], 'mism', p['decision_mismatches'])" || tail -3 $O/bench_$c.err
done
