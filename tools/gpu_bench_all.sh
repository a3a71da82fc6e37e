# headline bench (full JSON line) + per-config lines (no CPU / e2e legs)
mkdir -p gpurun_out/bench
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench/cfg2.json 2> gpurun_out/bench/cfg2.err; tail -c 3000 gpurun_out/bench/cfg2.json
for c in ${CFGS:-cfg1 cfg3-zf cfg3-mrc cfg4-fd cfg4-pd cfg5-pd512 cfg5-fd512 cfg5-pd1024 cfg5-fd1024}; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-20} --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/bench/$c.json 2> gpurun_out/bench/$c.err
  python -c "
import json,sys
d=json.loads(open('gpurun_out/bench/$c.json').read().strip().splitlines()[-1])
p=d['parity'] or {}
print('$c', '%.2f Gb/s %.4f ms frac %.3f' % (d['value'], d['ms_per_step'], d['roofline']['frac']), d['roofline']['kernel'], 'xhat %.1e dec %d/%d' % (p.get('xhat_normwise_max',0), p.get('decision_mismatches',0), p.get('symbols_checked',0)), d['clocks']['sm_mhz'])" || tail -5 gpurun_out/bench/$c.err
done
