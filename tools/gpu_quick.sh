# quick GPU iteration: gram tile test, full gpu tests, cfg bench lines, TC debug counters
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gram_tiles.py -x -q 2>&1 | tail -5
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for c in ${CFGS:-cfg2}; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/q_$c.json 2> gpurun_out/q_$c.err
  python -c "
import json
d=json.loads(open('gpurun_out/q_$c.json').read().strip().splitlines()[-1])
print('$c', round(d['value'],2), 'Gb/s', round(d['ms_per_step'],4), 'ms frac', round(d['roofline']['frac'],3), 'clk', d['clocks']['sm_mhz'])
" || tail -3 gpurun_out/q_$c.err
done
DBP_TC_DEBUG=1 timeout 120 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 2>&1 | grep -A5 "tc debug" | tail -6
