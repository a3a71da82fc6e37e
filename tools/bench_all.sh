#!/bin/bash
# one line per BASELINE config: value Gb/s, ms/step, roofline fraction
for c in "$@"; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu --e2e-steps 0 2>&1 | tail -1 | python -c "
import json,sys
t=sys.stdin.read()
try:
    d=json.loads(t); print('$c', round(d['value'],2), 'Gb/s', round(d['ms_per_step'],4), 'ms frac', round(d['roofline']['frac'],3), 'clk', d['clocks']['sm_mhz'])
except Exception: print('$c FAILED', t[-300:])
"
done
