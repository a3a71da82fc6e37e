# tensor-core vs SIMT streaming kernel per config (DBP_FORCE_SIMT)
for c in ${CFGS:-cfg4-pd cfg4-fd}; do
 for f in 0 1; do
  DBP_FORCE_SIMT=$f timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --e2e-steps 0 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$c force_simt=$f', round(d['ms_per_step'],4), 'ms', round(d['value'],2), 'Gb/s')"
 done
done
