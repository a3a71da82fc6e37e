# staging / solver-count sweep: TUNE="SMAX_KB:NS:NSOLV ..." (CFG=cfg2)
for cfg in ${TUNE:-64:2:5}; do
  IFS=: read sm ns nv <<< "$cfg"
  DBP_TC_SMAX=$sm DBP_TC_NS=$ns DBP_TC_NSOLV=$nv timeout 120 python bench.py --config ${CFG:-cfg2} --steps 20 --warmup 3 --no-cpu --e2e-steps 0 2>/dev/null | tail -1 | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); print('smax $sm NS $ns nsolv $nv:', round(d['ms_per_step'],4), 'ms', round(d['value'],2), 'Gb/s')
except Exception: print('smax $sm NS $ns nsolv $nv failed')"
done
