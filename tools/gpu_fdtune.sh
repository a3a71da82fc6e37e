# FD pipeline knobs on the TC kernel: pair (DBP_TC_PAIR) x solver count (DBP_TC_NSOLV) x staging
for c in ${CFGS:-cfg3-zf cfg1}; do
for cfg in ${TUNE:-2:5:64 1:5:64 2:6:48 1:6:48 2:4:64}; do
  IFS=: read pr nv sm <<< "$cfg"
  DBP_TC_PAIR=$pr DBP_TC_NSOLV=$nv DBP_TC_SMAX=$sm timeout 120 python bench.py --config $c --steps 30 --warmup 3 --no-cpu --e2e-steps 0 2>/dev/null | tail -1 | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); print('$c pair $pr nsolv $nv smax $sm:', round(d['ms_per_step'],4), 'ms', round(d['value'],2), 'Gb/s')
except Exception: print('$c pair $pr nsolv $nv smax $sm failed')"
done
done
