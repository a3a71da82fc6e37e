# H-ring depth study (DBP_TC_NS) with and without work (DBP_ABLATE=7)
for ns in 4 8 12 16 20; do
 for a in 0 7; do
  DBP_TC_NS=$ns DBP_ABLATE=$a timeout 120 python bench.py --steps 20 --warmup 3 --no-cpu --e2e-steps 0 2>/dev/null | tail -1 | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); print('NS $ns ablate $a', round(d['ms_per_step'],4), 'ms')
except Exception: print('NS $ns ablate $a failed')"
 done
done
DBP_TC_DEBUG=1 timeout 120 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 2>&1 | grep -A5 "tc debug" | tail -6
