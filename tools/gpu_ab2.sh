# interleaved A/B of library builds on one box: LIBS="a.so b.so" REPS=3 CFG=cfg2
for r in $(seq ${REPS:-3}); do
 for lib in ${LIBS}; do
  DBP_LIB=$PWD/paper_1808_04473_b200/$lib timeout 120 python bench.py --config ${CFG:-cfg2} --steps 30 --warmup 3 --no-cpu --e2e-steps 0 2>/dev/null | tail -1 | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step'],4), 'ms', round(d['value'],2), 'Gb/s')
except Exception: print('$lib failed')"
 done
done
