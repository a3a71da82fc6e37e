# A/B of library builds: LIBS="a.so b.so" ABL="0 7" CFG=cfg2
for lib in ${LIBS}; do
 for a in ${ABL:-0}; do
  DBP_LIB=$PWD/paper_1808_04473_b200/$lib DBP_ABLATE=$a timeout 120 python bench.py --config ${CFG:-cfg2} --steps 20 --warmup 3 --no-cpu --e2e-steps 0 2>/dev/null | tail -1 | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); print('$lib ablate $a', round(d['ms_per_step'],4), 'ms', round(d['value'],2), 'Gb/s')
except Exception: print('$lib ablate $a failed')"
 done
done
