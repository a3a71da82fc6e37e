# operand tile ring depth (DBP_TC_NOP builds) x staging: LIBS x TUNE="smax:ns:nsolv"
for lib in ${LIBS:-libdbp_b200.so}; do
for cfg in ${TUNE:-64:2:5}; do
  IFS=: read sm ns nv <<< "$cfg"
  DBP_LIB=$PWD/paper_1808_04473_b200/$lib DBP_TC_SMAX=$sm DBP_TC_NS=$ns DBP_TC_NSOLV=$nv timeout 120 python bench.py --config ${CFG:-cfg2} --steps 30 --warmup 3 --no-cpu --e2e-steps 0 2>/dev/null | tail -1 | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); print('$lib smax $sm NS $ns nsolv $nv:', round(d['ms_per_step'],4), 'ms', round(d['value'],2), 'Gb/s')
except Exception: print('$lib smax $sm NS $ns nsolv $nv failed')"
done
done
