# stream-only skeleton (DBP_ABLATE=132) vs staging geometry and wait flavour
for lib in libdbp_b200.so libdbp_spin.so; do
for cfg in 64:2 32:2 32:4 32:6 16:8; do
  IFS=: read sm ns <<< "$cfg"
  DBP_LIB=$PWD/paper_1808_04473_b200/$lib DBP_ABLATE=${ABL:-132} DBP_TC_SMAX=$sm DBP_TC_NS=$ns timeout 60 python bench.py --steps 30 --warmup 3 --no-cpu --e2e-steps 0 2>/dev/null | tail -1 | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); print('$lib smax $sm NS $ns:', round(d['ms_per_step'],4), 'ms')
except Exception: print('$lib smax $sm NS $ns failed')"
done
done
