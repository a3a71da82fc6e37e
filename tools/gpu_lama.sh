# LAMA configs: group-owned schedule (default) vs the team-wide one (ablate 64)
for c in ${CFGS:-cfg4-pd cfg4-fd}; do
for a in ${ABLS:-0 64}; do
  DBP_ABLATE=$a timeout 300 python bench.py --config $c --steps ${STEPS:-20} --warmup 3 --no-cpu --e2e-steps 0 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$c ablate $a', round(d['ms_per_step'],4), 'ms', round(d['value'],3), d['unit'])"
done
done
