# cfg2 skeleton studies: 128 = producer + converters only (no MMA / assembly / solve),
# 132 = producer + converter waits only, 7 = every hand-off without work, 0 = full
for a in ${ABLS:-0 7 128 132}; do
  DBP_ABLATE=$a timeout 60 python bench.py --steps 30 --warmup 3 --no-cpu --e2e-steps 0 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('ablate $a', round(d['ms_per_step'],4), 'ms')"
done
