# ablation timing of the cfg2 TC kernel: 1 = no solver work, 2 = no MMAs, 4 = no conversion
for a in ${ABLS:-0 1 3 5 7}; do
  DBP_ABLATE=$a timeout 120 python bench.py --steps 20 --warmup 3 --no-cpu --e2e-steps 0 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('ablate $a', round(d['ms_per_step'],4), 'ms')"
done
