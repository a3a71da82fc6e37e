# ablation timing of the SIMT stream kernel: 1 = no epilogue, 2 = no Gram, 3 = neither
for c in ${CFGS:-cfg5-pd512 cfg4-fd}; do
for a in ${ABLS:-0 1 2 3}; do
  DBP_ABLATE=$a timeout 300 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu --e2e-steps 0 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$c ablate $a', round(d['ms_per_step'],4), 'ms')"
done
done
