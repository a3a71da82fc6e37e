# SIMT kernel ring depth (DBP_SIMT_NS) vs time: 2 stages let two CTAs share an SM at U = 64
for c in ${CFGS:-cfg5-pd512 cfg5-fd512}; do
for ns in ${NSS:-3 2}; do
  DBP_SIMT_NS=$ns timeout 300 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu --e2e-steps 0 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$c ns $ns', round(d['ms_per_step'],4), 'ms', round(d['value'],3), d['unit'])"
done
done
