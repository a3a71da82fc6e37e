rm -f gpurun_out/parity_r02.jsonl
DBP_PARITY_OUT=gpurun_out/parity_r02.jsonl timeout 1500 python -m pytest tests/test_gpu_parity_scale.py -q -m gpu -s --timeout 600 ${PARITY_K:+-k "$PARITY_K"} 2>&1 | grep -v "^{" | tail -3
cat gpurun_out/parity_r02.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config'], 'xhat %.2e s2 %.2e nu %s dec %d/%d kern %d' % (d['xhat_normwise_max'], d['sigma2_entry_max'], ('%.2e'%d['nu_entry_max']) if 'nu_entry_max' in d else '-', d['decision_mismatches'], d['symbols_checked'], d['kernel']))"
