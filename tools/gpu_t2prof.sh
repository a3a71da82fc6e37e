timeout 1500 python -m pytest tests -q -m gpu --timeout 600 2>&1 | tail -3
rm -f gpurun_out/parity_r02.jsonl; DBP_PARITY_OUT=gpurun_out/parity_r02.jsonl timeout 900 python -m pytest tests/test_gpu_parity_scale.py -q -m gpu -s --timeout 600 2>&1 | grep -v "^{" | tail -2
for c in cfg2 cfg1 cfg3-zf cfg3-mrc; do timeout 60 python tools/t2_time.py $c 30; done
