timeout 600 python -m pytest tests/test_gpu_tc2.py -q -m gpu --timeout 120 2>&1 | tail -3
for c in cfg3-mrc; do timeout 60 python tools/t2_time.py $c 50; done
for c in cfg1 cfg3-zf; do DBP_LIB=build_study/libdbp_study.so DBP_TC_DEBUG=1 timeout 60 python tools/t2_time.py $c 3 2>&1 | tail -16; done
