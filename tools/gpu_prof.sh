# TC kernel debug counters + ncu full capture of the cfg2 hot kernel
mkdir -p gpurun_out
DBP_TC_DEBUG=1 timeout 120 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/dbg.log 2>&1
grep -A6 "tc debug" gpurun_out/dbg.log | tail -7
timeout 200 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_kernel -s 2 -c 1 -o gpurun_out/prof_tc python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ncu.log 2>&1
tail -3 gpurun_out/ncu.log
