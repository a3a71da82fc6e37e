set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
for c in cfg1 cfg2 cfg3-zf cfg3-mrc cfg4-fd cfg4-pd cfg5-pd512; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/b_tc_$c.json 2> gpurun_out/b_tc_$c.err; tail -1 gpurun_out/b_tc_$c.json | cut -c1-400
  DBP_FORCE_SIMT=1 timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/b_simt_$c.json 2>&1; tail -1 gpurun_out/b_simt_$c.json | cut -c1-300
done
DBP_TC_DEBUG=1 timeout 120 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 2>&1 | grep -A6 "tc debug" | tail -7
