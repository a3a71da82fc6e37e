# Round artifacts: full bench line (cfg2), per-config table, ncu launch list and
# one full capture of the hot kernel, reference arm.  Outputs in gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
timeout 600 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; tail -1 gpurun_out/bench_cfg2.json | cut -c1-300
for c in cfg1 cfg3-zf cfg3-mrc cfg4-fd cfg4-pd cfg5-pd512 cfg5-fd512 cfg5-pd1024 cfg5-fd1024; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  tail -1 gpurun_out/bench_$c.json | cut -c1-120
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2>&1; tail -1 gpurun_out/bench_reference.json | cut -c1-200
timeout 200 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc2_kernel -s 3 -c 1 -o gpurun_out/prof_final python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
