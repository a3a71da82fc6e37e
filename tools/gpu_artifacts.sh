# Round artifacts on one B200 (outputs in gpurun_out/$TAG/, TAG default r02):
#   headline bench line (cfg2, full JSON), per-config bench lines, reference arm,
#   launch list of the headline run, ncu --set full captures of the dominant
#   kernel of cfg2 / cfg3-zf / cfg4-fd / cfg5-pd512 (each after a clean run).
set -u
O=gpurun_out/${TAG:-r02}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
timeout 900 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err; tail -c 400 $O/bench_cfg2.json
for c in cfg1 cfg3-zf cfg3-mrc cfg4-fd cfg4-pd cfg5-pd512 cfg5-fd512 cfg5-pd1024 cfg5-fd1024; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --e2e-steps 0 > $O/bench_$c.json 2> $O/bench_$c.err
  tail -1 $O/bench_$c.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value'],2), 'Gb/s frac', round(d['roofline']['frac'],3), d['roofline']['kernel'])" || tail -3 $O/bench_$c.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2>&1; tail -1 $O/bench_reference.json | cut -c1-200
# launch list of the headline command
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 --no-parity > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_cfg2.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 --no-parity > $O/ncu_launch.log 2>&1
# full captures (one launch each, after warm-up)
cap() {  # name config kernel-regex skip
  timeout 300 python tools/t2_time.py $2 4 > $O/plain_$1.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c 1 -o $O/prof_$1 \
    python tools/t2_time.py $2 4 > $O/ncu_$1.log 2>&1
  tail -1 $O/ncu_$1.log
}
cap cfg2 cfg2 tc2_kernel 4
cap cfg3zf cfg3-zf tc2_kernel 4
cap cfg4fd cfg4-fd lama_kernel 2
cap cfg4pd cfg4-pd lama_kernel 2
cap cfg5pd512_stats cfg5-pd512 tcw_stats 3
cap cfg5pd512_solve cfg5-pd512 ^stats_kernel 3
cap cfg1 cfg1 tc2_kernel 4
ls -la $O
