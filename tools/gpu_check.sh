set -u
O=gpurun_out/${TAG:-r02m}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" ; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?; tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err; tail -c 300 $O/bench_cfg2.json
for c in cfg5-pd512 cfg5-fd512 cfg5-pd1024 cfg5-fd1024; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --e2e-steps 0 > $O/bench_$c.json 2> $O/bench_$c.err
  tail -1 $O/bench_$c.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value'],2), 'Gb/s ms', round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],3), d.get('parity'))" || tail -3 $O/bench_$c.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err; tail -c 300 $O/bench_reference.json
