# full GPU suite + headline bench (no CPU leg)
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 2>&1 | tail -25
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu --e2e-steps 0 2>&1 | tail -2
