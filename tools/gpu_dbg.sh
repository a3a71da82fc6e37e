for a in ${ABL:-0 7}; do
echo "== ablate $a"
DBP_ABLATE=$a DBP_TC_DEBUG=1 timeout 120 python bench.py --config ${CFG:-cfg2} --steps 3 --warmup 3 --no-cpu --e2e-steps 0 2>&1 | grep -A20 "tc debug" | tail -20
done
