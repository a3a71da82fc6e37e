ABLS="7 39 0 32" bash tools/gpu_ablate.sh 2>&1 | grep ablate
for a in 0 7; do DBP_LIB=$PWD/paper_1808_04473_b200/libdbp_b200_nop3.so DBP_TC_SMAX=32 DBP_TC_NS=3 DBP_TC_NSOLV=4 DBP_ABLATE=$a timeout 120 python bench.py --steps 20 --warmup 3 --no-cpu --e2e-steps 0 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('NOP3 smax32 ns3 nsolv4 ablate $a', round(d['ms_per_step'],4))"; done
for a in 0 7; do DBP_TC_SMAX=32 DBP_TC_NS=3 DBP_TC_NSOLV=5 DBP_ABLATE=$a timeout 120 python bench.py --steps 20 --warmup 3 --no-cpu --e2e-steps 0 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('NOP2 smax32 ns3 ablate $a', round(d['ms_per_step'],4))"; done
