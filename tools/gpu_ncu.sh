# ncu --set full of the tc kernel on the cfg2 bench (after a plain run exits 0)
mkdir -p gpurun_out
CFG=${CFG:-cfg2}
timeout 200 env $NCU_ENV python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/plain.log 2>&1 && \
timeout 900 env $NCU_ENV ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-tc_kernel} -s ${SKIP:-2} -c 1 -o gpurun_out/${OUT:-prof_tc} python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ncu.log 2>&1
tail -2 gpurun_out/ncu.log
