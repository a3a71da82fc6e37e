# one ncu --set full capture of a kernel of a workload (after a clean run)
# usage: bash tools/gpu_prof.sh TAG config kernel-regex skip [reps]
set -u
O=gpurun_out/$1; mkdir -p $O
timeout 300 python tools/t2_time.py $2 ${5:-4} > $O/plain_$2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c 1 -o $O/prof_$2 \
  python tools/t2_time.py $2 ${5:-4} > $O/ncu_$2.log 2>&1
tail -1 $O/ncu_$2.log
