# ncu --set full capture of the FD U = 64 solve kernel (stats_kernel<64, 128, XZ>) on cfg5-fd512
O=gpurun_out/${TAG:-r02fd64}; mkdir -p $O
timeout 300 python tools/t2_time.py cfg5-fd512 2 > $O/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:^stats_kernel -s 3 -c 1 -o $O/prof_cfg5fd512_solve \
  python tools/t2_time.py cfg5-fd512 2 > $O/ncu.log 2>&1
tail -2 $O/ncu.log
