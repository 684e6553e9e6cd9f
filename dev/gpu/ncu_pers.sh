cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --frames 2"
timeout 600 $CMD > gpurun_out/np_plain.json 2> gpurun_out/np_plain.err || { echo plain failed; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bilateral_kernel \
  -s 16 -c 1 -o gpurun_out/np_pers $CMD > gpurun_out/np_ncu.log 2>&1
tail -1 gpurun_out/np_ncu.log
