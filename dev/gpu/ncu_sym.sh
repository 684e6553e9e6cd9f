cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --frames 2"
timeout 600 $CMD > gpurun_out/ns_plain.json 2> gpurun_out/ns_plain.err || { echo plain failed; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bilateral_sym \
  -s 16 -c 1 -o gpurun_out/ns_sym $CMD > gpurun_out/ns_ncu.log 2>&1
tail -1 gpurun_out/ns_ncu.log
