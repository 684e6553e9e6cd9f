cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-strict --frames 16"
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:"bilateral_packed" -s 12 -c 1 -o gpurun_out/sym_bil $CMD > gpurun_out/sym_ncu.log 2>&1
tail -2 gpurun_out/sym_ncu.log
