cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --frames 2"
timeout 300 $CMD > gpurun_out/plain3.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bilateral_kernel -s 6 -c 1 -o gpurun_out/prof_bil $CMD > gpurun_out/ncu_bil.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:triangulate_kernel -s 1 -c 1 -o gpurun_out/prof_tri $CMD > gpurun_out/ncu_tri.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:laplacian_kernel -s 12 -c 1 -o gpurun_out/prof_lap $CMD > gpurun_out/ncu_lap.log 2>&1
ls -la gpurun_out/*.ncu-rep
