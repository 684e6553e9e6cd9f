#!/usr/bin/env bash
# Profile capture for the round (run on the B200 box through gpurun):
#   bash profiles/collect.sh <tag>
# At the BENCH'S OWN batch (16 C4 frames = 398 MB of fp32 input, > the 126 MB L2):
# 1. the bench command once without ncu (must exit 0),
# 2. the launch list (gpu__time_duration per launch, cold-cache, serialised),
# 3. one `ncu --set full` capture per hot kernel (one launch each, 1 GPU):
#    Laplacian pass 1 / packed passes, triangulation, bilateral iteration 1 / packed
#    iterations; quad_extras at C3 (512 frames); the strict fp64 kernels at C4.
# Outputs land in gpurun_out/; profiles/summarize.py turns them into profiles/<tag>_*.
set -u
TAG=${1:-r02}
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-strict --frames 16"
timeout 900 $CMD > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err || { echo "plain run failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv $CMD > /dev/null 2> gpurun_out/${TAG}_launches.err
NCU="ncu --set full --clock-control none --import-source on"
# warm-up: 3 steps; -s skips that many launches of the matching kernel
timeout 900 $NCU -k regex:"laplacian3_kernel" -s 3 -c 1 -o gpurun_out/${TAG}_lap1 $CMD > gpurun_out/${TAG}_ncu_lap1.log 2>&1
timeout 900 $NCU -k regex:"laplacian3p_kernel" -s 30 -c 1 -o gpurun_out/${TAG}_lap $CMD > gpurun_out/${TAG}_ncu_lap.log 2>&1
timeout 900 $NCU -k regex:"triangulate_kernel" -s 3 -c 1 -o gpurun_out/${TAG}_tri $CMD > gpurun_out/${TAG}_ncu_tri.log 2>&1
timeout 900 $NCU -k regex:"bilateral_packed" -s 12 -c 1 -o gpurun_out/${TAG}_bil $CMD > gpurun_out/${TAG}_ncu_bil.log 2>&1
timeout 900 $NCU -k regex:"bilateral_kernel" -s 3 -c 1 -o gpurun_out/${TAG}_bil1 $CMD > gpurun_out/${TAG}_ncu_bil1.log 2>&1
C3="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-strict --workload C3"
timeout 900 $C3 > gpurun_out/${TAG}_c3_plain.json 2> gpurun_out/${TAG}_c3_plain.err && \
timeout 900 $NCU -k regex:"quad_extras" -s 3 -c 1 -o gpurun_out/${TAG}_qx $C3 > gpurun_out/${TAG}_ncu_qx.log 2>&1
ST="python profiles/strict_driver.py --frames 16 --steps 2"
timeout 900 $ST > gpurun_out/${TAG}_strict_plain.txt 2>&1 && {
timeout 900 $NCU -k regex:"laplacian_f64" -s 12 -c 1 -o gpurun_out/${TAG}_lap64 $ST > gpurun_out/${TAG}_ncu_lap64.log 2>&1
timeout 900 $NCU -k regex:"bilateral_f64" -s 6 -c 1 -o gpurun_out/${TAG}_bil64 $ST > gpurun_out/${TAG}_ncu_bil64.log 2>&1; }
ls -la gpurun_out/${TAG}_*
