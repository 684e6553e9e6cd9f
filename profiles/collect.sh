#!/usr/bin/env bash
# Profile capture for the round (run on the B200 box through gpurun):
#   bash profiles/collect.sh <tag>
# 1. the bench command once without ncu (must exit 0),
# 2. the launch list (gpu__time_duration per launch, cold-cache, serialised),
# 3. one `ncu --set full` capture per hot kernel (one launch each, 1 GPU).
# Outputs land in gpurun_out/; profiles/summarize.py turns them into profiles/<tag>_*.
set -u
TAG=${1:-r01}
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --frames 2"
timeout 600 $CMD > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err || { echo "plain run failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv $CMD > /dev/null 2> gpurun_out/${TAG}_launches.err
# warm-up launches: 3 steps x 16 kernels; capture step 4's kernels
timeout 900 ncu --set full --clock-control none --import-source on -k regex:laplacian \
  -s 35 -c 1 -o gpurun_out/${TAG}_lap $CMD > gpurun_out/${TAG}_ncu_lap.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:triangulate_kernel \
  -s 3 -c 1 -o gpurun_out/${TAG}_tri $CMD > gpurun_out/${TAG}_ncu_tri.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bilateral_packed \
  -s 12 -c 1 -o gpurun_out/${TAG}_bil $CMD > gpurun_out/${TAG}_ncu_bil.log 2>&1
# bilateral iteration 1 (FC normals + pack + packed-plane writes)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bilateral_kernel" \
  -s 3 -c 1 -o gpurun_out/${TAG}_bil1 $CMD > gpurun_out/${TAG}_ncu_bil1.log 2>&1
ls -la gpurun_out/${TAG}_*
