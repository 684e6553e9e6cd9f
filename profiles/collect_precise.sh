#!/usr/bin/env bash
# ncu captures of the STRICT and MIXED precision chains (run on the B200 box via gpurun):
#   bash profiles/collect_precise.sh <tag>
# C4, 16 frames (profiles/strict_driver.py, eager launches): per precision the launch list
# and one `--set full` capture of the Laplacian pass, the FC-data kernel and the first
# bilateral iteration.  profiles/summarize_precise.py turns them into profiles/<tag>_precise_summary.md.
set -u
TAG=${1:-r02}
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
for P in strict mixed; do
  CMD="python profiles/strict_driver.py --frames 16 --steps 2 --precision $P"
  timeout 900 $CMD > gpurun_out/${TAG}_${P}_plain.txt 2>&1 || { echo "$P plain run failed"; continue; }
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_${P}_launches.csv $CMD > /dev/null 2>&1
  timeout 900 $NCU -k regex:"laplacian_f64_tma" -s 12 -c 1 -o gpurun_out/${TAG}_${P}_lap $CMD > /dev/null 2>&1
  timeout 900 $NCU -k regex:"fc_rows" -s 1 -c 1 -o gpurun_out/${TAG}_${P}_fc $CMD > /dev/null 2>&1
  if [ "$P" = strict ]; then K="bilateral_f64s"; else K="bilateral_kernel"; fi
  timeout 900 $NCU -k regex:"$K" -s 5 -c 1 -o gpurun_out/${TAG}_${P}_bil $CMD > /dev/null 2>&1
done
ls -la gpurun_out/${TAG}_*
