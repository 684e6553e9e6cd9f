cd $GRAFT_REPO_ROOT
ST="python profiles/strict_driver.py --frames 16 --steps 2"
$ST > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bilateral_f64" -s 6 -c 1 -o gpurun_out/r02d_bil64 $ST > gpurun_out/r02d_ncu_bil64.log 2>&1

tail -2 gpurun_out/r02d_ncu_bil64.log
