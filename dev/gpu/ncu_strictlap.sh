cd $GRAFT_REPO_ROOT
ST="python profiles/strict_driver.py --frames 16 --steps 2"
$ST > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"laplacian_f64" -s 12 -c 1 -o gpurun_out/lapsym $ST > gpurun_out/lapsym.log 2>&1
tail -1 gpurun_out/lapsym.log
