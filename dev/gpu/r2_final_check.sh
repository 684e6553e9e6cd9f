cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
ST="python profiles/strict_driver.py --frames 16 --steps 2"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bilateral_f64s" -s 6 -c 1 -o gpurun_out/r02e_bil64 $ST > gpurun_out/r02e_ncu_bil64.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"laplacian_f64" -s 12 -c 1 -o gpurun_out/r02e_lap64 $ST > gpurun_out/r02e_ncu_lap64.log 2>&1
tail -1 gpurun_out/r02e_ncu_lap64.log
