cd $GRAFT_REPO_ROOT
timeout 1400 python dev/stress_strict.py 2>&1 | tail -3
bash dev/gpu/r2_strictperf.sh
