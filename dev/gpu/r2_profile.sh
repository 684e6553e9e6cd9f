cd $GRAFT_REPO_ROOT
bash profiles/collect.sh r02a > gpurun_out/collect_r02a.log 2>&1
tail -30 gpurun_out/collect_r02a.log
