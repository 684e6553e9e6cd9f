cd $GRAFT_REPO_ROOT/dev
run() { timeout 60 ./tma_probe "$@" 2>&1 | tail -2 | tr '\n' ' '; echo; }
run 10 1 0 -1 204 18
run 10 1 -4 0 204 18
run 10 1 -4 -1 204 18
run 10 1 3 0 204 18
run 10 1 4 0 204 18
run 10 1 -1 0 204 18
run 10 1 -3 0 204 18
run 10 1 100 60 204 18
