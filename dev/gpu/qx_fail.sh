cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | grep -E "^(FAILED|E )" | head -20
