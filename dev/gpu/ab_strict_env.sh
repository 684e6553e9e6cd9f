# strict chain timing A/B over an environment switch (bash dev/gpu/ab_strict_env.sh VAR) + strict suites
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_strict.py tests/test_gpu_vs_reference.py tests/test_gpu_reference_cases.py -q -x -p no:cacheprovider 2>&1 | tail -1
for E in 0 1 0 1; do
  echo "$1=$E: $(env $1=$E timeout 300 python profiles/strict_driver.py --frames 16 --steps 6 2>&1 | tail -1)"
done
