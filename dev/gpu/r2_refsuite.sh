cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_reference_suite.py -q --timeout 900 -p no:cacheprovider -s > gpurun_out/pytest_refsuite.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_refsuite.log
tail -40 gpurun_out/pytest_refsuite.log
