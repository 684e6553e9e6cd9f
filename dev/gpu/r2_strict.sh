# strict-mode tests first, then the whole GPU suite
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_strict.py -q -x --timeout 300 -p no:cacheprovider -s > gpurun_out/pytest_strict.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_strict.log
grep -E "fast chain|FAILED|Error|passed|failed|rc=" gpurun_out/pytest_strict.log | tail -20
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
grep -E "FAILED|Error|passed|failed|rc=" gpurun_out/pytest_gpu.log | tail -30
