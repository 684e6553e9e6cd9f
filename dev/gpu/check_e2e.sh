# GPU suite + a bench line with e2e (incl. the file leg), no CPU baseline
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
grep -E "FAILED|Error|passed|failed|rc=" gpurun_out/pytest_gpu.log | tail -6
timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_e2e.err
python -c "import json; d=json.load(open('gpurun_out/bench_e2e.json')); print(round(d['value'],1), d['stage_ms_per_step']); print(json.dumps(d['e2e']))"
