# round 2 first call: fp64 probe, GPU suite, one bench line
cd $GRAFT_REPO_ROOT
./dev/probes/fp64_probe > gpurun_out/fp64_probe.txt 2>&1; cat gpurun_out/fp64_probe.txt
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
grep -E "FAILED|Error|passed|failed|rc=" gpurun_out/pytest_gpu.log | tail -6
timeout 900 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_check.json 2> gpurun_out/bench_check.err
python -c "import json; d=json.load(open('gpurun_out/bench_check.json')); print(round(d['value'],1), d['stage_ms_per_step'], d['roofline']['frac'])"
