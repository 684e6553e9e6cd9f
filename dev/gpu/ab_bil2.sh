# bilateral A/B (dev/ab/old.so vs new.so) + parity suites + randomised stress on the default build
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_strict.py tests/test_gpu_reference_cases.py -q -x -p no:cacheprovider > gpurun_out/ab_pytest.log 2>&1
grep -E "passed|failed|FAILED" gpurun_out/ab_pytest.log | tail -3
for L in old new old new old new; do
OPCFE_LIB=dev/ab/$L.so timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-strict > gpurun_out/ab_$L.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/ab_$L.json')); print('$L', round(d['value'],1), d['stage_ms_per_step'], d['clocks']['sm_mhz'])"
done
timeout 900 python dev/stress_randomised.py 2>&1 | tail -2
