# strict Laplacian A/B: strict + vs-reference suites on the default build, then strict chain timing old/new
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_strict.py tests/test_gpu_vs_reference.py -q -x -p no:cacheprovider 2>&1 | tail -2
for L in old new old new; do
  echo "$L: $(OPCFE_LIB=dev/ab/$L.so timeout 300 python profiles/strict_driver.py --frames 16 --steps 6 2>&1 | tail -3 | tr '\n' ' ')"
done
for L in old new; do
OPCFE_LIB=dev/ab/$L.so timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ab_$L.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/ab_$L.json')); print('$L strict', round(d['strict']['value'],1), d['strict'].get('stage_ms_per_step'))"
done
