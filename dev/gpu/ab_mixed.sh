# mixed-precision A/B (dev/ab/old.so vs new.so): device frames/s + chained parity, mixed tests
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_strict.py tests/test_gpu_vs_reference.py -q -x -p no:cacheprovider -k mixed 2>&1 | tail -1
for L in old new old new; do
  OPCFE_LIB=dev/ab/$L.so timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/abm_$L.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/abm_$L.json')); print('$L', round(d['mixed']['value'],1), d['mixed']['stage_ms_per_step'], d['parity']['chained']['mixed']['normals_abs'])"
done
