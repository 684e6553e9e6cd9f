cd $GRAFT_REPO_ROOT
for e in 0 1 0 1; do
OPCFE_QX_STAGED=$e timeout 300 python bench.py --workload C3 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-strict > gpurun_out/qx_$e.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/qx_$e.json')); print('staged=$e', round(d['value'],1), d['stage_ms_per_step'])"
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "lmax or normals_exact or configs or randomised" -p no:cacheprovider 2>&1 | tail -2
