cd $GRAFT_REPO_ROOT
for r in 1 2 4 8 16 1 4 8; do
OPCFE_QX_ROWS=$r timeout 300 python bench.py --workload C3 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-strict > gpurun_out/qx3.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/qx3.json')); print('rows=$r', round(d['value'],1), d['stage_ms_per_step']['triangulate'], d['roofline']['frac'])"
done
