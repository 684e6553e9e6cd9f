cd $GRAFT_REPO_ROOT
for i in 1 2; do
timeout 300 python bench.py --workload C3 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-strict > gpurun_out/qx2.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/qx2.json')); print(round(d['value'],1), d['stage_ms_per_step'], d['roofline']['frac'])"
done
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
