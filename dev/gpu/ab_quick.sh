# bench-only A/B of dev/ab/old.so vs new.so (3 alternations)
cd $GRAFT_REPO_ROOT
for L in old new old new old new; do
OPCFE_LIB=dev/ab/$L.so timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-strict > gpurun_out/ab_$L.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/ab_$L.json')); print('$L', round(d['value'],1), d['stage_ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['samples'])"
done
