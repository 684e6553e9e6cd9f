cd $GRAFT_REPO_ROOT
for w in C1 C3; do for cfg in "8 16" "32 64" "64 128"; do set -- $cfg
OPCFE_SLOT_MB=$1 OPCFE_SLOT_MAX=$2 timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e-files --no-cpu-baseline --no-strict --no-e2e-dropin > gpurun_out/e2e_$w.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/e2e_$w.json')); e=d['e2e']; print('$w slot_mb=$1 max=$2', round(e['value'],1), 'frames/run', e['frames_per_step'], 'compact', round(e['compact']['value'],1), 'selected', round(e['selected']['value'],1))"
done; done
