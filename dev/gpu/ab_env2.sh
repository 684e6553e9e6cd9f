# bench-only A/B over environment switches (prints value + ms_per_step)
cd $GRAFT_REPO_ROOT
for v in "" "$@"; do
  env $v timeout 600 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab.err || { echo "$v failed"; tail -3 gpurun_out/ab.err; continue; }
  python -c "import json,sys; d=json.load(open('gpurun_out/ab.json')); print(sys.argv[1] or 'default', round(d['value'],1), round(d['ms_per_step'],4), d['stage_ms_per_step'])" "$v"
done
