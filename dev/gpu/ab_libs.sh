# bench A/B across alternative library builds in dev/ab/ (OPCFE_LIB)
cd $GRAFT_REPO_ROOT
for L in "" dev/ab/*.so; do
  env ${L:+OPCFE_LIB=$PWD/$L} timeout 600 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab.err || { echo "$L failed"; tail -3 gpurun_out/ab.err; continue; }
  python -c "import json,sys; d=json.load(open('gpurun_out/ab.json')); print(sys.argv[1] or 'default', round(d['value'],1), d['stage_ms_per_step'])" "$L"
done
