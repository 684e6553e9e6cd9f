# bench A/B across alternative library builds in dev/ab/ (OPCFE_LIB) on one workload: ab_wl.sh C3 [steps]
cd $GRAFT_REPO_ROOT
W=${1:-C4}; S=${2:-30}
for rep in 1 2; do
for L in "" dev/ab/*.so; do
  env ${L:+OPCFE_LIB=$PWD/$L} timeout 600 python bench.py --workload $W --steps $S --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab.err || { echo "$L failed"; tail -3 gpurun_out/ab.err; continue; }
  python -c "import json,sys; d=json.load(open('gpurun_out/ab.json')); print(sys.argv[1] or 'default', round(d['value'],1), d['stage_ms_per_step'])" "$L"
done
done
