cd $GRAFT_REPO_ROOT
for F in 8 16 32; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --frames $F > gpurun_out/fs.json 2> gpurun_out/fs.err || { tail -3 gpurun_out/fs.err; continue; }
  python -c "import json,sys; d=json.load(open('gpurun_out/fs.json')); F=int(sys.argv[1]); print(F, round(d['value'],1), round(d['ms_per_step']/F,4), d['clocks']['sm_mhz'])" $F
done
