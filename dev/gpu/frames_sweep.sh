cd $GRAFT_REPO_ROOT
for F in 1 2 4 8; do
  timeout 600 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --frames $F > gpurun_out/fs.json 2> gpurun_out/fs.err || { tail -3 gpurun_out/fs.err; continue; }
  python -c "import json,sys; d=json.load(open('gpurun_out/fs.json')); F=int(sys.argv[1]); print(F, round(d['value'],1), {k: round(v/F,4) for k,v in d['stage_ms_per_step'].items()})" $F
done
