# GPU suite (default build) + bench A/B over environment switches: bash dev/gpu/ab_env.sh VAR=1 [VAR2=1 ...]
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
grep -E "FAILED|passed|failed|rc=" gpurun_out/pytest_gpu.log | tail -3
for v in "" "$@"; do
  env $v timeout 600 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab.err || { echo "$v failed"; tail -3 gpurun_out/ab.err; continue; }
  python -c "import json,sys; d=json.load(open('gpurun_out/ab.json')); print(sys.argv[1] or 'default', round(d['value'],1), d['stage_ms_per_step'])" "$v"
done
