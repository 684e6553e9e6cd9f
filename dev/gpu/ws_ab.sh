# A/B: warp-specialised persistent bilateral (default) vs direct kernel; full GPU suite
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for v in "" 1; do
env ${v:+OPCFE_BILATERAL_DIRECT=1} timeout 900 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_ws_$v.json 2> gpurun_out/bench_ws.err
python - "$v" <<'PY'
import json,sys
d=json.load(open(f"gpurun_out/bench_ws_{sys.argv[1]}.json")); print("direct" if sys.argv[1] else "ws", round(d["value"],1), d["stage_ms_per_step"], d["roofline"]["frac"])
PY
done
