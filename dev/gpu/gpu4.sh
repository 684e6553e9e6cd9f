cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench2.json 2> gpurun_out/bench2.err
OPCFE_BILATERAL_DIRECT=1 timeout 900 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench2_direct.json 2>> gpurun_out/bench2.err
python - <<'PY'
import json
for f in ("gpurun_out/bench2.json","gpurun_out/bench2_direct.json"):
    try:
        d=json.load(open(f)); print(f, round(d["value"],1), d["stage_ms_per_step"], d["roofline"]["kernel"], d["roofline"]["frac"])
    except Exception as e: print(f, e)
PY
