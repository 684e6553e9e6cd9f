cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench3.json 2> gpurun_out/bench3.err
python - <<'PY'
import json
d=json.load(open("gpurun_out/bench3.json")); print(round(d["value"],1), d["stage_ms_per_step"], d["roofline"]["kernel"], d["roofline"]["frac"], d["kernels"])
PY
