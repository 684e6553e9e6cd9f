cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench5.json 2> gpurun_out/bench5.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.load(open("gpurun_out/bench5.json")); print(round(d["value"],1), d["stage_ms_per_step"], d["e2e"]["value"], d["cpu_baseline"], d["roofline"], d["clocks"])
PY
