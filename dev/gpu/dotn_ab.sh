# A/B: dot-form normal term (OPCFE_BILATERAL_DOTN=1) vs difference form; parity under both
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
OPCFE_BILATERAL_DOTN=1 timeout 900 python -m pytest tests -m gpu -q --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/pytest_gpu_dotn.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_dotn.log
grep -E "FAILED|Error|passed|failed" gpurun_out/pytest_gpu_dotn.log | tail -8
for v in "" 1; do
env ${v:+OPCFE_BILATERAL_DOTN=1} timeout 900 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_dotn_$v.json 2> gpurun_out/bench_dotn.err
python - "$v" <<'PY'
import json,sys
d=json.load(open(f"gpurun_out/bench_dotn_{sys.argv[1]}.json")); print("dotn" if sys.argv[1] else "diff", round(d["value"],1), d["stage_ms_per_step"], d["roofline"]["frac"])
PY
done
