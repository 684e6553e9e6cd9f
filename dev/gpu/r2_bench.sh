cd $GRAFT_REPO_ROOT
( time timeout 1200 python bench.py --steps 30 --warmup 5 ) > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
tail -5 gpurun_out/bench_full.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_full.json").read().strip().splitlines()[-1])
print("value", round(d["value"], 1), "e2e", {k: (round(v["value"], 1) if isinstance(v, dict) and "value" in v else None) for k, v in d["e2e"].items() if isinstance(v, dict)}, round(d["e2e"]["value"], 1))
print("strict", d["strict"])
print("parity", json.dumps(d["parity"], indent=1))
print("cpu", d["cpu_baseline"])
PY
#( time timeout 900 python bench.py --impl reference --steps 200 --warmup 5 ) > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
#tail -4; cut -c1-600 gpurun_out/bench_ref.json
