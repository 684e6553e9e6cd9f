# the driver's default bench invocation once, summarised
cd $GRAFT_REPO_ROOT
( time timeout 900 python bench.py ) > gpurun_out/b1.json 2> gpurun_out/b1.err; echo "rc=$?"; tail -3 gpurun_out/b1.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/b1.json"))
print(round(d["value"],1), "e2e", round(d["e2e"]["value"],1), {k: (round(v["value"],1) if "value" in v else v) for k, v in d["e2e"].items() if isinstance(v, dict)}, "strict", round(d["strict"]["value"],1), "mixed", round(d["mixed"]["value"],1), d["mixed"]["stage_ms_per_step"], d["roofline"]["frac"], d["clocks"], d["stage_ms_per_step"])
print({k: v["normals_abs"] for k, v in d["parity"]["chained"].items() if isinstance(v, dict)})
PY
