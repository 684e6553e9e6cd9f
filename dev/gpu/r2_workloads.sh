# round-2 record: the driver's default invocation + reference arm (C4), then C1/C2/C3/C5
cd $GRAFT_REPO_ROOT
( time timeout 900 python bench.py ) > gpurun_out/r2_full.json 2> gpurun_out/r2_full.err; echo "full rc=$?"; tail -3 gpurun_out/r2_full.err
( time timeout 900 python bench.py --impl reference ) > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err; echo "ref rc=$?"; tail -3 gpurun_out/r2_ref.err
for w in C1 C2 C3 C5; do
  timeout 600 python bench.py --workload $w --steps 50 --warmup 5 --no-e2e-files > gpurun_out/r2_wl_$w.json 2> gpurun_out/r2_wl_$w.err; echo "$w rc=$?"
  timeout 300 python bench.py --workload $w --impl reference --steps 3 --warmup 1 > gpurun_out/r2_wl_${w}_ref.json 2> gpurun_out/r2_wl_${w}_ref.err; echo "$w ref rc=$?"
done
python - <<'PY'
import json
d = json.load(open("gpurun_out/r2_full.json")); r = json.load(open("gpurun_out/r2_ref.json"))
print("C4", round(d["value"],1), "e2e", round(d["e2e"]["value"],1), {k: round(v["value"],1) for k, v in d["e2e"].items() if isinstance(v, dict) and "value" in v}, "strict", round(d["strict"]["value"],1), "ref", round(r["value"],2), d["roofline"]["frac"], d["clocks"])
for w in ["C1","C2","C3","C5"]:
    try:
        d = json.load(open(f"gpurun_out/r2_wl_{w}.json")); r = json.load(open(f"gpurun_out/r2_wl_{w}_ref.json"))
        print(w, round(d["value"],1), "e2e", round(d["e2e"]["value"],1), "strict", d["strict"] and round(d["strict"]["value"],1), "mixed", d.get("mixed") and round(d["mixed"]["value"],1), "ref", round(r["value"],2), d["stage_ms_per_step"], d["roofline"]["kernel"], d["roofline"]["frac"], d["clocks"]["sm_mhz"])
        print("   parity", json.dumps(d["parity"]["chained"]["fast"]["normals_abs"] if d.get("parity") else None), json.dumps(d["parity"]["chained"]["strict"]["normals_abs"] if d.get("parity") else None))
    except Exception as e:
        print(w, "ERR", e)
PY
