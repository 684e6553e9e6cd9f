# secondary bench lines for BASELINE.json's other configs (C1, C2, C3, C5) + the reference arm
cd $GRAFT_REPO_ROOT
for w in C1 C2 C3 C5; do
  timeout 600 python bench.py --workload $w --steps 50 --warmup 5 --no-e2e-files > gpurun_out/wl_$w.json 2> gpurun_out/wl_$w.err; echo "$w rc=$?"
  timeout 300 python bench.py --workload $w --impl reference --steps 3 --warmup 1 > gpurun_out/wl_${w}_ref.json 2> gpurun_out/wl_${w}_ref.err; echo "$w ref rc=$?"
done
python - <<'PY'
import json
for w in ["C1","C2","C3","C5"]:
    try:
        d = json.load(open(f"gpurun_out/wl_{w}.json")); r = json.load(open(f"gpurun_out/wl_{w}_ref.json"))
        print(w, round(d["value"],1), "e2e", round(d["e2e"]["value"],1), "ref", round(r["value"],2), d["stage_ms_per_step"], d["roofline"]["kernel"], d["roofline"]["frac"], d["clocks"]["sm_mhz"])
    except Exception as e:
        print(w, "ERR", e)
PY
