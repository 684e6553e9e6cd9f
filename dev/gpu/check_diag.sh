# full GPU suite + bench line + bilateral error diagnostic
cd $GRAFT_REPO_ROOT
bash dev/gpu/check.sh
timeout 600 python dev/diag_bil_err.py > gpurun_out/diag_err.jsonl 2> gpurun_out/diag_err.err
python - <<'PY'
import json
for l in open("gpurun_out/diag_err.jsonl"):
    d = json.loads(l); print(d["config"], "per_iter_max %.2e" % max(d["per_iter_max"]), "chained %.2e" % d["chained_max"], "over1e-5", d["chained_over_1e-5"], "p9999 %.2e" % d["chained_p9999"])
PY
