# precision-mixed stage times (best of 6) under alternating values of one environment
# switch: ab_env_mixed.sh VAR v1 v2 ...
cd $GRAFT_REPO_ROOT
VAR=$1; shift
for rep in 1 2; do for val in "$@"; do
env $VAR=$val PREC=${PREC:-mixed} timeout 300 python - <<'PY'
import os, torch, paper_2007_12065_b200 as fe
eng = fe.FrontEnd(1080, 1920, 16, laplacian=fe.LaplacianParams(1.0, 3, 10), bilateral=fe.BilateralParams(0.1, 0.15, 3, 5), src_dtype=torch.float32 if os.environ.get("SRC") == "f32" else torch.float64, graph=False, precision=os.environ["PREC"])
eng.src.copy_(torch.from_numpy(fe.synthetic.config_c4()).cuda().to(eng.src.dtype).expand_as(eng.src))
ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
for e in ev: e.record()
best = [1e9] * 4
for _ in range(6):
    eng.launch_profiled(ev); torch.cuda.synchronize()
    best = [min(b, ev[i].elapsed_time(ev[i + 1])) for i, b in enumerate(best)]
print({k: v for k, v in os.environ.items() if k.startswith("OPCFE_")}, "stage ms (in, lap, tri, bil)", [round(b, 3) for b in best])
PY
done; done
