cd $GRAFT_REPO_ROOT
for L in dev/ab/lib_*.so; do
OPCFE_LIB=$L python - <<'PY'
import os, torch, paper_2007_12065_b200 as fe
eng = fe.FrontEnd(1080, 1920, 16, laplacian=fe.LaplacianParams(1.0, 3, 10), bilateral=fe.BilateralParams(0.1, 0.15, 3, 5), src_dtype=torch.float32, graph=False, precision="strict")
eng.src.copy_(torch.from_numpy(fe.synthetic.config_c4()).cuda().float().expand_as(eng.src))
ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
for e in ev: e.record()
best = 1e9
for _ in range(4):
    eng.launch_profiled(ev); torch.cuda.synchronize(); best = min(best, ev[3].elapsed_time(ev[4]))
print(os.environ["OPCFE_LIB"], "bilateral stage ms", round(best, 3))
PY
done
