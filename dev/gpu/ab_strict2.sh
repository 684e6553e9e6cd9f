# strict-chain A/B of dev/ab/old.so vs new.so (stage times, best of 6, 3 alternations)
cd $GRAFT_REPO_ROOT
for L in old new old new old new; do
OPCFE_LIB=dev/ab/$L.so timeout 300 python - <<'PY'
import os, torch, paper_2007_12065_b200 as fe
eng = fe.FrontEnd(1080, 1920, 16, laplacian=fe.LaplacianParams(1.0, 3, 10), bilateral=fe.BilateralParams(0.1, 0.15, 3, 5), src_dtype=torch.float64, graph=False, precision=os.environ.get("PREC", "strict"))
eng.src.copy_(torch.from_numpy(fe.synthetic.config_c4()).cuda().expand_as(eng.src))
ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
for e in ev: e.record()
best = [1e9] * 4
for _ in range(6):
    eng.launch_profiled(ev); torch.cuda.synchronize()
    best = [min(b, ev[i].elapsed_time(ev[i + 1])) for i, b in enumerate(best)]
print(os.path.basename(os.environ["OPCFE_LIB"]), "stage ms (in, lap, tri, bil)", [round(b, 3) for b in best])
PY
done
