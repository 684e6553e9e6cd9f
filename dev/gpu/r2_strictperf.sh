cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_strict.py -q -x -p no:cacheprovider 2>&1 | tail -2
python profiles/strict_driver.py --frames 16 --steps 4
python - <<'PY'
import torch, paper_2007_12065_b200 as fe
eng = fe.FrontEnd(1080, 1920, 16, laplacian=fe.LaplacianParams(1.0, 3, 10), bilateral=fe.BilateralParams(0.1, 0.15, 3, 5), src_dtype=torch.float32, graph=False, precision="strict")
eng.src.copy_(torch.from_numpy(fe.synthetic.config_c4()).cuda().float().expand_as(eng.src))
ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
for e in ev: e.record()
for _ in range(3): eng.launch_profiled(ev)
torch.cuda.synchronize()
print("stages ms", [round(ev[i].elapsed_time(ev[i+1]), 3) for i in range(4)])
PY
