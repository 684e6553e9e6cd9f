# C3 triangulation (normals + l_max fused): lmax tests, bench line, one ncu --set full capture
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -q -x -k "lmax or front_end_configs or golden_topology" -p no:cacheprovider 2>&1 | tail -3
timeout 600 python bench.py --workload C3 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/c3.json 2> gpurun_out/c3.err
python -c "import json; d=json.load(open('gpurun_out/c3.json')); print(round(d['value'],1), d['stage_ms_per_step'], d['kernels']['triangulate_kernel'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:triangulate_kernel -s 3 -c 1 -o gpurun_out/c3_tri -f python bench.py --workload C3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --frames 64 > gpurun_out/c3_ncu.log 2>&1; echo ncu rc=$?
