# the driver's default bench invocation + the reference arm, as recorded for the round
cd $GRAFT_REPO_ROOT
timeout 900 python bench.py > gpurun_out/full_bench.json 2> gpurun_out/full_bench.err; echo "rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/full_ref.json 2> gpurun_out/full_ref.err; echo "ref rc=$?"
python -m json.tool gpurun_out/full_bench.json | head -120
cat gpurun_out/full_ref.json
