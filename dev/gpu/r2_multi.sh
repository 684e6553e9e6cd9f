cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_multidevice.py -q -p no:cacheprovider 2>&1 | tail -3
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --workload C5 --steps 5 --warmup 3 --share-gpus --no-e2e --no-strict > gpurun_out/multi_gloo.json 2> gpurun_out/multi_gloo.err
echo "gloo rc=$?"; tail -3 gpurun_out/multi_gloo.err; python -c "
import json; d=json.loads(open('gpurun_out/multi_gloo.json').read().strip().splitlines()[-1]); print(d['value'], d['n_gpus'], d['distributed'])"
NCCL_DEBUG=INFO OPCFE_DIST_BACKEND=nccl timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --workload C5 --steps 5 --warmup 3 --share-gpus --no-e2e --no-strict > gpurun_out/multi_nccl.json 2> gpurun_out/multi_nccl.err
echo "nccl rc=$?"; grep -iE "duplicate|error|nranks|comm " gpurun_out/multi_nccl.err | head -8; tail -c 600 gpurun_out/multi_nccl.json
