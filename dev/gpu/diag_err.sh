cd $GRAFT_REPO_ROOT
for v in "" OPCFE_BILATERAL_DOTN=1 OPCFE_BILATERAL_WS=1; do
env $v timeout 600 python dev/diag_bil_err.py >> gpurun_out/diag_err.jsonl 2>> gpurun_out/diag_err.err
done
cat gpurun_out/diag_err.jsonl
