# whole GPU suite + smoke on the shipped tree
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fc_smoke.log 2>&1; tail -1 gpurun_out/fc_smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fc_pytest.log 2>&1; tail -3 gpurun_out/fc_pytest.log
