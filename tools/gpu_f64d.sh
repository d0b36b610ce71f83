cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/f64d_pytest.log 2>&1
grep -E "FAIL|Error" gpurun_out/f64d_pytest.log | head; tail -2 gpurun_out/f64d_pytest.log
