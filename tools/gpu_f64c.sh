cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/f64c_pytest.log 2>&1
tail -15 gpurun_out/f64c_pytest.log | cut -c1-300
timeout 900 python tools/configs_bench.py --configs C1,C2,C3,C4 --dtypes f64 --out gpurun_out/configs_f64_v12.json 2>&1 | cut -c1-260
