cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -q -x -k "float64 or f64 or C1 or C2" --timeout 600 > gpurun_out/f64_pytest.log 2>&1
tail -3 gpurun_out/f64_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python tools/configs_bench.py --configs C1,C2,C3,C4 --dtypes f64 --out gpurun_out/configs_f64_v11.json > gpurun_out/configs_f64.log 2>&1
cut -c1-330 gpurun_out/configs_f64.log
