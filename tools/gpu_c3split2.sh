mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "C3 or order or split or seed or sharding" > gpurun_out/pytest_c3.log 2>&1; echo rc=$? >> gpurun_out/pytest_c3.log
timeout 900 python tools/configs_bench.py --configs C3,C4 > gpurun_out/c3split2.log 2>&1
timeout 900 python tools/configs_bench.py --configs C3 --dtypes f64 >> gpurun_out/c3split2.log 2>&1
AIDW_SPLIT=7 timeout 900 python tools/configs_bench.py --configs C3 --dtypes f64 >> gpurun_out/c3split2.log 2>&1
for n in 32768 128000; do TUNE_CFG=C4 timeout 120 python tools/tune_knn.py $n; done >> gpurun_out/c3split2.log 2>&1
echo done
