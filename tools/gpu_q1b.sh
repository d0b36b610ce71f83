mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "q1 or split or sharding or C1 or C2 or C3 or idw or graph" > gpurun_out/pytest_q1b.log 2>&1; echo rc=$? >> gpurun_out/pytest_q1b.log
for q in 0 1; do AIDW_INTERP_Q1=$q timeout 600 python tools/configs_bench.py --configs C2,C3; done > gpurun_out/q1b_cfg.log 2>&1
timeout 600 python tools/configs_bench.py --configs C1,C2,C3 > gpurun_out/q1b_auto.log 2>&1
for n in 20000 100000 128000; do timeout 120 python tools/tune_interp.py $n; done >> gpurun_out/q1b_auto.log 2>&1
echo done
