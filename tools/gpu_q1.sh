mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "q1 or split or sharding or C1 or C2 or idw" > gpurun_out/pytest_q1.log 2>&1; echo rc=$? >> gpurun_out/pytest_q1.log
timeout 900 python tools/configs_bench.py --out gpurun_out/configs_v13.json > gpurun_out/configs_v13.log 2>&1
timeout 900 python tools/graph_bench.py --out gpurun_out/graph_v13.json > gpurun_out/graph_v13.log 2>&1
echo done
