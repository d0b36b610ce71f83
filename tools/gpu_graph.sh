cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "graph" -rA > gpurun_out/pytest_graph.log 2>&1
tail -3 gpurun_out/pytest_graph.log; grep -E "Error|error" gpurun_out/pytest_graph.log | head -10
timeout 300 python tools/graph_bench.py --out gpurun_out/graph.json
