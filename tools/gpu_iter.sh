# quick iteration: GPU tests + interp variant sweep + bench (under gpurun)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-iter}
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/${TAG}_pytest.log 2>&1
tail -3 gpurun_out/${TAG}_pytest.log
for v in ${VARIANTS:-0}; do AIDW_INTERP_VARIANT=$v timeout 300 python tools/tune_interp.py 1024000 --check; done > gpurun_out/${TAG}_tune.log 2>&1
cat gpurun_out/${TAG}_tune.log
AIDW_KNN_FILTER=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_nofilter.json 2>&1
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
cat gpurun_out/${TAG}_bench_nofilter.json gpurun_out/${TAG}_bench.json
