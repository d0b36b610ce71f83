cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-it}
nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/mix_bench.cu -o /tmp/mix_bench && /tmp/mix_bench > gpurun_out/${TAG}_mix.log 2>&1
cat gpurun_out/${TAG}_mix.log
for v in ${KVARIANTS:-0}; do AIDW_KNN_VARIANT=$v timeout 300 python tools/tune_knn.py --check; done > gpurun_out/${TAG}_knn.log 2>&1
cat gpurun_out/${TAG}_knn.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/${TAG}_pytest.log 2>&1
tail -3 gpurun_out/${TAG}_pytest.log
