cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in 0 6 7 8 9; do AIDW_KNN_VARIANT=$v timeout 300 python tools/tune_knn.py --check; done > gpurun_out/knn_variants.log 2>&1
cat gpurun_out/knn_variants.log
timeout 300 python tools/configs_bench.py --configs C2,C3 > gpurun_out/configs.jsonl 2>&1
cut -c1-250 gpurun_out/configs.jsonl
