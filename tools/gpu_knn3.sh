cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in 8 3 16 17 18 19; do AIDW_KNN_VARIANT=$v timeout 300 python tools/tune_knn.py --check; done > gpurun_out/knn_variants.log 2>&1
cat gpurun_out/knn_variants.log
