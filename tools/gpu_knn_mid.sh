cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for nq in 128000 256000 512000; do
  timeout 300 python tools/tune_knn.py $nq
  for v in 3 8 14 15; do AIDW_SPLIT=0 AIDW_KNN_VARIANT=$v timeout 300 python tools/tune_knn.py $nq; done
done > gpurun_out/knn_mid.log 2>&1
cat gpurun_out/knn_mid.log
