# GPU check (r02r): per-query seeds for the fp16 kNN -- tests + timing
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r02r}
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu.py -q -rf -k "h16 or golden and C4 or graph or order or seed or split or C3" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for qs in 1 0; do
  for nq in 1024000 128000; do AIDW_KNN_QSEED=$qs timeout 120 python tools/tune_knn.py $nq >> $O/tune_knn.log 2>&1; done
  AIDW_KNN_QSEED=$qs TUNE_CFG=C3 timeout 120 python tools/tune_knn.py >> $O/tune_knn.log 2>&1
done
echo done
