# quick GPU check (r02f): kNN fp16 pre-filter -- tests, timing sweep, ncu of the H16 kernel
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r02g}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu.py -q -rf -k "h16 or golden and C4 or order or seed or split or graph" > $O/pytest_h16.log 2>&1; echo rc=$? >> $O/pytest_h16.log
for m in 0 1 2; do
  for nq in 1024000 128000; do AIDW_KNN_H16=$m timeout 120 python tools/tune_knn.py $nq >> $O/tune_knn.log 2>&1; done
  AIDW_KNN_H16=$m TUNE_CFG=C3 timeout 120 python tools/tune_knn.py >> $O/tune_knn.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"knn_filter" -c 1 -o $O/prof_knn python bench.py --profile --warmup 0 > $O/ncu_knn.log 2>&1
python tools/ncu_summary.py $O/prof_knn.ncu-rep --json $O/ncu_knn_summary.json > /dev/null 2>&1
echo done
