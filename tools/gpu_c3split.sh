# C3 (clustered, k = 15) kNN against the seeded split factor (AIDW_SPLIT forces it)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for s in auto 0 2 3 4 5 6 7 8; do
  if [ $s = auto ]; then TUNE_CFG=C3 timeout 120 python tools/tune_knn.py --check; else AIDW_SPLIT=$s TUNE_CFG=C3 timeout 120 python tools/tune_knn.py --check; fi
done > gpurun_out/c3split.log 2>&1
for n in 32768 50000 65536 200000; do
  for s in auto 0; do
    if [ $s = auto ]; then TUNE_CFG=C4 timeout 120 python tools/tune_knn.py $n; else AIDW_SPLIT=$s TUNE_CFG=C4 timeout 120 python tools/tune_knn.py $n; fi
  done
done >> gpurun_out/c3split.log 2>&1
echo done
