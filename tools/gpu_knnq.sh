# kNN Q/G for ordered batches of a strong-scaled size (nd = 1M, k = 10)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for n in 32768 65536 128000 256000; do
  for v in 0 7 3 9; do AIDW_KNN_VARIANT=$v TUNE_CFG=C4 timeout 120 python tools/tune_knn.py $n; done
done > gpurun_out/knnq.log 2>&1
echo done
