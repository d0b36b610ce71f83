mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "seed or split or order or sharded or sharding or C1 or C2 or C3 or ragged or q1 or graph or filter or coincident or empty or single" > gpurun_out/pytest_seed.log 2>&1; echo rc=$? >> gpurun_out/pytest_seed.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/small_v13d.csv python tools/small_launches.py > gpurun_out/small_v13d.log 2>&1
for n in 2000 4096 10240 20000 30000; do
  AIDW_KNN_SEED=0 TUNE_CFG=C2 timeout 120 python tools/tune_knn.py $n --check >> gpurun_out/tune_seed.log 2>&1
  TUNE_CFG=C2 timeout 120 python tools/tune_knn.py $n --check >> gpurun_out/tune_seed.log 2>&1
done
for n in 16000 128000 1024000; do
  TUNE_CFG=C4 timeout 300 python tools/tune_knn.py $n --check >> gpurun_out/tune_seed.log 2>&1
done
echo done
