mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "split or order or sharded or sharding or C1 or C2 or C3 or ragged or q1 or graph" > gpurun_out/pytest_merge.log 2>&1; echo rc=$? >> gpurun_out/pytest_merge.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/small_v13c.csv python tools/small_launches.py > gpurun_out/small_v13c.log 2>&1
TUNE_CFG=C4 timeout 300 python tools/tune_knn.py 128000 --check > gpurun_out/knn128k.log 2>&1
TUNE_CFG=C4 timeout 300 python tools/tune_knn.py --check >> gpurun_out/knn128k.log 2>&1
echo done
