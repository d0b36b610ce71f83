# seeded ordered kNN split: parity tests + C3/C4 kNN timings (under gpurun)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -q -x -k "order or split or sharding or graph" --timeout 600 > gpurun_out/seed_pytest.log 2>&1
tail -3 gpurun_out/seed_pytest.log
for s in default 0 2 3 5 7; do if [ $s = default ]; then timeout 300 python tools/tune_knn.py --check; else AIDW_SPLIT=$s timeout 300 python tools/tune_knn.py --check; fi | sed "s/^/split=$s /"; done > gpurun_out/seed_knn.log 2>&1
cat gpurun_out/seed_knn.log
timeout 300 python tools/configs_bench.py --configs C2,C3 2>&1 | cut -c1-300
