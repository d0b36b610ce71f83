# GPU check (r02u): default fp16 kNN shapes -- tests + sizes
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r02u}
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu.py -q -rf -k "h16 or golden and C4 or graph or order or seed or split or C3" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for nq in 1024000 512000 256000 128000 32768; do timeout 120 python tools/tune_knn.py $nq >> $O/tune_knn.log 2>&1; done
echo done
