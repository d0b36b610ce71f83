# GPU A/B (r02v): ring refill by the last releasing warp (libaidw_ringlast.so) vs thread 0
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r02v}
mkdir -p $O
cp paper_1511_02186_b200/libaidw.so /tmp/libaidw_A.so
for lib in A B; do
  if [ $lib = B ]; then cp paper_1511_02186_b200/libaidw_ringlast.so paper_1511_02186_b200/libaidw.so; fi
  echo "== $lib" >> $O/ab.log
  timeout 120 python tools/tune_knn.py >> $O/ab.log 2>&1
  timeout 120 python tools/tune_knn.py 128000 >> $O/ab.log 2>&1
  timeout 120 python tools/tune_interp.py >> $O/ab.log 2>&1
  timeout 120 python tools/tune_interp.py 128000 >> $O/ab.log 2>&1
  if [ $lib = B ]; then timeout 900 python -m pytest tests/test_gpu.py -q -x -k "not C5" > $O/pytest_B.log 2>&1; echo rc=$? >> $O/pytest_B.log; fi
done
cp /tmp/libaidw_A.so paper_1511_02186_b200/libaidw.so
echo done
