# Round-2 measurement sweeps (run under gpurun from the repo root):
#   bash tools/gpu_sweeps.sh strip TAG       kNN strip pre-test: shapes (AIDW_KNN_VARIANT) and
#                                            strip on/off (AIDW_KNN_STRIP) at C4 sizes, C3, C5
#   bash tools/gpu_sweeps.sh ksplit TAG      kNN seeded split factor (AIDW_SPLIT) at C4 and the shares
#   bash tools/gpu_sweeps.sh tail TAG        weighting pass: wave quantisation (time per query
#                                            at grids of 32.0 .. 48.05 waves)
#   bash tools/gpu_sweeps.sh ncu_interp TAG  ncu --set full of the weighting kernel + its
#                                            SASS source page (stall samples per instruction)
#   bash tools/gpu_sweeps.sh ncu_knn TAG     the same for the kNN kernel
cd "${GRAFT_REPO_ROOT:-.}"
MODE=${1:?mode}
O=gpurun_out/${2:-$MODE}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
case $MODE in
strip)
  for nq in 1024000 512000 128000 32768; do
    for v in 0 25 31 26; do timeout 300 env AIDW_KNN_VARIANT=$v python tools/tune_knn.py $nq --check >> $O/tune.log 2>&1; done
    timeout 300 env AIDW_KNN_STRIP=0 python tools/tune_knn.py $nq | sed 's/^/strip0 /' >> $O/tune.log 2>&1
  done
  for c in C3 C5; do
    timeout 300 env TUNE_CFG=$c python tools/tune_knn.py >> $O/tune.log 2>&1
    timeout 300 env TUNE_CFG=$c AIDW_KNN_STRIP=0 python tools/tune_knn.py | sed 's/^/strip0 /' >> $O/tune.log 2>&1
  done
  timeout 900 python -m pytest tests -m gpu -q -k "h16 or golden or knn" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
  ;;
ksplit)
  for nq in 1024000 512000 128000; do
    for sp in auto 0 2 3 4 5 6 8; do
      if [ $sp = auto ]; then timeout 300 python tools/tune_knn.py $nq >> $O/tune.log 2>&1
      else timeout 300 env AIDW_SPLIT=$sp python tools/tune_knn.py $nq >> $O/tune.log 2>&1; fi
    done
  done
  ;;
tail)
  for nq in 1024000 1022976 1017856 1011712 1000000 989184 682240 681984; do
    timeout 300 python tools/tune_interp.py $nq >> $O/tail.log 2>&1
  done
  ;;
ncu_interp)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"interp_f32x2" -c 1 -o $O/prof_interp \
      python bench.py --profile --warmup 0 > $O/ncu.log 2>&1
  ncu -i $O/prof_interp.ncu-rep --page source --csv --print-source sass > $O/source_sass.csv 2>/dev/null
  ;;
ncu_knn)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"knn_filter" -c 1 -o $O/prof_knn \
      python bench.py --profile --warmup 0 > $O/ncu.log 2>&1
  ncu -i $O/prof_knn.ncu-rep --page source --csv --print-source sass > $O/source_sass.csv 2>/dev/null
  rm -f $O/prof_knn.ncu-rep
  ;;
esac
rm -f $O/*.ncu-rep
echo done
