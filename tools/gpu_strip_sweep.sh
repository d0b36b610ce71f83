# Strip group-size / kernel-shape sweep (run under gpurun from the repo root)
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/${1:-strip_d}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for nq in 1024000 512000 128000 32768; do
 for s in 1 4; do
  for v in 0 25 31 26; do AIDW_KNN_STRIP=$s AIDW_KNN_VARIANT=$v timeout 300 python tools/tune_knn.py $nq --check | sed "s/^/strip$s /" >> $O/tune.log 2>&1; done
 done
done
for s in 1 4; do TUNE_CFG=C3 AIDW_KNN_STRIP=$s timeout 300 python tools/tune_knn.py | sed "s/^/strip$s /" >> $O/tune.log 2>&1; done
for s in 1 4; do TUNE_CFG=C5 AIDW_KNN_STRIP=$s timeout 300 python tools/tune_knn.py | sed "s/^/strip$s /" >> $O/tune.log 2>&1; done
timeout 600 python -m pytest tests -m gpu -q -k "(h16 or golden) and not C5" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
AIDW_KNN_STRIP=4 timeout 600 python -m pytest tests -m gpu -q -k "(h16 or golden) and not C5" >> $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
