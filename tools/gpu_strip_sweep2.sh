# Strip group 128 vs 256 points, then the iteration evidence (run under gpurun)
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/${1:-strip_e}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for nq in 1024000 128000; do
 for s in 1 8; do AIDW_KNN_STRIP=$s timeout 300 python tools/tune_knn.py $nq --check | sed "s/^/strip$s /" >> $O/tune.log 2>&1; done
done
for s in 1 8; do TUNE_CFG=C3 AIDW_KNN_STRIP=$s timeout 300 python tools/tune_knn.py | sed "s/^/strip$s /" >> $O/tune.log 2>&1; done
AIDW_KNN_STRIP=8 timeout 600 python -m pytest tests -m gpu -q -k "h16 and not C5" > $O/pytest8.log 2>&1; echo rc=$? >> $O/pytest8.log
PYTEST_K="not C5" bash tools/gpu_eval.sh ${1:-strip_e}
