# Strip pre-test evaluation (run under gpurun from the repo root): bash tools/gpu_strip.sh TAG
cd "${GRAFT_REPO_ROOT:-.}"
TAG=${1:-strip}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 900 python -m pytest tests -m gpu -q -rf -k "h16 or knn or golden or seed or split" > $O/pytest_knn.log 2>&1; echo rc=$? >> $O/pytest_knn.log
for nq in 1024000 128000 32768; do
  for v in 0 31 24 25 26 27 28 29 30; do
    AIDW_KNN_VARIANT=$v timeout 300 python tools/tune_knn.py $nq >> $O/tune.log 2>&1
  done
  AIDW_KNN_STRIP=0 timeout 300 python tools/tune_knn.py $nq | sed 's/^/strip0 /' >> $O/tune.log 2>&1
done
TUNE_CFG=C3 timeout 300 python tools/tune_knn.py >> $O/tune.log 2>&1
TUNE_CFG=C3 AIDW_KNN_STRIP=0 timeout 300 python tools/tune_knn.py | sed 's/^/strip0 /' >> $O/tune.log 2>&1
echo done
