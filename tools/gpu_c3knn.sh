cd $GRAFT_REPO_ROOT
for v in 0 16 17 18 19 20; do AIDW_KNN_VARIANT=$v TUNE_CFG=C3 timeout 300 python tools/tune_knn.py --check 2>&1 | tail -1; done
for v in 0 17 18; do AIDW_SPLIT=0 AIDW_KNN_VARIANT=$v TUNE_CFG=C3 timeout 300 python tools/tune_knn.py 2>&1 | tail -1; done
