cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() { timeout 300 python tools/tune_knn.py "$@" 2>&1 | tail -1; }
for s in 0 2 3 4 5 8; do AIDW_SPLIT=$s run 128000; done
unset AIDW_SPLIT; run 128000
for s in 0 2 3 5 7; do AIDW_SPLIT=$s TUNE_CFG=C3 run; done
TUNE_CFG=C3 run
for s in 0 2 3 5; do AIDW_SPLIT=$s run 256000; done
