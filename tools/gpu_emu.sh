cd $GRAFT_REPO_ROOT
for v in 0 40 41 42 43 44; do AIDW_INTERP_VARIANT=$v timeout 300 python tools/tune_interp.py --check 2>&1 | tail -1; done
