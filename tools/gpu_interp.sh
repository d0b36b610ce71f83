cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in 0 36 3; do AIDW_INTERP_VARIANT=$v timeout 300 python tools/tune_interp.py --check; done > gpurun_out/interp_variants.log 2>&1
cat gpurun_out/interp_variants.log
