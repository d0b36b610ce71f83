# GPU sweep (r02w): weighting occupancy variants (10 CTAs/SM at 48 registers)
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r02w}
mkdir -p $O
for v in 0 39 40 41; do AIDW_INTERP_VARIANT=$v timeout 120 python tools/tune_interp.py >> $O/tune_interp.log 2>&1; done
echo done
