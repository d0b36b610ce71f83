cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
./tools/pipe_peaks > gpurun_out/pipe_peaks2.json 2>&1
for v in 1 2 3 4 5 6 7 8; do AIDW_INTERP_VARIANT=$v timeout 300 python tools/tune_interp.py $v 1024000 --check; done > gpurun_out/tune_interp.log 2>&1
cat gpurun_out/pipe_peaks2.json gpurun_out/tune_interp.log
