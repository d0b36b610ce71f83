cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/pipe_peaks.cu -o /tmp/pipe_peaks && /tmp/pipe_peaks
