# ncu evidence for the bench workload (run under gpurun; one GPU).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-prof}
# 1) launch list of the bench command (cold-cache, serialised: compare shares)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e \
    > gpurun_out/${TAG}_launches_bench.log 2>&1
# 2) full sets of the two hot kernels (one launch each)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:interp_kernel -c 1 \
    -o gpurun_out/${TAG}_interp python bench.py --profile --warmup 0 > gpurun_out/${TAG}_interp.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:knn_robs_kernel -c 1 \
    -o gpurun_out/${TAG}_knn python bench.py --profile --warmup 0 > gpurun_out/${TAG}_knn.log 2>&1
ls -la gpurun_out
