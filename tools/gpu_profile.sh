# ncu evidence for the bench workload (run under gpurun; one GPU).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-prof}
# 1) launch list of the bench command (cold-cache, serialised: compare shares)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e \
    > gpurun_out/${TAG}_launches_bench.log 2>&1
# 2) full sets of the two hot kernels (one launch each)
for K in interp_f32x2_kernel knn_filter_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 \
      -o gpurun_out/${TAG}_$K python bench.py --profile --warmup 0 > gpurun_out/${TAG}_$K.log 2>&1
done
ls -la gpurun_out | tail -8
for K in interp_f32x2_kernel knn_filter_kernel; do
  python tools/ncu_summary.py gpurun_out/${TAG}_$K.ncu-rep --json gpurun_out/${TAG}_$K.json > /dev/null 2>&1
  ncu -i gpurun_out/${TAG}_$K.ncu-rep --page source --csv > gpurun_out/${TAG}_${K}_source.csv 2>/dev/null
done
