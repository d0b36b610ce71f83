# ncu --set full of chosen kernels on the bench workload (under gpurun, 1 GPU)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-ncu}
for K in ${KERNELS:-knn_filter_kernel interp_f32x2_kernel}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 \
      -o gpurun_out/${TAG}_$K python bench.py --profile --warmup 0 > gpurun_out/${TAG}_$K.log 2>&1
done
ls -la gpurun_out | tail
