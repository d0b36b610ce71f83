cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sanitizer
for tool in memcheck synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 7 python tools/sanitize.py > gpurun_out/sanitizer/r01_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitizer/r01_$tool.log
done
# 2-rank logic test of the multi-GPU bench path (gloo, ranks share the one GPU)
AIDW_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --nq 200000 --no-e2e > gpurun_out/gloo2.json 2> gpurun_out/gloo2.err
echo "gloo2 rc=$?"; cut -c1-300 gpurun_out/gloo2.json; tail -3 gpurun_out/gloo2.err
