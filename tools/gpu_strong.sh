# Strong scaling of C4 (BASELINE: 1M x 1M, 1 GPU vs 8 GPUs query-sharded): one rank's share
# timed on one GPU for P = 2, 4, 8, plus a 2-rank strong-scaling logic run (gloo, one GPU).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for nq in 512000 256000 128000; do
  timeout 300 python bench.py --nq $nq --no-cpu-baseline --no-e2e > gpurun_out/strong_share_$nq.json 2> gpurun_out/strong_share_$nq.err
done
AIDW_DIST_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --scaling strong --steps 3 --warmup 3 \
  --no-cpu-baseline > gpurun_out/strong_gloo2.json 2> gpurun_out/strong_gloo2.err
echo done
