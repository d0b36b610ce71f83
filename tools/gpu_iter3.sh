cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-it}
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/${TAG}_pytest.log 2>&1
tail -5 gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --mode fixed --no-cpu-baseline > gpurun_out/${TAG}_bench_fixed.json 2>> gpurun_out/${TAG}_bench.err
AIDW_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 1 --nq 262144 > gpurun_out/${TAG}_bench_2rank.json 2> gpurun_out/${TAG}_bench_2rank.err
cat gpurun_out/${TAG}_bench.json gpurun_out/${TAG}_bench_fixed.json gpurun_out/${TAG}_bench_2rank.json
tail -5 gpurun_out/${TAG}_bench.err gpurun_out/${TAG}_bench_2rank.err
