cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --exchange p2p --no-cpu-baseline > gpurun_out/bench_p2p1.json 2> gpurun_out/bench_p2p1.err
echo "n1 rc=$?"; python -c "
import json;r=json.load(open('gpurun_out/bench_p2p1.json'));print(r['value'], r['ms_per_step'], r['phases_ms'], r['e2e'], r['config']['bounds_exchange'])"; tail -2 gpurun_out/bench_p2p1.err
for ex in nccl p2p; do
AIDW_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29544 bench.py --gpus 2 --steps 3 --warmup 1 --nq 200000 --exchange $ex > gpurun_out/gloo2_$ex.json 2> gpurun_out/gloo2_$ex.err
echo "gloo2 $ex rc=$?"; python -c "
import json;r=json.load(open('gpurun_out/gloo2_$ex.json'));print(r['value'], r['ms_per_step'], r['phases_ms'], r['e2e']['value'], r['config']['bounds_exchange'])"; tail -2 gpurun_out/gloo2_$ex.err
done
