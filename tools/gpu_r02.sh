# Round-2 evidence run on one B200 (run under gpurun from the repo root):
#   bash tools/gpu_r02.sh TAG [quick]
# build + smoke, pytest -m gpu, bench (C4 default line with the fp64 sub-record, e2e,
# e2e_full, CPU baselines), C5 strong N=1, a 2-rank gloo logic run of the strong-scaled
# bench (ranks share the GPU: logic only), pipe peaks, the ncu launch list of the bench
# step and ncu --set full captures of the two O(nq nd) kernels with the pipe counters
# `full` leaves out (tools/ncu_summary.py), the reference (oracle) arm.
cd "${GRAFT_REPO_ROOT:-.}"
TAG=${1:-r02}
MODE=${2:-full}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
if [ "$MODE" = "quick" ]; then echo done; exit 0; fi
timeout 600 python bench.py --config C5 --steps 3 --no-f64 --no-cpu-baseline > $O/bench_c5.json 2>> $O/bench.err
AIDW_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu-baseline \
    --no-f64 > $O/bench_gloo2.json 2> $O/bench_gloo2.err
nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/pipe_peaks.cu -o /tmp/pipe_peaks && /tmp/pipe_peaks > $O/pipe_peaks.jsonl 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo tools/knn_loop_bench.cu -o /tmp/knn_loop_bench && timeout 300 /tmp/knn_loop_bench > $O/knn_loop_bench.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --profile --warmup 1 > /dev/null 2>&1
XM=sm__inst_executed_pipe_xu.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_fmalite.sum,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_active.avg
timeout 900 ncu --set full --metrics $XM --clock-control none --import-source on -k regex:"interp_f32x2|knn_filter" \
    -s 0 -c 2 -o $O/prof python bench.py --profile --warmup 0 > $O/ncu_full.log 2>&1
python tools/ncu_summary.py $O/prof.ncu-rep --json $O/ncu_summary.json > /dev/null 2>&1
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_ref.json 2>> $O/bench.err
echo done
