# Round-2 final evidence (run under gpurun from the repo root): bash tools/gpu_final_r02.sh TAG
# build + smoke, pytest -m gpu (C4 + C5 golden), the default bench line, C5 strong N = 1,
# a 2-rank gloo logic run of the default bench (ranks share the GPU), the reference
# (oracle) arm, the ncu launch list of the bench step, ncu captures of the kNN and the
# weighting kernel, the C4 strong-scaling shares, every config per stage, the Table-1 ablation.
cd "${GRAFT_REPO_ROOT:-.}"
TAG=${1:-r02final}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 1800 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --config C5 --steps 3 --no-f64 --no-cpu-baseline > $O/bench_c5.json 2>> $O/bench.err
AIDW_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 3 --warmup 3 > $O/bench_gloo2.json 2> $O/bench_gloo2.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_ref.json 2>> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --profile --warmup 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"knn_filter" -c 1 -o $O/prof_knn python bench.py --profile --warmup 0 > $O/ncu_knn.log 2>&1
python tools/ncu_summary.py $O/prof_knn.ncu-rep --json $O/ncu_knn_summary.json > /dev/null 2>&1
XM=sm__inst_executed_pipe_xu.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_fmalite.sum,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_active.avg,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $XM --clock-control none -k regex:"interp_f32x2|knn_filter" -c 2 --csv --page raw python bench.py --profile --warmup 0 > $O/ncu_xu.csv 2> $O/ncu_xu.err
# strong-scaling shares of C4: each rank's block (1,024,000 / P queries) timed alone
for share in 512000 256000 128000; do
  timeout 600 python bench.py --nq $share --no-f64 --no-cpu-baseline --no-e2e > $O/share_$share.json 2>> $O/bench.err
done
python tools/strong_shares.py $O/bench.json $O/share_512000.json $O/share_256000.json $O/share_128000.json \
    > $O/strong_shares.json 2>> $O/bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"interp_f32x2" -c 1 -o $O/prof_interp python bench.py --profile --warmup 0 > $O/ncu_interp.log 2>&1
python tools/ncu_summary.py $O/prof_interp.ncu-rep --json $O/ncu_interp_summary.json > /dev/null 2>&1
timeout 900 python tools/configs_bench.py --out $O/configs_f32.json > $O/configs.log 2>&1
timeout 900 python tools/configs_bench.py --configs C1,C2,C3,C4 --dtypes f64 --out $O/configs_f64.json >> $O/configs.log 2>&1
timeout 1200 python tools/table1.py --out $O/table1.md --json $O/table1.jsonl > $O/table1.log 2>&1
rm -f $O/*.ncu-rep  # summaries kept; gpurun copies back <= 64 MiB
echo done
