# quick GPU checks (r02c): kNN loop microbenchmark, ncu of the weighting kernel with the
# XU counters (own invocation), pytest -m gpu
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r02c}
mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo tools/knn_loop_bench.cu -o /tmp/knn_loop_bench && timeout 300 /tmp/knn_loop_bench > $O/knn_loop_bench.jsonl 2>&1
XM=sm__inst_executed_pipe_xu.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_fmalite.sum,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_active.avg,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $XM --clock-control none -k regex:"interp_f32x2" -c 1 --csv --page raw python bench.py --profile --warmup 0 > $O/ncu_interp_xu.csv 2> $O/ncu_interp_xu.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"interp_f32x2" -c 1 -o $O/prof_interp python bench.py --profile --warmup 0 > $O/ncu_interp_full.log 2>&1
python tools/ncu_summary.py $O/prof_interp.ncu-rep --json $O/ncu_interp_summary.json > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
echo done
