# Round-2 evidence refresh (run under gpurun from the repo root): bash tools/gpu_evidence.sh TAG
# compute-sanitizer memcheck/synccheck/racecheck over tools/sanitize.py, every BASELINE config
# per stage (tools/configs_bench.py, both precisions), strong-scaling shares of C4 (one
# rank's block timed on one GPU), ncu --set full of the kNN and weighting kernels (separate
# invocations; the weighting's XU counters in their own --metrics pass).
cd "${GRAFT_REPO_ROOT:-.}"
TAG=${1:-r02i}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py > $O/sanitizer_$tool.log 2>&1
  echo "rc=$?" >> $O/sanitizer_$tool.log
done
timeout 900 python tools/configs_bench.py --out $O/configs_f32.json > $O/configs.log 2>&1
timeout 900 python tools/configs_bench.py --configs C1,C2,C3,C4 --dtypes f64 --out $O/configs_f64.json >> $O/configs.log 2>&1
for nq in 512000 256000 128000; do
  timeout 300 python bench.py --nq $nq --no-cpu-baseline --no-e2e --no-f64 > $O/strong_share_$nq.json 2>> $O/bench.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"knn_filter" -c 1 -o $O/prof_knn python bench.py --profile --warmup 0 > $O/ncu_knn.log 2>&1
python tools/ncu_summary.py $O/prof_knn.ncu-rep --json $O/ncu_knn_summary.json > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"interp_f32x2" -c 1 -o $O/prof_interp python bench.py --profile --warmup 0 > $O/ncu_interp.log 2>&1
python tools/ncu_summary.py $O/prof_interp.ncu-rep --json $O/ncu_interp_summary.json > /dev/null 2>&1
XM=sm__inst_executed_pipe_xu.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_fmalite.sum,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_active.avg,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $XM --clock-control none -k regex:"interp_f32x2|knn_filter" -c 2 --csv --page raw python bench.py --profile --warmup 0 > $O/ncu_xu.csv 2> $O/ncu_xu.err
echo done
