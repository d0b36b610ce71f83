# ncu source-level capture of the C4 weighting kernel (under gpurun; one GPU)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-interpprof}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:interp_f32x2_kernel -c 1 \
    -o gpurun_out/${TAG} python bench.py --profile --warmup 0 > gpurun_out/${TAG}.log 2>&1
ncu -i gpurun_out/${TAG}.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sass.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/${TAG}.ncu-rep --json gpurun_out/${TAG}.json > /dev/null 2>&1
ncu -i gpurun_out/${TAG}.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ls -la gpurun_out | tail -4
