# C3 configs check + ncu source-level capture of the C4 kNN kernel (under gpurun; one GPU)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-knnprof}
timeout 300 python tools/configs_bench.py --configs C2,C3 > gpurun_out/${TAG}_configs.jsonl 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:knn_filter_kernel -c 1 \
    -o gpurun_out/${TAG}_knn python bench.py --profile --warmup 0 > gpurun_out/${TAG}_knn.log 2>&1
ncu -i gpurun_out/${TAG}_knn.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_knn_sass.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/${TAG}_knn.ncu-rep --json gpurun_out/${TAG}_knn.json > /dev/null 2>&1
cut -c1-400 gpurun_out/${TAG}_configs.jsonl
ls -la gpurun_out | tail -5
