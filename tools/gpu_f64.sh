cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/configs_bench.py --configs C3,C4 --dtypes f64 --out gpurun_out/configs_f64.json > gpurun_out/configs_f64.log 2>&1
cut -c1-330 gpurun_out/configs_f64.log
