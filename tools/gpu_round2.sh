# evidence refresh: tests, configs C1-C5, bench (global/fixed/fixed3), ncu launch list + full captures
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-v10}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rA > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python tools/configs_bench.py --out gpurun_out/configs_${TAG}.json > gpurun_out/configs.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench.err
timeout 600 python bench.py --mode fixed > gpurun_out/bench_fixed_${TAG}.json 2>> gpurun_out/bench.err
timeout 600 python bench.py --mode fixed3 > gpurun_out/bench_fixed3_${TAG}.json 2>> gpurun_out/bench.err
bash tools/gpu_profile.sh ${TAG} > /dev/null 2>&1
tail -2 gpurun_out/smoke.log
tail -2 gpurun_out/pytest_gpu.log
cut -c1-200 gpurun_out/configs.log
for f in bench bench_fixed bench_fixed3; do cut -c1-200 gpurun_out/${f}_${TAG}.json; done
ls gpurun_out | grep ${TAG}
