# evidence refresh (v13): build, then the round3 set (smoke, pytest -m gpu, configs, bench
# global/fixed/fixed3/f64, ncu launch list + full captures, pipe peaks) + strong shares
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-v13}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash tools/gpu_round3.sh ${TAG}
for nq in 512000 256000 128000; do
  timeout 300 python bench.py --nq $nq --no-cpu-baseline --no-e2e > gpurun_out/strong_share_${nq}_${TAG}.json 2>/dev/null
done
python tools/configs_bench.py --configs C1,C2,C3 --dtypes f64 --out gpurun_out/configs_f64_${TAG}.json > /dev/null 2>&1
echo done
