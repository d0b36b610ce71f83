mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "order or split or sharding or C3 or graph or fused or filter" > gpurun_out/pytest_ord.log 2>&1; echo rc=$? >> gpurun_out/pytest_ord.log
run() {  # $1 = tag, rest = env
  tag=$1; shift
  env "$@" timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/small_$tag.csv python tools/small_launches.py > gpurun_out/small_$tag.log 2>&1
}
run v13b AIDW_X=1
run v13b_ord1 AIDW_KNN_ORDER_MIN=1
run v13b_ord2k AIDW_KNN_ORDER_MIN=2048
for n in 4096 10240 20000; do
  AIDW_KNN_ORDER_MIN=1 TUNE_CFG=C2 timeout 120 python tools/tune_knn.py $n --check >> gpurun_out/tune_small.log 2>&1
  TUNE_CFG=C2 timeout 120 python tools/tune_knn.py $n --check >> gpurun_out/tune_small.log 2>&1
done
timeout 900 python tools/configs_bench.py --configs C3,C4 > gpurun_out/configs_c34.log 2>&1
echo done
