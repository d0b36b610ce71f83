# small-config launch lists under several tuning settings + pytest -m gpu
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
run() {  # $1 = tag, rest = env
  tag=$1; shift
  env "$@" timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/small_$tag.csv python tools/small_launches.py > gpurun_out/small_$tag.log 2>&1
}
run new AIDW_X=1
run oldq AIDW_INTERP_Q1=0
run ord0 AIDW_KNN_ORDER_MIN=1
run ord4k AIDW_KNN_ORDER_MIN=4096
timeout 600 python tools/configs_bench.py --configs C1,C2,C3 > gpurun_out/configs_small.log 2>&1
echo done
