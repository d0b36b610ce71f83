mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for q in 0 1; do AIDW_INTERP_Q1=$q timeout 600 python tools/configs_bench.py --configs C2,C3 --dtypes f64; done > gpurun_out/q1f64.log 2>&1
echo done
