# calibrate the small-grid Q = 1 threshold of the weighting pass (nd = 1M, fp32)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for n in ${NQS:-2000 4096 8192 12000 16000 20000 30000 40000 60000}; do
  for q in 0 1; do AIDW_INTERP_Q1=$q timeout 120 python tools/tune_interp.py $n; done
done > gpurun_out/q1sweep.log 2>&1
echo done
