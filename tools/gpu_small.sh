# ncu launch list of the small configs' whole GLOBAL path (tools/small_launches.py)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --csv \
  --log-file gpurun_out/small_launches.csv python tools/small_launches.py > gpurun_out/small.log 2>&1
echo rc=$? >> gpurun_out/small.log
