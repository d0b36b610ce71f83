cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(nproc; nvidia-smi -L; lscpu | grep "Model name") > gpurun_out/box.txt 2>&1
./tools/pipe_peaks > gpurun_out/pipe_peaks.json 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rA > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -5 gpurun_out/pytest_gpu.log
cat gpurun_out/bench.json
