# quick GPU check (r02e): pytest -m gpu, bench, weighting EMU sweep at C4
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r02e}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rf -x -k "not C5" > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline --no-f64 > $O/bench.json 2> $O/bench.err
for v in 0 26 36 37 38; do AIDW_INTERP_VARIANT=$v timeout 120 python tools/tune_interp.py >> $O/tune_interp.log 2>&1; done
AIDW_EXP2_CLAMP=1 timeout 120 python tools/tune_interp.py >> $O/tune_interp.log 2>&1
echo done
