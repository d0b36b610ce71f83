# Iteration evidence (run under gpurun from the repo root): bash tools/gpu_eval.sh TAG
# build + smoke, pytest -m gpu (C5 golden deselected while it is generated), the default
# bench line, the ncu launch list, one ncu --set full capture of the kNN, the XU pass.
cd "${GRAFT_REPO_ROOT:-.}"
TAG=${1:-eval}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -rf ${PYTEST_K:+-k "$PYTEST_K"} > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --profile --warmup 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"knn_filter" -c 1 -o $O/prof_knn python bench.py --profile --warmup 0 > $O/ncu_knn.log 2>&1
python tools/ncu_summary.py $O/prof_knn.ncu-rep --json $O/ncu_knn_summary.json > /dev/null 2>&1
echo done
