# GPU check (r02h): full pytest -m gpu, bench (fp32 + fp64 sub-record), launch list
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r02h}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --profile --warmup 1 --no-f64 > /dev/null 2>&1
echo done
