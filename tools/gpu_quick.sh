# GPU check (r02n): pytest -m gpu (k = 15 fp16 pre-filter), configs C3 timing
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r02n}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rf -k "not C5" > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
timeout 600 python tools/configs_bench.py --configs C2,C3 --out $O/configs_c3.json > $O/configs.log 2>&1
echo done
