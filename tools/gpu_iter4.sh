cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-it}
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/${TAG}_pytest.log 2>&1
grep -E "FAILED|passed|failed" gpurun_out/${TAG}_pytest.log | tail -5
for v in ${KVARIANTS:-}; do AIDW_KNN_VARIANT=$v timeout 300 python tools/tune_knn.py --check; done
for v in ${IVARIANTS:-}; do AIDW_INTERP_VARIANT=$v timeout 300 python tools/tune_interp.py --check; done
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --mode fixed --no-cpu-baseline > gpurun_out/${TAG}_bench_fixed.json 2>> gpurun_out/${TAG}_bench.err
python -c "
import json
for f in ['gpurun_out/${TAG}_bench.json','gpurun_out/${TAG}_bench_fixed.json']:
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d['value'], d['ms_per_step'], d['phases_ms'], d['roofline']['frac'], d['roofline'].get('path_frac'), d['clocks'])
"
