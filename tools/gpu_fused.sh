cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for o in 1 0; do
AIDW_KNN_ORDER=$o timeout 600 python bench.py --mode fixed --no-cpu-baseline --no-e2e > gpurun_out/bench_fixed_$o.json 2> gpurun_out/bench_fixed.err
python -c "
import json;r=json.load(open('gpurun_out/bench_fixed_$o.json'))
print('order=$o', r['value'], r['ms_per_step'], r.get('phases_ms'))"
done
timeout 600 python bench.py --mode fixed3 --no-cpu-baseline --no-e2e > gpurun_out/bench_fixed3.json 2> gpurun_out/bench_fixed.err
python -c "
import json;r=json.load(open('gpurun_out/bench_fixed3.json'))
print('fixed3', r['value'], r['ms_per_step'], r.get('phases_ms'))"
