# tests + configs + bench (under gpurun)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -rA > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python tools/configs_bench.py --configs C2,C3,C4 > gpurun_out/configs.jsonl 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -2 gpurun_out/smoke.log
grep -E "FAIL|Error|error" gpurun_out/pytest_gpu.log | head -20
tail -2 gpurun_out/pytest_gpu.log
python - <<'P'
import json
for l in open("gpurun_out/configs.jsonl"):
    try: r=json.loads(l)
    except Exception: print(l.strip()); continue
    print(r["config"], r["dtype"], "knn %.3f alpha %.3f interp %.3f total %.3f ms" % (r["knn_ms"], r["alpha_ms"], r["interp_ms"], r["total_ms"]))
r=json.loads(open("gpurun_out/bench.json").read())
print("bench", r["value"], r["ms_per_step"], r["phases_ms"], r["roofline"]["frac"], r["roofline"].get("path_frac"), r["clocks"])
P
timeout 600 python bench.py --mode fixed --no-cpu-baseline --no-e2e > gpurun_out/bench_fixed.json 2> gpurun_out/bench_fixed.err
python -c "
import json;r=json.load(open('gpurun_out/bench_fixed.json'))
print('fixed', r['value'], r['ms_per_step'], r.get('phases_ms'))"
