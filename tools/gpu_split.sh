cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -rA > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python tools/tune_split.py --out gpurun_out/split.jsonl > gpurun_out/split.log 2>&1
timeout 300 python tools/configs_bench.py --configs C1,C2,C3,C4 > gpurun_out/configs_split.jsonl 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/smoke.log
grep -E "FAIL|Error|error" gpurun_out/pytest_gpu.log | head -20
tail -3 gpurun_out/pytest_gpu.log
python - <<'P'
import json
for l in open("gpurun_out/split.jsonl"):
    r=json.loads(l); print(r["case"], r["nq"], r["split"], "knn %.3f interp %.3f" % (r["knn_ms"], r["interp_ms"]))
for l in open("gpurun_out/configs_split.jsonl"):
    try: r=json.loads(l)
    except Exception: print(l.strip()); continue
    print(r["config"], r["dtype"], "knn %.3f alpha %.3f interp %.3f total %.3f ms" % (r["knn_ms"], r["alpha_ms"], r["interp_ms"], r["total_ms"]))
P
cut -c1-400 gpurun_out/bench.json
