cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -rA > gpurun_out/pytest_gpu.log 2>&1
for v in 0 3 5 6 7; do AIDW_KNN_VARIANT=$v timeout 300 python tools/tune_knn.py --check; done > gpurun_out/knn_variants.log 2>&1
AIDW_KNN_ORDER=0 timeout 300 python tools/tune_knn.py >> gpurun_out/knn_variants.log 2>&1
timeout 300 python tools/configs_bench.py --configs C2,C3,C4 > gpurun_out/configs.jsonl 2>&1
grep -E "FAIL|Error|error" gpurun_out/pytest_gpu.log | head -20
tail -3 gpurun_out/pytest_gpu.log
cat gpurun_out/knn_variants.log
python - <<'P'
import json
for l in open("gpurun_out/configs.jsonl"):
    try: r=json.loads(l)
    except Exception: print(l.strip()); continue
    print(r["config"], r["dtype"], "knn %.3f alpha %.3f interp %.3f total %.3f ms" % (r["knn_ms"], r["alpha_ms"], r["interp_ms"], r["total_ms"]))
P
