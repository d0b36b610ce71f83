# GPU check (r02l): fused exp2 range reduction -- tests + offload sweep
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r02l}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rf -k "not C5" > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
for v in 0 36 38 26 37; do AIDW_INTERP_VARIANT=$v timeout 120 python tools/tune_interp.py 1024000 --check >> $O/tune_interp.log 2>&1; done
echo done
