# ncu full capture of the fp64 weighting kernel at C4 sizes (one launch)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cat > /tmp/f64run.py <<'P'
import sys; sys.path.insert(0, ".")
import torch, datagen, paper_1511_02186_b200 as P
x, y, z = datagen.make_data("C4"); qx, qy = datagen.make_queries("C4", nq=256000)
eng = P.AIDW(x, y, z, dtype=torch.float64)
Z = eng.run(qx, qy, 10, datagen.ALPHA_LEVELS, P.GLOBAL); torch.cuda.synchronize(); print("ok")
P
timeout 900 ncu --set full --clock-control none --import-source on -k regex:interp_kernel -c 1 \
    -o gpurun_out/f64interp python /tmp/f64run.py > gpurun_out/f64interp.log 2>&1
python tools/ncu_summary.py gpurun_out/f64interp.ncu-rep --json gpurun_out/f64interp.json > /dev/null 2>&1
ncu -i gpurun_out/f64interp.ncu-rep --page source --csv --print-source sass > gpurun_out/f64interp_sass.csv 2>/dev/null
ncu -i gpurun_out/f64interp.ncu-rep --page raw --csv > gpurun_out/f64interp_raw.csv 2>/dev/null
tail -3 gpurun_out/f64interp.log
