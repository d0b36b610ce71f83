cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/pipe_peaks.cu -o /tmp/pipe_peaks 2>&1 | tail -2
timeout 600 ncu --metrics sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed --csv /tmp/pipe_peaks > gpurun_out/pipe_ncu.csv 2>&1
python - <<'P'
import csv,io
rows=list(csv.reader(open('gpurun_out/pipe_ncu.csv')))
hi=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hi]; ik=h.index('Kernel Name'); im=h.index('Metric Name'); iv=h.index('Metric Value'); iid=h.index('ID')
for r in rows[hi+1:]:
    if len(r)>iv: print(r[iid], r[ik][:20], r[im], r[iv])
P
