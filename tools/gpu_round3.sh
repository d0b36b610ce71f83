# evidence refresh: round2 set + fp64 bench line + pipe peaks (DFMA)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-v12}
bash tools/gpu_round2.sh ${TAG}
timeout 900 python bench.py --dtype f64 --steps 3 --warmup 3 > gpurun_out/bench_f64_${TAG}.json 2> gpurun_out/bench_f64.err
cut -c1-300 gpurun_out/bench_f64_${TAG}.json
nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/pipe_peaks.cu -o /tmp/pipe_peaks && /tmp/pipe_peaks > gpurun_out/pipe_peaks_${TAG}.jsonl
cat gpurun_out/pipe_peaks_${TAG}.jsonl
