# GPU check (r02q): kNN shape by batch size -- tests, strong shares, bench
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r02q}
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu.py -q -rf -k "h16 or golden and C4 or graph or order or seed or split" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for nq in 512000 256000 128000; do
  timeout 300 python bench.py --nq $nq --no-cpu-baseline --no-e2e --no-f64 > $O/strong_share_$nq.json 2>> $O/bench.err
done
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2>> $O/bench.err
echo done
