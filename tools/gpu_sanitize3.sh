python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sanitizer
for tool in memcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 7 python tools/sanitize.py > gpurun_out/sanitizer/r01_${tool}_v13.log 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/sanitizer/r01_${tool}_v13.log
done
