cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_multirank_gpu.py -x -q -s > gpurun_out/mr.log 2>&1
echo "mr rc=$?" >> gpurun_out/mr.log
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py small at xchg > gpurun_out/san_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/san_$tool.log
done
