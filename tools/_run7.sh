cd $GRAFT_REPO_ROOT
timeout -s KILL 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/gpu_all7.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_all7.log
timeout -s KILL 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke7.log 2>&1; echo "rc=$?" >> gpurun_out/smoke7.log
