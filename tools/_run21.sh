cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r21_bench.json 2> gpurun_out/r21_bench.err
GMI_ADAM_STREAM=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r21_bench_as.json 2> gpurun_out/r21_bench_as.err
