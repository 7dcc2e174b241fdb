cd $GRAFT_REPO_ROOT
timeout 900 ncu --section SourceCounters --section WarpStateStats --section SpeedOfLight --warp-sampling-interval 0 --warp-sampling-max-passes 20 --clock-control none --import-source on --kernel-name-base demangled -k 'regex:gemm_tcgen05_kernel<\(int\)256, \(int\)0, \(int\)0, \(int\)0, \(int\)1, \(int\)0>' -s 61 -c 1 -o gpurun_out/fwd_src python bench.py --steps 1 --warmup 1 --no-multi-gmi --no-cpu-baseline > gpurun_out/ncu8.log 2>&1
echo done
