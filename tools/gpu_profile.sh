#!/bin/bash
# Standard GPU-box capture (run under gpurun from the repo root): the bench line, the ncu launch
# list of a short bench run (per-launch time + DRAM bytes), and one `ncu --set full` capture of
# the dominant kernel (training-forward GEMM). Outputs land in gpurun_out/<tag>_*.
tag=${1:-cap}
out=gpurun_out
mkdir -p $out
timeout 900 python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $out/${tag}_launches.csv python bench.py --steps 2 --warmup 1 --no-multi-gmi --no-cpu-baseline \
  > $out/${tag}_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:gemm_tcgen05_kernel<\(int\)256, \(int\)0, \(int\)0, \(int\)0, \(int\)1, \(int\)0>' -s 60 -c 2 -o $out/${tag}_fwd_full \
  python bench.py --steps 1 --warmup 1 --no-multi-gmi --no-cpu-baseline > $out/${tag}_ncu2.log 2>&1
echo done
