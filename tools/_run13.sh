cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --no-cpu-baseline --no-multi-gmi --comm peer --steps 20 > gpurun_out/r13_bench_peer.json 2> gpurun_out/r13_bench_peer.err
for c in hm_8192env_4gmi at_4096env_decoupled at_4096env_3x256; do
  timeout 600 ncu --profile-from-start off --clock-control none --csv --metrics gpu__time_duration.sum,sm__cycles_active.sum,sm__cycles_elapsed.avg.per_second --log-file gpurun_out/r13_util_$c.csv python tools/sm_util.py probe configs/$c.cfg 2 /tmp/x.json > /dev/null 2>&1
  timeout 300 python tools/sm_util.py probe configs/$c.cfg 2 gpurun_out/r13_util_probe_$c.json > /dev/null 2>&1
  python tools/sm_util.py report gpurun_out/r13_util_$c.csv gpurun_out/r13_util_probe_$c.json > gpurun_out/r13_util_$c.json 2>&1
done
