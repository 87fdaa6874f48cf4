#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rapid.py tests/test_gpu_configs.py -x -q -p no:cacheprovider > gpurun_out/refine2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/refine2_tests.log
tail -3 gpurun_out/refine2_tests.log
RMX_LSQ_STATS=1 timeout 600 python tools/bench_rapid.py --config c5 --passes 1 --perms 6000 > gpurun_out/refine2_stats.log 2>&1
grep "second refinement" gpurun_out/refine2_stats.log | head -5
for i in 1 2; do timeout 600 python tools/rapid_phases.py --config c5 > gpurun_out/phases_c5_$i.json 2> gpurun_out/phases_c5_$i.err; tail -c 1500 gpurun_out/phases_c5_$i.json; done
nproc; cat /proc/cpuinfo | grep "model name" | head -1
