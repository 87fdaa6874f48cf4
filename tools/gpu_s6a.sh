mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rapid.py tests/test_gpu_configs.py -x -q -p no:cacheprovider > gpurun_out/s6a_test.log 2>&1; echo "rc=$?" >> gpurun_out/s6a_test.log
tail -4 gpurun_out/s6a_test.log
RMX_CG_STATS=1 RMX_GROUSE_HOSTPROF=1 timeout 400 python tools/rapid_phases.py --config c5 2>&1 | grep "rmx cg\|grouse_host\|total_s" | tail -4 | cut -c1-330
RMX_GROUSE_TRACE=gpurun_out/s6a_trace.txt timeout 400 python tools/rapid_phases.py --config c5 > gpurun_out/s6a_phases.json 2>/dev/null
cut -c1-120 gpurun_out/s6a_phases.json
