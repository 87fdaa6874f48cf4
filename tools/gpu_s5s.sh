mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/s5s_test.log 2>&1; echo "rc=$?" >> gpurun_out/s5s_test.log
tail -3 gpurun_out/s5s_test.log
RMX_TRACE_BASIS=1 timeout 400 python tools/rapid_phases.py --config c5 2>&1 | grep "basis-init\|total_s" | tail -4 | cut -c1-600
timeout 400 python tools/bench_rapid.py --config c5 2>&1 | tail -1 | cut -c1-120
timeout 400 python tools/bench_rapid.py --config c5 2>&1 | tail -1 | cut -c1-120
