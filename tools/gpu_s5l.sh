mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rapid.py tests/test_gpu_configs.py -x -q -p no:cacheprovider > gpurun_out/s5l_test.log 2>&1; echo "rc=$?" >> gpurun_out/s5l_test.log
tail -4 gpurun_out/s5l_test.log
RMX_GROUSE_TRACE=gpurun_out/s5l_trace.txt timeout 400 python tools/rapid_phases.py --config c5 > gpurun_out/s5l.json 2> gpurun_out/s5l.err
RMX_LSQ_STREAMS=1 timeout 400 python tools/rapid_phases.py --config c5 > gpurun_out/s5l_b.json 2>> gpurun_out/s5l.err
cat gpurun_out/s5l.json gpurun_out/s5l_b.json; tail -3 gpurun_out/s5l.err
