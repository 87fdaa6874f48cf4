mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rapid.py -x -q -p no:cacheprovider > gpurun_out/s5h_test.log 2>&1; echo "rc=$?" >> gpurun_out/s5h_test.log
tail -4 gpurun_out/s5h_test.log
RMX_GROUSE_TRACE=gpurun_out/s5h_trace.txt timeout 400 python tools/rapid_phases.py --config c5 > gpurun_out/s5h.json 2> gpurun_out/s5h.err
timeout 400 python tools/rapid_phases.py --config c5 > gpurun_out/s5h_b.json 2>> gpurun_out/s5h.err
cat gpurun_out/s5h.json gpurun_out/s5h_b.json; tail -3 gpurun_out/s5h.err
