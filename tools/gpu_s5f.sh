mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rapid.py -x -q -p no:cacheprovider > gpurun_out/s5f_test.log 2>&1; echo "rc=$?" >> gpurun_out/s5f_test.log
tail -5 gpurun_out/s5f_test.log
RMX_GROUSE_HOSTPROF=1 RMX_CG_STATS=1 timeout 400 python tools/rapid_phases.py --config c5 > gpurun_out/s5f_la.json 2> gpurun_out/s5f_la.err
RMX_GROUSE_PROFILE=2 timeout 400 python tools/rapid_phases.py --config c5 > gpurun_out/s5f_p2.json 2> gpurun_out/s5f_p2.err
RMX_GROUSE_PROFILE=1 timeout 400 python tools/rapid_phases.py --config c5 > gpurun_out/s5f_p1.json 2> gpurun_out/s5f_p1.err
grep "grouse_host\|rmx cg" gpurun_out/s5f_la.err | tail -3; grep grouse_phase gpurun_out/s5f_p2.err gpurun_out/s5f_p1.err | tail -2; cat gpurun_out/s5f_la.json
