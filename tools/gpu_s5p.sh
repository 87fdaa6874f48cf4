mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/s5p_test.log 2>&1; echo "rc=$?" >> gpurun_out/s5p_test.log
tail -4 gpurun_out/s5p_test.log
timeout 900 python bench.py > gpurun_out/s5p_bench.json 2> gpurun_out/s5p_bench.err; echo "bench rc=$?" >> gpurun_out/s5p_bench.err
RMX_GROUSE_TRACE=gpurun_out/s5p_trace.txt timeout 400 python tools/rapid_phases.py --config c5 > gpurun_out/s5p_phases.json 2> gpurun_out/s5p_phases.err
tail -2 gpurun_out/s5p_bench.err; cat gpurun_out/s5p_phases.json | cut -c1-200
