mkdir -p gpurun_out
RMX_GROUSE_TRACE=gpurun_out/s5g_trace.txt timeout 400 python tools/rapid_phases.py --config c5 > gpurun_out/s5g.json 2> gpurun_out/s5g.err
cat gpurun_out/s5g.json; wc -l gpurun_out/s5g_trace.txt
