mkdir -p gpurun_out
RMX_GROUSE_HOSTPROF=1 timeout 400 python tools/rapid_phases.py --config c5 > gpurun_out/s5c_la.json 2> gpurun_out/s5c_la.err
RMX_GROUSE_HOSTPROF=1 RMX_GROUSE_LOOKAHEAD=0 timeout 400 python tools/rapid_phases.py --config c5 > gpurun_out/s5c_ser.json 2> gpurun_out/s5c_ser.err
grep grouse_host gpurun_out/s5c_la.err gpurun_out/s5c_ser.err; cat gpurun_out/s5c_la.json gpurun_out/s5c_ser.json
