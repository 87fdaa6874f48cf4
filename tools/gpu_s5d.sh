mkdir -p gpurun_out
RMX_GROUSE_PROFILE=2 timeout 400 python tools/rapid_phases.py --config c5 > gpurun_out/s5d_la.json 2> gpurun_out/s5d_la.err
RMX_CG_STATS=1 timeout 400 python tools/rapid_phases.py --config c5 > gpurun_out/s5d_cg.json 2> gpurun_out/s5d_cg.err
RMX_CG_STATS=1 RMX_GROUSE_LOOKAHEAD=0 timeout 400 python tools/rapid_phases.py --config c5 > gpurun_out/s5d_cgs.json 2> gpurun_out/s5d_cgs.err
grep grouse_phase gpurun_out/s5d_la.err; grep "rmx cg" gpurun_out/s5d_cg.err gpurun_out/s5d_cgs.err
