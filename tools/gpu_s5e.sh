mkdir -p gpurun_out
RMX_CG_STATS=1 timeout 400 python tools/rapid_phases.py --config c5 > gpurun_out/s5e_cg.json 2> gpurun_out/s5e_cg.err
RMX_CG_STATS=1 RMX_GROUSE_LOOKAHEAD=0 timeout 400 python tools/rapid_phases.py --config c5 > gpurun_out/s5e_cgs.json 2> gpurun_out/s5e_cgs.err
grep "rmx cg" gpurun_out/s5e_cg.err gpurun_out/s5e_cgs.err
