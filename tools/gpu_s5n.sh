RMX_CG_STATS=1 timeout 400 python tools/rapid_phases.py --config c5 2>&1 | grep "rmx cg" | tail -2
RMX_CG_STATS=1 RMX_GROUSE_LOOKAHEAD=0 timeout 400 python tools/rapid_phases.py --config c5 2>&1 | grep "rmx cg" | tail -2
