RMX_GROUSE_HOSTPROF=1 timeout 400 python tools/rapid_phases.py --config c5 2>&1 | grep "grouse_host" | tail -1
RMX_GROUSE_HOSTPROF=1 RMX_GROUSE_REBASE=4096 timeout 400 python tools/rapid_phases.py --config c5 2>&1 | grep "grouse_host" | tail -1
