RMX_TRACE_BASIS=1 RMX_RAPID_HOSTMARKS=1 timeout 400 python tools/bench_rapid.py --config c5 2>&1 | grep "basis-init\|host-mark" | tail -30
