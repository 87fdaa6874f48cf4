RMX_RAPID_HOSTMARKS=1 timeout 400 python tools/bench_rapid.py --config c5 2>&1 | grep "host-mark\|train_s" | cut -c1-160 | tail -22
