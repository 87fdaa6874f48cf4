for i in 1 2 3; do
echo "== run $i"
RMX_GROUSE_HOSTPROF=1 RMX_RAPID_HOSTMARKS=1 timeout 400 python tools/bench_rapid.py --config c5 2>&1 | grep "host-mark\|grouse_host\|train_s" | cut -c1-110 | tail -17
done
