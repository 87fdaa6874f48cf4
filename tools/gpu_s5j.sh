mkdir -p gpurun_out
for i in 1 2; do
RMX_GROUSE_HOSTPROF=1 RMX_RAPID_SYNC_BEFORE_GROUSE=1 timeout 400 python tools/bench_rapid.py --config c5 2>&1 | grep "grouse_host\|train_s" | tail -2 | cut -c1-130
RMX_GROUSE_HOSTPROF=1 timeout 400 python tools/bench_rapid.py --config c5 2>&1 | grep "grouse_host\|train_s" | tail -2 | cut -c1-130
done
