for v in "RMX_RAPID_SYNC_BEFORE_GROUSE=1" "RMX_NOOP=1"; do
echo "== $v"
env $v RMX_GROUSE_HOSTPROF=1 timeout 400 python tools/bench_rapid.py --config c5 2>&1 | grep "grouse_host\|train_s" | cut -c1-110 | tail -2
done
nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader -lms 100 > gpurun_out/s5t_smi.txt 2>&1 &
SMI=$!
RMX_GROUSE_HOSTPROF=1 timeout 400 python tools/bench_rapid.py --config c5 2>&1 | grep "grouse_host" | tail -1
kill $SMI
awk -F, '{print $1}' gpurun_out/s5t_smi.txt | sort | uniq -c | sort -rn | head -6
