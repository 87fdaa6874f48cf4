for v in "RMX_CHOL_NOLA=1" "RMX_X=1" "RMX_CHOL_NOLA=1" "RMX_X=1"; do
env $v timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum --kernel-name-base demangled -k "regex:k_chol_solve<\(int\)256, float>" -c 1 --csv python tools/bench_rapid.py --config c5 --passes 1 --perms 2100 2>/dev/null | grep -E "k_chol" | awk -F'","' -v v="$v" '{print v, $NF}' | head -2
done
timeout 600 python -m pytest tests/test_gpu_rapid.py -q 2>&1 | tail -2
