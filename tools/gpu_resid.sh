timeout 600 python -m pytest tests/test_gpu_rapid.py -q -x -k "lsq or recovery or rapid" 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --kernel-name-base demangled -k "regex:k_lsq_resid" -c 2 --csv python tools/bench_rapid.py --config c5 --passes 1 --perms 2100 2>/dev/null | grep -E "k_lsq_resid" | cut -c1-60,150-400 | head -6
timeout 600 python tools/diag_rapid.py --config c5 2>&1 | grep -E "mark\] (grouse|recover)|run_rapid" | cut -c1-100
