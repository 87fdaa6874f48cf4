mkdir -p gpurun_out
timeout 300 python tools/diag_rapid.py --config c5 --passes 1 --perms 2400 --dump-every 60 > gpurun_out/diag_small.log 2>&1; echo "rc=$?" >> gpurun_out/diag_small.log
timeout 900 python tools/diag_rapid.py --config c5 --dump-every 90 > gpurun_out/diag_full.log 2>&1; echo "rc=$?" >> gpurun_out/diag_full.log
tail -5 gpurun_out/diag_small.log; grep -v "^  File\|^    " gpurun_out/diag_full.log | head -40
