RMX_GROUSE_PROFILE=1 RMX_PDL=0 timeout 600 python tools/diag_rapid.py --config c5 2>&1 | grep -E "grouse_phase|run_rapid" | cut -c1-250
for i in 1 2; do timeout 600 python tools/diag_rapid.py --config c5 2>&1 | grep -E "mark\] (train_o|grouse|recover)|run_rapid" | cut -c1-100; done
