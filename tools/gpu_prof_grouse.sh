# GROUSE per-update launch list (config 5, one pass = 400 updates) + full C5 timing
mkdir -p gpurun_out
timeout 300 python tools/diag_rapid.py --config c5 --passes 1 --perms 500 > gpurun_out/r02_grouse_p1.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_grouse_launches.csv \
  python tools/diag_rapid.py --config c5 --passes 1 --perms 500 > gpurun_out/r02_grouse_launches.log 2>&1
python tools/launch_table.py gpurun_out/r02_grouse_launches.csv > gpurun_out/r02_grouse_launches_summary.txt 2>&1
timeout 600 python tools/diag_rapid.py --config c5 > gpurun_out/r02_rapid_c5_full.log 2>&1
head -40 gpurun_out/r02_grouse_launches_summary.txt; grep -v "^  File\|^    " gpurun_out/r02_rapid_c5_full.log | tail -20
