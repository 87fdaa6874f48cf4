mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rapid.py tests/test_gpu_stream_io.py -q -o faulthandler_timeout=300 > gpurun_out/r02_rapidtests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_rapidtests.log
tail -n 25 gpurun_out/r02_rapidtests.log
timeout 600 python tools/diag_rapid.py --config c5 > gpurun_out/r02_rapid_c5_full.log 2>&1
grep -v "^  File\|^    " gpurun_out/r02_rapid_c5_full.log | tail -16
# recovery launch list (c5: 1 pass, 20,400 perms) and per-kernel ncu of the GROUSE products / new chol
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_rapid_launches.csv \
  python tools/bench_rapid.py --config c5 --passes 1 --perms 20400 > gpurun_out/r02_rapid_launches.log 2>&1
python tools/launch_table.py gpurun_out/r02_rapid_launches.csv > gpurun_out/r02_rapid_launches_summary.txt 2>&1
head -30 gpurun_out/r02_rapid_launches_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_dgemm_rm|k_chol_cluster|k_trsv_warp|k_cg_solve" -s 200 -c 6 \
  -o gpurun_out/r02_grouse_kernels python tools/bench_rapid.py --config c5 --passes 1 --perms 2400 > gpurun_out/r02_grouse_kernels_ncu.log 2>&1
tail -3 gpurun_out/r02_grouse_kernels_ncu.log
