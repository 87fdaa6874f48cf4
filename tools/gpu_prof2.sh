# round-2 profiling pass: f3 tests, recovery / GROUSE launch lists, chol ncu
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stream_io.py -x -q > gpurun_out/r02_streamio.log 2>&1; echo "rc=$?" >> gpurun_out/r02_streamio.log
for nt in 256 512; do
  RMX_CHOL_NT=$nt timeout 600 python tools/bench_rapid.py --config c5 --passes 1 --perms 20400 > gpurun_out/r02_rapid_c5_p1_nt$nt.json 2> gpurun_out/r02_rapid_c5_p1_nt$nt.err
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_rapid_launches.csv \
  python tools/bench_rapid.py --config c5 --passes 1 --perms 20400 > gpurun_out/r02_rapid_launches.log 2>&1
python tools/launch_table.py gpurun_out/r02_rapid_launches.csv > gpurun_out/r02_rapid_launches_summary.txt 2>&1
for nt in 256 512; do
  RMX_CHOL_NT=$nt timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_chol_solve<(256|512), float>" -c 4 \
    -o gpurun_out/r02_chol_f32_nt$nt python tools/bench_rapid.py --config c5 --passes 1 --perms 2000 > gpurun_out/r02_chol_ncu_nt$nt.log 2>&1
done
tail -3 gpurun_out/r02_streamio.log; cat gpurun_out/r02_rapid_c5_p1_nt*.json; head -30 gpurun_out/r02_rapid_launches_summary.txt
