# Round-2 profile set.  Reports are summarised to text on the box
# (tools/ncu_report.py, tools/launch_table.py) and deleted, so what comes
# back through gpurun_out/ stays small; summaries are copied into profiles/.
mkdir -p gpurun_out/r02
O=gpurun_out/r02
summ() {  # summ NAME: text summary of $O/NAME.ncu-rep, then drop the report
  python tools/ncu_report.py $O/$1.ncu-rep 14 > $O/$1_ncu.txt 2>&1
  rm -f $O/$1.ncu-rep
}
# 1. NaivePT launch list (config 4, 2 full passes)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv \
  python tools/profile_naive.py --config c4 --repeat 2 > $O/launches_c4.log 2>&1
python tools/launch_table.py $O/launches_c4.csv > $O/launches_c4_summary.txt 2>&1
gzip -f $O/launches_c4.csv
# 2. K1 full capture (L = 37,888 as in round 1) and the DRAM bytes of one full-L launch
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tfill_tc -c 1 \
  -o $O/k1_c4 python tools/profile_naive.py --config c4 --repeat 1 --perms 37888 > $O/k1_c4.log 2>&1
summ k1_c4
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_tfill_tc -c 1 --csv \
  --log-file $O/k1_traffic_c4.csv python tools/profile_naive.py --config c4 --repeat 1 > $O/k1_traffic.log 2>&1
# 3. recovery kernels (config 5 shapes, one full batch of 1,667 systems)
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_chol_solve<\(int\)256, float>|k_trsv_warp|k_lsq_resid|k_gram_tc|k_rapid_stats_warp|k_complete" -c 7 \
  -o $O/recovery_c5 python tools/bench_rapid.py --config c5 --passes 1 --perms 2100 > $O/recovery_c5.log 2>&1
summ recovery_c5
# 4. GROUSE kernels and launch list (one pass = 400 updates)
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_dgemm_rm|k_cg_solve|k_gather_urows_vals|k_resid_defer_vec" -s 300 -c 6 \
  -o $O/grouse_c5 python tools/bench_rapid.py --config c5 --passes 1 --perms 500 > $O/grouse_c5.log 2>&1
summ grouse_c5
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/grouse_launches.csv \
  python tools/bench_rapid.py --config c5 --passes 1 --perms 500 > $O/grouse_launches.log 2>&1
python tools/launch_table.py $O/grouse_launches.csv > $O/grouse_launches_summary.txt 2>&1
gzip -f $O/grouse_launches.csv
RMX_GROUSE_PROFILE=1 RMX_PDL=0 timeout 600 python tools/diag_rapid.py --config c5 > $O/grouse_phases.log 2>&1
# 5. config-level parity numbers (tests/test_gpu_configs.py -> JSON)
RMX_PARITY_OUT=$O/parity_configs.json timeout 900 python -m pytest tests/test_gpu_configs.py -q > $O/parity_configs.log 2>&1
du -sh $O; ls $O; tail -n 2 $O/*.log | tail -30
