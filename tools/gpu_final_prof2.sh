# Round-2 final profile set (look-ahead GROUSE, K1 at HEAD).  Reports are
# summarised to text on the box and deleted; summaries are copied into profiles/.
mkdir -p gpurun_out/r02f
O=gpurun_out/r02f
summ() {
  python tools/ncu_report.py $O/$1.ncu-rep 14 > $O/$1_ncu.txt 2>&1
  rm -f $O/$1.ncu-rep
}
# 0. plain runs first (each ncu pass only after the same command exited 0 without ncu)
timeout 600 python tools/profile_naive.py --config c4 --repeat 1 > $O/plain_naive.log 2>&1; echo "naive rc=$?" >> $O/plain_naive.log
timeout 600 python tools/bench_rapid.py --config c5 --passes 1 --perms 500 > $O/plain_rapid.log 2>&1; echo "rapid rc=$?" >> $O/plain_rapid.log
# 1. NaivePT launch list (config 4, 2 full passes)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv \
  python tools/profile_naive.py --config c4 --repeat 2 > $O/launches_c4.log 2>&1
python tools/launch_table.py $O/launches_c4.csv > $O/launches_c4_summary.txt 2>&1
gzip -f $O/launches_c4.csv
# 2. K1 full capture (L = 37,888)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tfill_tc -c 1 \
  -o $O/k1_c4 python tools/profile_naive.py --config c4 --repeat 1 --perms 37888 > $O/k1_c4.log 2>&1
summ k1_c4
# 3. GROUSE kernels (serialised by ncu) and launch list (one pass = 400 updates)
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_dgemm_rm|k_cg_solve|k_gather_urows_vals|k_late|k_resid_defer_vec|k_h_g_part|k_sparse_terms_rows" -s 400 -c 8 \
  -o $O/grouse_c5 python tools/bench_rapid.py --config c5 --passes 1 --perms 500 > $O/grouse_c5.log 2>&1
summ grouse_c5
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/grouse_launches.csv \
  python tools/bench_rapid.py --config c5 --passes 1 --perms 500 > $O/grouse_launches.log 2>&1
python tools/launch_table.py $O/grouse_launches.csv > $O/grouse_launches_summary.txt 2>&1
gzip -f $O/grouse_launches.csv
# 4. in-stream phases: serial chain and the look-ahead main stream
RMX_GROUSE_PROFILE=1 timeout 600 python tools/rapid_phases.py --config c5 > $O/phases_serial.json 2> $O/phases_serial.err
RMX_GROUSE_PROFILE=2 timeout 600 python tools/rapid_phases.py --config c5 > $O/phases_la.json 2> $O/phases_la.err
RMX_CG_STATS=1 timeout 600 python tools/rapid_phases.py --config c5 > $O/phases_cg.json 2> $O/phases_cg.err
# 5. config-level parity numbers
RMX_PARITY_OUT=$O/parity_configs.json timeout 900 python -m pytest tests/test_gpu_configs.py -q -p no:cacheprovider > $O/parity_configs.log 2>&1
# 6. default bench + reference arm
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench rc=$?" >> $O/bench_c4.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?" >> $O/bench_ref.err
du -sh $O; ls $O; tail -n 2 $O/*.log $O/*.err | tail -40
