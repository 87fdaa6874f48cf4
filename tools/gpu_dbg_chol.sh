mkdir -p gpurun_out
for combo in "RMX_CHOL_CTA=1 RMX_TRSV_CTA=1" "RMX_CHOL_CTA=1" "RMX_TRSV_CTA=1" ""; do
  echo "== $combo" >> gpurun_out/dbg_chol.log
  env $combo timeout 300 python -m pytest tests/test_gpu_rapid.py -q -k tensor_core_gram 2>&1 | grep -E "passed|failed|AssertionError: \(" >> gpurun_out/dbg_chol.log
done
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_chol_cluster|k_trsv_warp" -c 2 -o gpurun_out/r02_chol_cluster \
  python -m pytest tests/test_gpu_rapid.py -q -k "tensor_core_gram and 20000" > gpurun_out/dbg_chol_ncu.log 2>&1
cat gpurun_out/dbg_chol.log; tail -2 gpurun_out/dbg_chol_ncu.log
RMX_CHOL_CTA=1 timeout 600 python tools/diag_rapid.py --config c5 > gpurun_out/r02_rapid_c5_full.log 2>&1
grep -v "^  File\|^    " gpurun_out/r02_rapid_c5_full.log | tail -16
RMX_CHOL_CTA=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_dgemm_rm|k_cg_solve" -s 200 -c 6 \
  -o gpurun_out/r02_grouse_kernels python tools/bench_rapid.py --config c5 --passes 1 --perms 2400 > gpurun_out/r02_grouse_kernels_ncu.log 2>&1
tail -2 gpurun_out/r02_grouse_kernels_ncu.log
