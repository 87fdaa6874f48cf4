mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rapid.py -q -o faulthandler_timeout=300 > gpurun_out/r02_rapidtests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_rapidtests.log
tail -n 4 gpurun_out/r02_rapidtests.log
for v in "RMX_GROUSE_PROFILE=1" "RMX_CHOL_CLUSTER=1"; do
  echo "== $v"; env $v timeout 600 python tools/diag_rapid.py --config c5 2>&1 | grep -E "mark\] (train_omegas|grouse|recover)|run_rapid|grouse_phase" | cut -c1-300
done
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_dgemm_rm" -s 200 -c 3 \
  -o gpurun_out/r02_grouse_dgemm python tools/bench_rapid.py --config c5 --passes 1 --perms 2400 > gpurun_out/r02_grouse_kernels_ncu.log 2>&1
RMX_CHOL_CLUSTER=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_chol_cluster|k_chol_solve<256, float>" -c 2 -o gpurun_out/r02_chol_cluster \
  python -m pytest tests/test_gpu_rapid.py -q -k "tensor_core_gram and 20000" > gpurun_out/dbg_chol_ncu.log 2>&1
tail -1 gpurun_out/dbg_chol_ncu.log
