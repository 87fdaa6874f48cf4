mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rapid.py tests/test_gpu_stream_io.py -q -o faulthandler_timeout=300 > gpurun_out/r02_rapidtests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_rapidtests.log
tail -n 6 gpurun_out/r02_rapidtests.log
for v in "" "RMX_CHOL_CTA=1"; do
  echo "== $v"; env $v timeout 600 python tools/diag_rapid.py --config c5 2>&1 | grep -E "mark\] (grouse|recover)|run_rapid" | cut -c1-200
done
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_chol_cluster|k_trsv_warp|k_chol_solve<256, float>" -c 3 -o gpurun_out/r02_chol_cluster \
  python -m pytest tests/test_gpu_rapid.py -q -k "tensor_core_gram and 20000" > gpurun_out/dbg_chol_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_dgemm_rm|k_cg_solve" -s 200 -c 6 \
  -o gpurun_out/r02_grouse_kernels python tools/bench_rapid.py --config c5 --passes 1 --perms 2400 > gpurun_out/r02_grouse_kernels_ncu.log 2>&1
tail -2 gpurun_out/r02_grouse_kernels_ncu.log
