mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rapid.py -q -x -o faulthandler_timeout=300 > gpurun_out/r02_rapidtests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_rapidtests.log
tail -n 3 gpurun_out/r02_rapidtests.log
for v in "RMX_PREFETCH_SERIAL=1" "RMX_PDL=1" "RMX_PDL=1"; do
  echo "== $v"; env $v timeout 600 python tools/diag_rapid.py --config c5 2>&1 | grep -E "mark\]|run_rapid" | cut -c1-110
done
