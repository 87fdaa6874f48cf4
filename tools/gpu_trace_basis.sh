for v in "RMX_TRACE_BASIS=1" "RMX_TRACE_BASIS=1" "RMX_TRACE_BASIS=1 RMX_PREFETCH_SERIAL=1" "RMX_TRACE_BASIS=1 RMX_PREFETCH_SERIAL=1"; do
  echo "== $v"; env $v timeout 600 python tools/diag_rapid.py --config c5 2>&1 | grep -E "basis-init|mark\] (x_up|basis_n|train_o|grouse)|run_rapid" | cut -c1-100
done
timeout 600 python -m pytest tests/test_gpu_rapid.py tests/test_gpu_configs.py -q -x 2>&1 | tail -2
