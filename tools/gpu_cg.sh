for v in "RMX_CG_STATS=1" "RMX_CG_STATS=1 RMX_CG_SMEM=1"; do
  echo "== $v"; env $v timeout 600 python tools/diag_rapid.py --config c5 --passes 2 --perms 1000 2>&1 | grep -E "rmx cg|run_rapid" | cut -c1-260
done
timeout 900 python -m pytest tests/test_gpu_rapid.py tests/test_gpu_configs.py -q -x 2>&1 | tail -2
timeout 600 python tools/diag_rapid.py --config c5 2>&1 | grep -E "mark\] (train_o|grouse)|run_rapid" | cut -c1-100
