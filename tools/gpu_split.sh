for v in "RMX_DGEMM_SPLIT_MAX=8" "RMX_DGEMM_SPLIT_MAX=4" "RMX_DGEMM_SPLIT_MAX=2" "RMX_DGEMM_SPLIT_MAX=1"; do
  echo "== $v"; env $v RMX_GROUSE_PROFILE=1 RMX_PDL=0 timeout 600 python tools/diag_rapid.py --config c5 --passes 3 --perms 1300 2>&1 | grep -E "grouse_phase" | cut -c1-250
  env $v timeout 600 python tools/diag_rapid.py --config c5 --passes 10 --perms 4400 2>&1 | grep -E "mark\] (train_o|grouse)" | cut -c1-100
done
