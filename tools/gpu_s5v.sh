for v in "RMX_NOOP=1" "RMX_POOL_TRIM=1" "RMX_NOOP=1"; do
env $v timeout 600 python bench.py --steps 5 --warmup 3 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', 'ms',round(d['ms_per_step'],2),'e2e_ms',round(1e3*d['e2e']['s_per_step'],2),'first',round(d['e2e']['first_call_s'],3),'rapid',round(d['rapid']['max_null_s'],2))"
done
