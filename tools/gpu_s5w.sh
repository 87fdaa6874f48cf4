for rb in 64 1024 4096 20480; do
RMX_GROUSE_HOSTPROF=1 RMX_GROUSE_REBASE=$rb timeout 400 python tools/bench_rapid.py --config c5 2>&1 | grep "grouse_host\|sigma" | python -c "
import sys,json
for l in sys.stdin:
    l=l.strip()
    if 'grouse_host' in l: print('rebase $rb', l[:70])
    else:
        d=json.loads(l); print('   sigma %.16g mu %.16g max_head %s' % (d['sigma'], d['mu'], d['max_head'][1:3]))"
done
