for i in 1 2 3; do
timeout 400 python tools/rapid_phases.py --config c5 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); m=dict(d['train_marks_s']); print('total',round(d['total_s'],3),'train',round(d['train_s'],3),'grouse',round(m['grouse']-m['basis_upload+qr'],3),'pre',round(m['basis_upload+qr'],3),'phases',d['phases_s'])"
timeout 400 python tools/bench_rapid.py --config c5 2>&1 | tail -1 | cut -c1-120
done
