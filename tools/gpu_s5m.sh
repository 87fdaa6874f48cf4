mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,clocks_throttle_reasons.active,temperature.gpu --format=csv,noheader -lms 200 > gpurun_out/s5m_smi.txt 2>&1 &
SMI=$!
for i in 1 2 3; do
date +%s.%N >> gpurun_out/s5m_t.txt
timeout 400 python tools/rapid_phases.py --config c5 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); m=dict(d['train_marks_s']); print('total',round(d['total_s'],3),'grouse',round(m['grouse']-m['basis_upload+qr'],3),'phases',d['phases_s'])"
done
kill $SMI
sort gpurun_out/s5m_smi.txt | uniq -c | sort -rn | head -12
