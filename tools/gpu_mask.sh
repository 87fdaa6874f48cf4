#!/bin/bash
# K1 from indicator bit rows: naive GPU tests, c4 bench, int8 peak, K1 traffic capture
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_naive.py tests/test_gpu_golden.py tests/test_gpu_stream_io.py -x -q -p no:cacheprovider > gpurun_out/mask_tests.log 2>&1; echo "rc=$?" >> gpurun_out/mask_tests.log
tail -2 gpurun_out/mask_tests.log
timeout 600 python bench.py --no-rapid > gpurun_out/mask_bench.json 2> gpurun_out/mask_bench.err; echo "bench rc=$?"
timeout 300 python tools/measure_int8_peak.py gpurun_out/int8_peak.json > gpurun_out/int8_peak.log 2>&1; echo "peak rc=$?"
tail -c 600 gpurun_out/int8_peak.log
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_tfill_tc -c 1 --csv \
  --log-file gpurun_out/mask_k1_traffic.csv python tools/profile_naive.py --config c4 --repeat 1 > gpurun_out/mask_k1_traffic.log 2>&1
echo "ncu rc=$?"; grep -E "dram__bytes|gpu__time" gpurun_out/mask_k1_traffic.csv | cut -c1-300
python -c "
import json;d=json.loads(open('gpurun_out/mask_bench.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['frac'],d['roofline']['kernel_ms'],d['clocks'],d['parity'])"
