#!/bin/bash
# conditional second refinement step: rapid tests, second-step counts, bench
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rapid.py tests/test_gpu_configs.py -x -q -p no:cacheprovider > gpurun_out/refine_tests.log 2>&1; echo "rc=$?" >> gpurun_out/refine_tests.log
tail -3 gpurun_out/refine_tests.log
RMX_LSQ_STATS=1 timeout 600 python tools/bench_rapid.py --config c5 --passes 1 --perms 6000 > gpurun_out/refine_stats.log 2>&1
grep -c "second refinement" gpurun_out/refine_stats.log; grep "second refinement" gpurun_out/refine_stats.log | head -5
timeout 900 python bench.py > gpurun_out/refine_bench.json 2> gpurun_out/refine_bench.err; echo "bench rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/refine_bench.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['frac'],d['roofline'].get('int8_measured'),d['clocks'],d['rapid'])"
