#!/bin/bash
# Round-2 re-entry check: GPU tests + default bench at HEAD.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/head_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/head_gputest.log 2>&1
echo "pytest exit $?" >> gpurun_out/head_gputest.log
timeout 600 python __graft_entry__.py smoke > gpurun_out/head_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/head_smoke.log
timeout 900 python bench.py > gpurun_out/head_bench.json 2> gpurun_out/head_bench.err
echo "bench exit $?" >> gpurun_out/head_bench.err
tail -3 gpurun_out/head_gputest.log
