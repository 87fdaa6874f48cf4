set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest.log 2>&1; echo "gputest rc=$?" >> gpurun_out/r02_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02_smoke.log
timeout 900 python bench.py > gpurun_out/r02_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r02_bench.log
tail -3 gpurun_out/r02_gputest.log gpurun_out/r02_smoke.log; tail -c 3000 gpurun_out/r02_bench.log
