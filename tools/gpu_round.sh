# round-end style pass: GPU tests, smoke, default bench (+ GROUSE profile)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -o faulthandler_timeout=300 > gpurun_out/r02_gputest.log 2>&1; echo "gputest rc=$?" >> gpurun_out/r02_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02_smoke.log
timeout 900 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$?" >> gpurun_out/r02_bench.err
[ -n "$PROF_GROUSE" ] && bash tools/gpu_prof_grouse.sh
tail -n 15 gpurun_out/r02_gputest.log; tail -n 2 gpurun_out/r02_smoke.log; tail -n 12 gpurun_out/r02_bench.err; tail -c 2500 gpurun_out/r02_bench.json
