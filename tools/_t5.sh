mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t5_test.log 2>&1; echo "rc=$?" >> gpurun_out/t5_test.log
tail -3 gpurun_out/t5_test.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t5_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/t5_smoke.log; tail -2 gpurun_out/t5_smoke.log | cut -c1-100
timeout 900 python bench.py > gpurun_out/t5_bench.json 2> gpurun_out/t5_bench.err; echo "bench rc=$?" >> gpurun_out/t5_bench.err; tail -1 gpurun_out/t5_bench.err
RMX_GROUSE_TRACE=gpurun_out/t5_trace.txt timeout 400 python tools/rapid_phases.py --config c5 > gpurun_out/t5_phases.json 2> /dev/null
cut -c1-400 gpurun_out/t5_phases.json
