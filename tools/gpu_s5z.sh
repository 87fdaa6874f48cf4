mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/s5z_bench.json 2> gpurun_out/s5z_bench.err; echo "bench rc=$?" >> gpurun_out/s5z_bench.err
timeout 400 python tools/rapid_phases.py --config c5 > gpurun_out/s5z_phases.json 2> gpurun_out/s5z_phases.err
tail -2 gpurun_out/s5z_bench.err
