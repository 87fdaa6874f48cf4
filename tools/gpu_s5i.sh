mkdir -p gpurun_out
RMX_BENCH_RAPID_MARKS=1 timeout 900 python bench.py > gpurun_out/s5i_bench.json 2> gpurun_out/s5i_bench.err
timeout 400 python tools/bench_rapid.py --config c5 > gpurun_out/s5i_br.log 2>&1
tail -5 gpurun_out/s5i_br.log
