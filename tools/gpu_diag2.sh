mkdir -p gpurun_out
timeout 700 python -c "import faulthandler,sys; faulthandler.dump_traceback_later(120, repeat=True); sys.argv=['bench.py','--steps','3','--warmup','3']; exec(compile(open('bench.py').read(),'bench.py','exec'))" > gpurun_out/diag_bench.log 2>&1; echo "rc=$?" >> gpurun_out/diag_bench.log
timeout 1000 python -m pytest tests/test_gpu_configs.py -x -v -o faulthandler_timeout=200 > gpurun_out/diag_configs.log 2>&1; echo "rc=$?" >> gpurun_out/diag_configs.log
grep -v "^  File\|^    " gpurun_out/diag_bench.log | tail -c 2500; grep -E "PASS|FAIL|rc=|Timeout|Thread|File" gpurun_out/diag_configs.log | head -60
