mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rapid.py -x -q -p no:cacheprovider -k "lookahead_matches_serial or grouse" > gpurun_out/s5y_test.log 2>&1; echo "rc=$?" >> gpurun_out/s5y_test.log
tail -15 gpurun_out/s5y_test.log
