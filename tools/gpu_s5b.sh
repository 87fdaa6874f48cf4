# look-ahead GROUSE: correctness (rapid tests + config-level parity) then C5 timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rapid.py -x -q -p no:cacheprovider -k "grouse or reproducible or trained_model" > gpurun_out/s5b_test.log 2>&1; echo "rc=$?" >> gpurun_out/s5b_test.log
tail -5 gpurun_out/s5b_test.log
timeout 400 python tools/rapid_phases.py --config c5 > gpurun_out/s5b_phases.json 2> gpurun_out/s5b_phases.err
RMX_GROUSE_LOOKAHEAD=0 timeout 400 python tools/rapid_phases.py --config c5 > gpurun_out/s5b_phases_serial.json 2>> gpurun_out/s5b_phases.err
tail -3 gpurun_out/s5b_phases.err; cat gpurun_out/s5b_phases.json gpurun_out/s5b_phases_serial.json
