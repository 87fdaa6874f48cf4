mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_rapid.py -x -q -p no:cacheprovider -k "grouse_matches_oracle_numpy_restatement and cg and lookahead or halt_redraw_at_checkpoints and 63,71,95 and lookahead" > gpurun_out/s5x_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/s5x_memcheck.log
tail -12 gpurun_out/s5x_memcheck.log
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_rapid.py -x -q -p no:cacheprovider -k "grouse_matches_oracle_numpy_restatement and cg and lookahead" > gpurun_out/s5x_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/s5x_racecheck.log
tail -8 gpurun_out/s5x_racecheck.log
