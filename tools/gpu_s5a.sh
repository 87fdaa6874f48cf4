# session check: C5 RapidPT phase marks (twice) + GROUSE in-stream phases
mkdir -p gpurun_out
timeout 400 python tools/rapid_phases.py --config c5 > gpurun_out/s5_phases_a.json 2> gpurun_out/s5_phases_a.err
timeout 400 python tools/rapid_phases.py --config c5 > gpurun_out/s5_phases_b.json 2>> gpurun_out/s5_phases_a.err
RMX_GROUSE_PROFILE=1 timeout 400 python tools/rapid_phases.py --config c5 > gpurun_out/s5_phases_prof.json 2> gpurun_out/s5_phases_prof.err
tail -3 gpurun_out/s5_phases_a.err; cat gpurun_out/s5_phases_a.json gpurun_out/s5_phases_b.json; grep grouse_phase gpurun_out/s5_phases_prof.err
