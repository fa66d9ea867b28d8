set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r2aa_pytest.log 2>&1; tail -2 gpurun_out/r2aa_pytest.log
python tools/tick_phases.py > gpurun_out/r2aa_phases.jsonl 2>&1; cat gpurun_out/r2aa_phases.jsonl
python tools/cold_split.py > gpurun_out/r2aa_cold_split.jsonl 2>&1; cat gpurun_out/r2aa_cold_split.jsonl
TA_NO_EVENTS=1 python tools/step_times.py --phases --mini --flush --ticks 80 > gpurun_out/r2aa_stamps.txt 2>&1; tail -12 gpurun_out/r2aa_stamps.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tick_front|k_pause_restore|k_plan|k_close" -s 300 -c 4 -o gpurun_out/r2aa_sched python tools/step_times.py --mini --no-timing --flush --ticks 80 > gpurun_out/r2aa_ncu.log 2>&1; tail -3 gpurun_out/r2aa_ncu.log
ncu -i gpurun_out/r2aa_sched.ncu-rep --page raw --csv > gpurun_out/r2aa_sched_raw.csv 2>/dev/null; wc -l gpurun_out/r2aa_sched_raw.csv
