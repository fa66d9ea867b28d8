python -m pytest tests -m gpu -x -q > gpurun_out/r2af_pytest.log 2>&1; tail -2 gpurun_out/r2af_pytest.log
python tools/tick_phases.py --decide-only --ticks 200 > gpurun_out/r2af_phases.jsonl 2>&1; cat gpurun_out/r2af_phases.jsonl
python bench.py --steps 20 --warmup 5 > gpurun_out/r2af_bench.json 2> gpurun_out/r2af_bench.err; echo bench_rc=$?
