python -m pytest tests -m gpu -x -q > gpurun_out/r2ah_pytest.log 2>&1; tail -2 gpurun_out/r2ah_pytest.log
python tools/tick_phases.py --decide-only --ticks 200 2>&1 | tail -1
python bench.py --steps 20 --warmup 5 > gpurun_out/r2ah_bench.json 2> gpurun_out/r2ah_bench.err; echo bench_rc=$?
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
