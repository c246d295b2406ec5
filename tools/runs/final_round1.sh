# full GPU test suite, smoke, headline bench (configs[3]) and the configs[4] pipeline line
python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py --workload c4_sbm10m --no-stability --steps 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
tail -n 2 gpurun_out/gputests.log gpurun_out/smoke.log
