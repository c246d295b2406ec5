# round 2: stability regression test, then the bench line (configs[3])
python -m pytest tests -q -m gpu -x -k "stability" 2>&1 | tail -2
python tools/stab_probe.py
python bench.py > gpurun_out/r02_bench_c3.json 2> gpurun_out/r02_bench_c3.err; echo "bench rc=$?"
