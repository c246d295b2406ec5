#!/bin/bash
# final verification: GPU suite, smoke, default bench
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/fc_gputests.log 2>&1; echo "tests_rc=$?" >> gpurun_out/fc_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fc_smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/fc_smoke.log
timeout 900 python bench.py > gpurun_out/fc_bench.json 2> gpurun_out/fc_bench.err; echo "bench_rc=$?" >> gpurun_out/fc_bench.err
tail -3 gpurun_out/fc_gputests.log; tail -2 gpurun_out/fc_smoke.log; head -c 300 gpurun_out/fc_bench.json
