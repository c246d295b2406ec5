#!/bin/bash
# full GPU suite + smoke + default bench at HEAD
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/v_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/v_gputests.log 2>&1; echo "tests_rc=$?" >> gpurun_out/v_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/v_smoke.log
timeout 600 python bench.py > gpurun_out/v_bench.json 2> gpurun_out/v_bench.err; echo "bench_rc=$?" >> gpurun_out/v_bench.err
tail -3 gpurun_out/v_gputests.log; tail -2 gpurun_out/v_smoke.log; cat gpurun_out/v_bench.json | head -c 600
