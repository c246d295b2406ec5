#!/bin/bash
# round 2 (session 3) verification: whole GPU suite, smoke, default bench; then the launch
# list of the cluster pipeline (sc_cluster on configs[3]) under ncu
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/fa_gputests.log 2>&1; echo "tests_rc=$?" >> gpurun_out/fa_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fa_smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/fa_smoke.log
timeout 900 python bench.py > gpurun_out/fa_bench.json 2> gpurun_out/fa_bench.err; echo "bench_rc=$?" >> gpurun_out/fa_bench.err
tail -2 gpurun_out/fa_gputests.log; tail -2 gpurun_out/fa_smoke.log; head -c 400 gpurun_out/fa_bench.json
python tools/time_cluster.py c3_sbm1m 1 > gpurun_out/fa_cluster_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/fa_cluster_launches.csv python tools/time_cluster.py c3_sbm1m 1 > gpurun_out/fa_cluster_ncu.log 2>&1
echo "ncu_rc=$?"
