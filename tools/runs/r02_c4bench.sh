# round 2: configs[4] bench line with the tensor-screen k-means
timeout 3000 python bench.py --workload c4_sbm10m --steps 2 --warmup 3 --no-stability > gpurun_out/r02_bench_c4.json 2> gpurun_out/r02_bench_c4.err; echo "bench rc=$?"
tail -3 gpurun_out/r02_bench_c4.err
