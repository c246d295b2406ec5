# dynamic tile scheduling of the step kernel (SC_DYN_TILES=1 default) against the static schedule
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "filter_f32_parity and streaming" 2>&1 | tail -n 1 || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "filter or p2p or grid or moments or lambda or full_size or cluster or stability or dist" 2>&1 | tail -n 1
for i in 1 2 3; do
  for v in 1 0; do
    echo "dyn=$v $(SC_DYN_TILES=$v timeout 300 python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 3 | python -c 'import sys,json; print([json.loads(l)["ms_per_pass"] for l in sys.stdin if l.startswith("{")])')"
  done
done
for v in 1 0; do echo "dyn=$v f64 $(SC_DYN_TILES=$v timeout 300 python tools/sweep_filter.py --workload c3_sbm1m --chunks 16 --dtype f64 --reps 2 | python -c 'import sys,json; print([json.loads(l)["ms_per_pass"] for l in sys.stdin if l.startswith("{")])')"; done
