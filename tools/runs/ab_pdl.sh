# programmatic dependent launch of the step kernels (SC_PDL=1 default) against SC_PDL=0
python -m pytest tests/test_gpu_parity.py -q -x -k "filter or p2p or grid or moments or lambda or full_size or cluster or stability or dist" 2>&1 | tail -n 1
for i in 1 2 3; do
  for v in 1 0; do
    echo "pdl=$v $(SC_PDL=$v python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 3 | python -c 'import sys,json; print([json.loads(l)["ms_per_pass"] for l in sys.stdin if l.startswith("{")])')"
  done
done
for v in 1 0; do echo "pdl=$v c2 $(SC_PDL=$v SC_RESIDENT=0 python tools/sweep_filter.py --workload c2_sbm100k --chunks 48 --reps 5 | python -c 'import sys,json; print([json.loads(l)["ms_per_pass"] for l in sys.stdin if l.startswith("{")])')"; done
