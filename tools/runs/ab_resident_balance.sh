# resident kernel: CTA ranges balanced by nnz + 2 rows (SC_RESIDENT_BALANCE=1 default) vs equal tile counts
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "filter or stability or cluster or moments" 2>&1 | tail -n 1
for i in 1 2 3; do
  for v in 1 0; do
    echo "bal=$v c2 $(SC_RESIDENT_BALANCE=$v python tools/time_filter.py c2_sbm100k) c1 $(SC_RESIDENT_BALANCE=$v python tools/time_filter.py c1_gmm20k)"
  done
done
