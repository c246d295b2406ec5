# fp64 moments kernel (lambda_k): per-tile warp-reduced moment partials, EB 4 / 5 / 6
L=$PWD/paper_1509_08863_b200
for lib in libsc_b200 libsc_b200_mom5 libsc_b200_mom6 libsc_b200; do
  echo "== $lib"; SC_B200_LIB=$L/$lib.so python tools/time_cluster.py c3_sbm1m 2>&1 | cut -c1-100
done
SC_B200_LIB=$L/libsc_b200_mom5.so python -m pytest tests/test_gpu_parity.py -q -k "moments or lambda_k" 2>&1 | tail -n 1
python -m pytest tests/test_gpu_parity.py -q -k "moments or lambda_k or stability or cluster" 2>&1 | tail -n 1
