# fp64 gathers in flight per lane (SC_EB_F64 builds): c3 fp64 filter pass and lambda_k (fp64 moments)
L=$PWD/paper_1509_08863_b200
for lib in libsc_b200 libsc_b200_f64e5 libsc_b200_f64e6 libsc_b200; do
  echo "== $lib"
  SC_B200_LIB=$L/$lib.so python tools/sweep_filter.py --workload c3_sbm1m --chunks 16 --dtype f64 --reps 2 2>&1 | cut -c1-120
  SC_B200_LIB=$L/$lib.so python tools/time_cluster.py c3_sbm1m 2>&1 | cut -c1-110
done
