# fp32 gathers in flight per lane (SC_EB_F32 builds) on configs[4] (64 + 32 chunks, DRAM-bound
# gathers) and configs[3]
L=$PWD/paper_1509_08863_b200
for lib in libsc_b200 libsc_b200_f32e7 libsc_b200_f32e8 libsc_b200; do
  SC_B200_LIB=$L/$lib.so SC_CHUNK=64 python tools/sweep_filter.py --workload c4_sbm10m --chunks 64 --reps 1 --tag $lib 2>&1 | cut -c1-120
done
for lib in libsc_b200 libsc_b200_f32e7 libsc_b200_f32e8; do
  SC_B200_LIB=$L/$lib.so python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 3 --tag $lib 2>&1 | cut -c1-120
done
