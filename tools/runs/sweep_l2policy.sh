L=paper_1509_08863_b200
o=gpurun_out/sweep4.txt; : > $o
for lib in libsc_b200 libsc_b200_el libsc_b200_en; do
  SC_B200_LIB=$PWD/$L/$lib.so python tools/sweep_filter.py --workload c3_sbm1m --chunks 16,24,32 --reps 3 --tag $lib >> $o 2>&1
done
for mb in 48 64 96; do
  SC_PERSIST_MB=$mb python tools/sweep_filter.py --workload c3_sbm1m --chunks 16,24,32 --reps 3 --tag persist$mb >> $o 2>&1
done
SC_PERSIST_MB=64 SC_B200_LIB=$PWD/$L/libsc_b200_el.so python tools/sweep_filter.py --workload c3_sbm1m --chunks 16,24 --reps 3 --tag persist64_el >> $o 2>&1
