# CSR ring depth of the step kernel (SC_NSTAGES builds), configs[3], alternating
L=$PWD/paper_1509_08863_b200
for i in 1 2; do
  for lib in libsc_b200 libsc_b200_ns4; do
    SC_B200_LIB=$L/$lib.so python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 3 --tag $lib 2>&1 | python -c "import sys,json; [print(json.loads(l)[\"tag\"], json.loads(l)[\"ms_per_pass\"]) for l in sys.stdin if l.startswith(\"{\")]"
  done
done
