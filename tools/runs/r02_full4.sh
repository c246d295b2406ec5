# round 2: full GPU suite + smoke on the current build
( time timeout 2400 python -m pytest tests -m gpu -x -q --durations=10 ) > gpurun_out/r02_full4.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02_full4.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" >> gpurun_out/r02_full4.txt 2>&1
