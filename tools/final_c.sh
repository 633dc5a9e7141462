# round-end evidence (part C, after the last sharded changes): all GPU tests, bench,
# loopback scaling table, GPU-busy per-rank sums
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; head -c 300 gpurun_out/bench.json; echo
timeout 900 python tools/slabs_time.py C5 1 2 4 8 > gpurun_out/slabs_table.txt 2>&1
timeout 600 python tools/slabs_time.py C2 1 2 4 8 >> gpurun_out/slabs_table.txt 2>&1
timeout 900 python tools/slabs_time.py C3 1 8 >> gpurun_out/slabs_table.txt 2>&1
cat gpurun_out/slabs_table.txt
rm -f gpurun_out/kernel_sums.txt
for c in C5 C2; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s1.csv python tools/one_case.py $c > /dev/null 2>&1
  python tools/kernel_sums.py gpurun_out/s1.csv 1 | sed "s/^/$c single /" >> gpurun_out/kernel_sums.txt
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s8.csv python tools/slabs_one.py $c 8 > /dev/null 2>&1
  python tools/kernel_sums.py gpurun_out/s8.csv 8 | sed "s/^/$c slabs8 /" >> gpurun_out/kernel_sums.txt
  python tools/launches.py gpurun_out/s8.csv 40 > gpurun_out/launches_slabs8_$c.txt
  rm -f gpurun_out/s1.csv gpurun_out/s8.csv
done
cat gpurun_out/kernel_sums.txt
