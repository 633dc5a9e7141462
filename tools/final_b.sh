# round-end evidence (part B): GPU-busy per-rank sums of the 8-slab loopback, then tools/prof_round2.sh
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
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
bash tools/prof_round2.sh > gpurun_out/prof.log 2>&1
ls gpurun_out/prof
