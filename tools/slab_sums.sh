# GPU-busy time (sum of ncu kernel durations, generator excluded) of the
# single call and of the 8-slab loopback, C5 and C2
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in C5 C2; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s1.csv python tools/one_case.py $c > /dev/null 2>&1
  python tools/kernel_sums.py gpurun_out/s1.csv 1 | sed "s/^/$c single /" >> gpurun_out/kernel_sums.txt
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s8.csv python tools/slabs_one.py $c 8 > /dev/null 2>&1
  python tools/kernel_sums.py gpurun_out/s8.csv 8 | sed "s/^/$c slabs8 /" >> gpurun_out/kernel_sums.txt
  rm -f gpurun_out/s1.csv gpurun_out/s8.csv
done
cat gpurun_out/kernel_sums.txt
