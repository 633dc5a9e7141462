mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s1.csv python tools/one_case.py C5 > /dev/null 2>&1
python tools/launches.py gpurun_out/s1.csv 40 > gpurun_out/launches_C5_single.txt
rm -f gpurun_out/s1.csv
cat gpurun_out/launches_C5_single.txt
