set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python tools/slabs_time.py C5 1 8 > gpurun_out/slabs_C5.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_slabs8_C2.csv python tools/slabs_one.py C2 8 > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_slabs8_C2.csv 40 > gpurun_out/launches_slabs8_C2.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_slabs1_C2.csv python tools/slabs_one.py C2 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_slabs1_C2.csv 40 > gpurun_out/launches_slabs1_C2.txt
rm -f gpurun_out/*.csv
