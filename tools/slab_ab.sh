# sharded GPU tests + loopback timings (C2, C5) + launch lists of the 8-slab runs
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q > gpurun_out/pytest_sharded.log 2>&1; tail -3 gpurun_out/pytest_sharded.log
timeout 600 python tools/slabs_time.py C2 1 2 4 8 > gpurun_out/slabs_C2.txt 2>&1
timeout 900 python tools/slabs_time.py C5 1 2 4 8 > gpurun_out/slabs_C5.txt 2>&1
for c in C2 C5; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l8.csv python tools/slabs_one.py $c 8 > /dev/null 2>&1
python tools/launches.py gpurun_out/l8.csv 30 > gpurun_out/launches_slabs8_$c.txt
rm -f gpurun_out/l8.csv
done
cat gpurun_out/slabs_C2.txt gpurun_out/slabs_C5.txt
