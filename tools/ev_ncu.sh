# sharded tests, C5 8-slab timing, ncu --set full of the C3 walk launches: slab (C5 / 8) vs single (C5)
mkdir -p gpurun_out/prof
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q > gpurun_out/pytest_sharded.log 2>&1; tail -2 gpurun_out/pytest_sharded.log
timeout 600 python tools/slabs_time.py C5 8 > gpurun_out/slabs_ev.txt 2>&1
cat gpurun_out/slabs_ev.txt
cap() {
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^k_events$' -s $3 -c 2 \
    -o gpurun_out/prof/$1 python $2 > /dev/null 2>&1
  ncu -i gpurun_out/prof/$1.ncu-rep --page raw --csv > gpurun_out/prof/$1_raw.csv
  rm -f gpurun_out/prof/$1.ncu-rep
}
cap ev_slab "tools/slabs_one.py C5 8" 16
cap ev_single "tools/one_case.py C5" 0
python tools/ncu_quick_csv.py gpurun_out/prof/ev_slab_raw.csv > gpurun_out/prof/ev_slab.txt 2>&1
python tools/ncu_quick_csv.py gpurun_out/prof/ev_single_raw.csv > gpurun_out/prof/ev_single.txt 2>&1
head -40 gpurun_out/prof/ev_slab.txt gpurun_out/prof/ev_single.txt
