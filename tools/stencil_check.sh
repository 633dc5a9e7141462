# stencil iteration: bit-exact tests that cover the dense stencil, C2 timing, one ncu capture of it
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "parity_configs or fast_stencil or tracking_equals or golden or degenerate or misaligned" > gpurun_out/stencil_pytest.log 2>&1; tail -2 gpurun_out/stencil_pytest.log
REPS=3 timeout 300 python tools/quick_time.py C2 > gpurun_out/stencil_qt.log 2>&1
mkdir -p gpurun_out/prof
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stencil_key2 -c 1 -o gpurun_out/prof/stencil python tools/one_case.py C2 > /dev/null 2>&1
ncu -i gpurun_out/prof/stencil.ncu-rep --page raw --csv > gpurun_out/prof/stencil_raw.csv
ncu -i gpurun_out/prof/stencil.ncu-rep --page source --csv --print-source sass > gpurun_out/prof/stencil_src.csv
rm -f gpurun_out/prof/stencil.ncu-rep
python tools/ncu_quick_csv.py gpurun_out/prof/stencil_raw.csv gpurun_out/prof/stencil_src.csv > gpurun_out/stencil_ncu.txt 2>&1
