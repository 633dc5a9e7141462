# round-end evidence: bench line, launch lists (C2, C3), ncu full captures of the top kernels (C2)
set -x
python -c "import __graft_entry__ as g; g.build()"
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv python tools/one_case.py C2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C3.csv python tools/one_case.py C3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_stencil_fast -c 1 -o gpurun_out/p_stencil_fast python tools/one_case.py C2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_events -s 2 -c 2 -o gpurun_out/p_events python tools/one_case.py C2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_stencil_list -c 1 -o gpurun_out/p_stencil_list python tools/one_case.py C2 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:k_count_edit -c 1 -o gpurun_out/p_count_edit python tools/one_case.py C2 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:k_saddle_order -c 1 -o gpurun_out/p_saddle_order python tools/one_case.py C2 > /dev/null 2>&1
python tools/config_sweep.py C1 C2 C3 C4 C5 > gpurun_out/config_sweep.json 2> gpurun_out/config_sweep.err
