set -x
python -c "import __graft_entry__ as g; g.build()"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv python tools/one_case.py C2 > gpurun_out/launch_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_stencil -c 1 -o gpurun_out/p_stencil python tools/one_case.py C2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_stencil_compact -c 1 -o gpurun_out/p_compact python tools/one_case.py C2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_events -c 2 -o gpurun_out/p_events python tools/one_case.py C2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_stencil_sparse -s 2 -c 1 -o gpurun_out/p_sparse python tools/one_case.py C2 > /dev/null 2>&1
ls -la gpurun_out
