# C3 (combustion 560^3) diagnosis: timeline launch list, per-pass stats, one ncu capture of R4 and events
set -x
python -c "import __graft_entry__ as g; g.build()"
python tools/walkstats.py C3 > gpurun_out/c3_walkstats.log 2>&1
REPS=2 python tools/quick_time.py C3 > gpurun_out/c3_time.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C3.csv python tools/one_case.py C3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_saddle_order -s 3 -c 1 -o gpurun_out/p_c3_order python tools/one_case.py C3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_events -s 4 -c 2 -o gpurun_out/p_c3_events python tools/one_case.py C3 > /dev/null 2>&1
