python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for fl in 0 4194304; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2_$fl.csv python tools/one_case.py C2 "" $fl > /dev/null 2>&1
python tools/timeline.py gpurun_out/launches_C2_$fl.csv > gpurun_out/timeline_C2_$fl.txt
done
