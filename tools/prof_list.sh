python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/prof
for v in key:0 float:4194304; do n=${v%%:*}; fl=${v##*:};
timeout 900 ncu --set full --clock-control none -k regex:k_stencil_list -s 1 -c 1 -o gpurun_out/prof/list_$n python tools/one_case.py C2 "" $fl > /dev/null 2>&1
ncu -i gpurun_out/prof/list_$n.ncu-rep --page raw --csv > gpurun_out/prof/list_${n}_raw.csv
ncu -i gpurun_out/prof/list_$n.ncu-rep --page details --csv > gpurun_out/prof/list_${n}_details.csv
rm -f gpurun_out/prof/list_$n.ncu-rep
done
