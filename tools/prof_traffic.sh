# ncu --set full captures of the main kernels of a C2 correction -> raw/source CSVs
# (tools/make_traffic.py turns them into profiles/traffic.json)
set -x
mkdir -p gpurun_out/prof
python -c "import __graft_entry__ as g; g.build()"
cap() {  # name, kernel regex, launches to skip
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 \
    -o gpurun_out/prof/$1 python tools/one_case.py ${CFG:-C2} > /dev/null 2>&1
  ncu -i gpurun_out/prof/$1.ncu-rep --page raw --csv > gpurun_out/prof/$1_raw.csv
  ncu -i gpurun_out/prof/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/prof/$1_src.csv
  rm -f gpurun_out/prof/$1.ncu-rep
}
cap stencil 'k_stencil_key2' 0
cap events '^k_events$' 2
cap list 'k_stencil_list' 0
cap edit 'k_count_edit' 0
cap order 'k_saddle_order' 0
ls -la gpurun_out/prof
