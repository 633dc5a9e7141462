# round-end evidence: the bench line, the ncu launch list of a short bench run, ncu --set full
# of the main kernels (-> profiles/traffic.json via tools/make_traffic.py)
set -x
mkdir -p gpurun_out/prof
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 1 --no-ocr --no-reformulated --no-cpu-baseline > gpurun_out/bench_under_ncu.json 2>&1
python tools/launches.py gpurun_out/launches_bench.csv 40 > gpurun_out/launches_bench.txt
cap() {  # name, kernel regex, launches to skip
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 \
    -o gpurun_out/prof/$1 python tools/one_case.py ${CFG:-C2} > /dev/null 2>&1
  ncu -i gpurun_out/prof/$1.ncu-rep --page raw --csv > gpurun_out/prof/$1_raw.csv
  ncu -i gpurun_out/prof/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/prof/$1_src.csv
  rm -f gpurun_out/prof/$1.ncu-rep
  python tools/ncu_quick_csv.py gpurun_out/prof/$1_raw.csv gpurun_out/prof/$1_src.csv > gpurun_out/prof/$1_summary.txt 2>&1
}
cap stencil 'k_stencil_key2' 0
cap events '^k_events$' 2
cap list 'k_stencil_list' 0
cap edit 'k_count_edit' 0
cap order 'k_saddle_order' 0
cap fclean '^k_fclean$' 6
ls -la gpurun_out/prof
