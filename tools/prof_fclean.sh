# ncu --set full of k_fclean (join list, C2, a mid round) and k_events / k_fpaths for comparison
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/prof
cap() {
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -o gpurun_out/prof/$1 python tools/one_case.py ${4:-C2} > /dev/null 2>&1
  ncu -i gpurun_out/prof/$1.ncu-rep --page raw --csv > gpurun_out/prof/$1_raw.csv
  ncu -i gpurun_out/prof/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/prof/$1_src.csv
  ncu -i gpurun_out/prof/$1.ncu-rep --page details --csv > gpurun_out/prof/$1_details.csv
  rm -f gpurun_out/prof/$1.ncu-rep
}
cap fclean '^k_fclean$' 4
cap events '^k_events$' 30
cap fpaths '^k_fpaths$' 0
cap fpaths3 '^k_fpaths$' 0 C3
for n in fclean events fpaths fpaths3; do python tools/ncu_quick_csv.py gpurun_out/prof/${n}_raw.csv gpurun_out/prof/${n}_src.csv > gpurun_out/prof/${n}_summary.txt 2>&1; done
for fl in 0 0x100000; do QT_FLAGS=$fl REPS=3 python tools/quick_time.py C2 | grep "rep 2" | sed "s/^/flags $fl C2 /"; QT_FLAGS=$fl REPS=2 python tools/quick_time.py C3 | grep "rep 1" | sed "s/^/flags $fl C3 /"; done > gpurun_out/pipe_ab.log 2>&1
