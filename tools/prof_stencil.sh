# ncu captures of the first dense stencil launch of C2 for the given exactz flags
for fl in "$@"; do
  ncu --set full --clock-control none --import-source on -k regex:k_stencil -c 1 -o gpurun_out/p_st_$fl python tools/one_case.py C2 "" $fl > /dev/null 2>&1
done
