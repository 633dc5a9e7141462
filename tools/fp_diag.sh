# fpaths overflow diagnostics (EXACTZ_TIMELINE prints them) for C2 / C3
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in C2 C3; do EXACTZ_TIMELINE=1 timeout 300 python tools/one_case.py $c 2>&1 | grep -v "^pass" ; done > gpurun_out/fp_diag.log 2>&1
