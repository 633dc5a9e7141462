mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python tools/config_sweep.py C1 C2 C3 C4 C5 > gpurun_out/config_sweep.json 2> gpurun_out/config_sweep.err
tail -c 2000 gpurun_out/config_sweep.json | head -c 2000
