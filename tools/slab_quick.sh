# sharded + parity tests, C5 / C2 8-slab timing
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_sp.log 2>&1; tail -2 gpurun_out/pytest_sp.log
timeout 600 python tools/slabs_time.py C5 8 > gpurun_out/slabs_q.txt 2>&1
timeout 600 python tools/slabs_time.py C2 8 >> gpurun_out/slabs_q.txt 2>&1
cat gpurun_out/slabs_q.txt
