# round-end evidence (part A): build, smoke, all GPU tests, bench line, loopback scaling table
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; head -c 400 gpurun_out/bench.json
timeout 900 python tools/slabs_time.py C5 1 2 4 8 > gpurun_out/slabs_table.txt 2>&1
timeout 600 python tools/slabs_time.py C2 1 2 4 8 >> gpurun_out/slabs_table.txt 2>&1
timeout 900 python tools/slabs_time.py C3 1 8 >> gpurun_out/slabs_table.txt 2>&1
cat gpurun_out/slabs_table.txt
