set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "tracking or clean_path or parity_configs or host or nccl or slabs" > gpurun_out/dbg_pytest.log 2>&1; tail -3 gpurun_out/dbg_pytest.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "host" > gpurun_out/dbg_memcheck.log 2>&1; tail -3 gpurun_out/dbg_memcheck.log
