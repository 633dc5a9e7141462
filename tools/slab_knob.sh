# A/B of the sharded C3-cache start (EXACTZ_SLAB_CACHE_DIV: start once V_t * div <= bricks)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for d in 4 1 0; do
  echo "div $d" >> gpurun_out/slab_knob.txt
  EXACTZ_SLAB_CACHE_DIV=$d timeout 600 python tools/slabs_time.py C5 8 >> gpurun_out/slab_knob.txt 2>&1
  EXACTZ_SLAB_CACHE_DIV=$d timeout 600 python tools/slabs_time.py C2 8 >> gpurun_out/slab_knob.txt 2>&1
done
cat gpurun_out/slab_knob.txt
