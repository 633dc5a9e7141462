mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for e in "" "EXACTZ_SERIAL=1" "EXACTZ_NO_PRIO=1"; do
  echo "env: $e" >> gpurun_out/serial_ab.txt
  env $e REPS=5 timeout 300 python tools/quick_time.py C2 >> gpurun_out/serial_ab.txt 2>&1
done
cat gpurun_out/serial_ab.txt
