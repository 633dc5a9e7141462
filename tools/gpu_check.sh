# one GPU call: build, smoke, GPU tests, bench line, C2/C3 launch lists (timelines)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/bench.json | head -c 600
if [ -n "$TIMELINES" ]; then
for c in $TIMELINES; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python tools/one_case.py $c > /dev/null 2>&1
python tools/timeline.py gpurun_out/launches_$c.csv > gpurun_out/timeline_$c.txt
done
fi
if [ -n "$QT" ]; then
for c in $QT; do REPS=3 timeout 300 python tools/quick_time.py $c >> gpurun_out/quick_time.log 2>&1; done
fi
