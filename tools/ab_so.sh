# dev: kernel times (ncu launch list: round 2 dense stencil, rounds 10-12 list stencil) and
# whole-correction timing per library build in _ab/*.so
cp paper_2604_01397_b200/libexactz.so _ab/cur.so.bak
for so in _ab/*.so; do
  cp "$so" paper_2604_01397_b200/libexactz.so
  for fl in ${FLS:-0}; do
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l.csv python tools/one_case.py ${CFG:-C2} "" $fl > /dev/null 2>&1
    echo "$(basename $so) flags $fl: $(python tools/timeline.py gpurun_out/l.csv | sed -n 3p | grep -o 'stencil_key2[^=]*=[0-9]*') $(python tools/timeline.py gpurun_out/l.csv | sed -n 11,13p | grep -o 'stencil_list[a-z_]*=[0-9]*' | tr '\n' ' ')"
    echo "$(basename $so) flags $fl: $(QT_FLAGS=$fl REPS=3 python tools/quick_time.py ${CFG:-C2} | grep 'rep 2')"
  done
done
cp _ab/cur.so.bak paper_2604_01397_b200/libexactz.so
