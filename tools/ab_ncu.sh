# dev: A/B of the builds in _ab/*.so: C2 timing twice, plus the ncu time of the round-0 dense stencil
cp paper_2604_01397_b200/libexactz.so /tmp/cur.so
for r in 1 2; do for so in _ab/*.so; do
  cp "$so" paper_2604_01397_b200/libexactz.so
  echo "$(basename $so) C2: $(python tools/quick_time.py C2 2>&1 | grep 'rep 2')"
done; done
for so in _ab/*.so; do
  cp "$so" paper_2604_01397_b200/libexactz.so
  echo "$(basename $so) ncu: $(ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:k_stencil_fast -c 1 python tools/one_case.py C2 2>&1 | grep -E 'duration|inst_executed' | tr -s ' ' | tr '\n' ' ')"
done
cp /tmp/cur.so paper_2604_01397_b200/libexactz.so
