# dev: walk memo on/off (EXACTZ_NO_MEMO) for the builds in _ab/*.so, C2 and C3
cp paper_2604_01397_b200/libexactz.so /tmp/cur.so
for so in _ab/*.so; do
  cp "$so" paper_2604_01397_b200/libexactz.so
  for cfg in ${CFGS:-C2 C3}; do
    echo "$(basename $so) $cfg memo: $(python tools/quick_time.py $cfg 2>&1 | grep 'rep 2')"
    echo "$(basename $so) $cfg nomemo: $(EXACTZ_NO_MEMO=1 python tools/quick_time.py $cfg 2>&1 | grep 'rep 2')"
  done
done
cp /tmp/cur.so paper_2604_01397_b200/libexactz.so
