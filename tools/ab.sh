# dev: A/B timing of library builds placed in _ab/*.so (C2 unless $1), interleaved twice
cfg=${1:-C2}
cp paper_2604_01397_b200/libexactz.so /tmp/cur.so
for r in 1 2; do
  for so in _ab/*.so; do
    cp "$so" paper_2604_01397_b200/libexactz.so
    echo "$(basename $so) $cfg: $(python tools/quick_time.py $cfg 2>&1 | grep 'rep 2')"
  done
done
cp /tmp/cur.so paper_2604_01397_b200/libexactz.so
