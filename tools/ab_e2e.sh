# dev: end-to-end (host buffers) timing of the builds in _ab/*.so, C2
cp paper_2604_01397_b200/libexactz.so /tmp/cur.so
for so in _ab/*.so; do
  cp "$so" paper_2604_01397_b200/libexactz.so
  echo "$(basename $so): $(python tools/e2e_time.py 2>&1 | tail -2 | tr '\n' ' ')"
done
cp /tmp/cur.so paper_2604_01397_b200/libexactz.so
