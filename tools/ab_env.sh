# dev: A/B timing of library builds in _ab/*.so over EXACTZ_CACHE_DIV values (C2 and C3)
cp paper_2604_01397_b200/libexactz.so /tmp/cur.so
for so in _ab/*.so; do
  cp "$so" paper_2604_01397_b200/libexactz.so
  if [ -n "$TESTS" ]; then
    echo "$(basename $so) tests: $(timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1)"
  fi
  for cfg in ${CFGS:-C2 C3}; do
    for cd in ${DIVS:-4}; do
      echo "$(basename $so) $cfg div=$cd: $(EXACTZ_CACHE_DIV=$cd python tools/quick_time.py $cfg 2>&1 | grep 'rep 2')"
    done
  done
done
cp /tmp/cur.so paper_2604_01397_b200/libexactz.so
