for cfg in "--skew 64" "--skew 32" "--skew 128" "--skew 64 --gps 8" "--skew 64 --streams 48"; do
  echo "== $cfg"; timeout 600 python tools/e2e_timeline.py --bin-ms 10 $cfg 2>&1 | tail -4
done
