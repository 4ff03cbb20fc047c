# e2e knob sweep (C2 through the API from pinned host tiles)
python tools/e2e_probe.py --streams 32 --gps 4 --skew 64 2>&1 | tail -3
for cfg in "--streams 32 --gps 4 --skew 32 --no-bw" "--streams 32 --gps 4 --skew 128 --no-bw" "--streams 32 --gps 8 --skew 64 --no-bw" "--streams 48 --gps 4 --skew 64 --no-bw" "--streams 32 --gps 4 --skew 64 --depth 256 --no-bw" "--streams 32 --gps 4 --skew 64 --prefetch 0 --no-bw"; do
  echo "== $cfg"; python tools/e2e_probe.py $cfg 2>&1 | grep "e2e step" | tail -1
done
