#!/bin/bash
for args in "--skew 32" "--skew 32 --stage-stream 1" "--tile-block 8 --stage-stream 1 --stage-window 256" "--skew 32 --stage-stream 1 --stage-window 256"; do
  echo "== $args"; timeout 300 python tools/e2e_timeline.py --bin-ms 5 $args 2>&1 | tail -12
done
