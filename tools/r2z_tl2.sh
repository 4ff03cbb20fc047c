#!/bin/bash
for args in "--tile-block 8 --stage-stream 1 --flush-priority 100000" "--tile-block 8 --stage-stream 1 --stage-window 256 --flush-priority 100000" "--tile-block 4 --stage-stream 1 --flush-priority 100000" "--tile-block 16 --stage-stream 1 --flush-priority 100000"; do
  echo "== $args"; timeout 300 python tools/e2e_timeline.py --bin-ms 5 $args 2>&1 | tail -12
done
