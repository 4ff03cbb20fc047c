#!/bin/bash
for args in "--skew 32 --stage-stream 1 --tail-ms 30" "--skew 32 --stage-stream 1 --tail-ms 30 --flush-priority 100000"; do
  echo "== $args"; timeout 300 python tools/e2e_timeline.py --bin-ms 5 $args 2>&1 | tail -14
done
