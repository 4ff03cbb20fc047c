#!/bin/bash
for args in "--skew 32 --skew-block 16 --stage-stream 1" "--skew 32 --skew-block 8 --stage-stream 1" "--skew 64 --skew-block 16 --stage-stream 1" "--skew 16 --skew-block 16 --stage-stream 1" ; do
  echo "== $args"; timeout 300 python tools/e2e_timeline.py --bin-ms 5 $args 2>&1 | tail -6
done
