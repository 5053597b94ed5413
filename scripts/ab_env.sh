#!/bin/bash
# A/B of an environment knob on one box: ab_env.sh VAR "v1 v2 ..." [configs]
VAR=$1; VALS=$2; CFGS=${3:-"c2 c1 c3"}
for v in $VALS; do
  echo "== $VAR=$v"
  for i in 1 2; do
    for c in $CFGS; do
      n=4; [ $c = c3 ] && n=3
      env $VAR=$v python scripts/profile_search.py --config $c --searches $n 2>/dev/null | tail -1 | cut -c1-110
    done
  done
done
