#!/bin/bash
# Same-box A/B of an environment knob through bench.py: ab_bench.sh VAR "v1 v2" [configs] [reps]
VAR=$1; VALS=$2; CFGS=${3:-"c2 c3 c4"}; REPS=${4:-2}
for r in $(seq $REPS); do
  for c in $CFGS; do
    for v in $VALS; do
      st=10; [ $c = c3 ] && st=5; [ $c = c4 ] && st=3
      echo "$VAR=$v $c: $(env $VAR=$v python bench.py --config $c --steps $st --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), "ms e2e", round(d["e2e"]["value"]/1e9,4))')"
    done
  done
done
