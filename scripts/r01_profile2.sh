#!/bin/bash
# C3 epoch-loop window: launch list of 400 launches mid-search + full captures
mkdir -p gpurun_out
python scripts/profile_search.py --config c3 --searches 1 > gpurun_out/c3w_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --launch-skip 3000 --launch-count 400 \
  --log-file gpurun_out/c3w_launches.csv python scripts/profile_search.py --config c3 --searches 1 > gpurun_out/c3w_ncu.log 2>&1
full() {  # cfg kernel-regex skip tag
  ncu --set full --clock-control none --import-source on -k regex:$2 --launch-skip $3 -c 1 \
    -o gpurun_out/$4 -f python scripts/profile_search.py --config $1 --searches 1 > gpurun_out/$4.log 2>&1
}
full c3 survivors 300 c3_survivors
full c3 merge 300 c3_merge2
full c3 branch 300 c3_branch
ls gpurun_out
