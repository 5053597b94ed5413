#!/bin/bash
# Round-1 profiling pass: launch lists (C2, C3) + ncu --set full of the top kernels.
set -x
mkdir -p gpurun_out
for cfg in c2 c3; do
  python scripts/profile_search.py --config $cfg --searches 2 > gpurun_out/${cfg}_plain.log 2>&1 || exit 1
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${cfg}_launches.csv \
    python scripts/profile_search.py --config $cfg --searches 2 > gpurun_out/${cfg}_ncu.log 2>&1
done
full() {  # cfg kernel-regex skip tag
  ncu --set full --clock-control none --import-source on -k regex:$2 --launch-skip $3 -c 1 \
    -o gpurun_out/$4 -f python scripts/profile_search.py --config $1 --searches 2 > gpurun_out/$4.log 2>&1
}
full c2 root_colpad 1 c2_root_colpad
full c2 score_cube8 3 c2_cube8
full c3 cache_probe 300 c3_cache_probe
full c3 cache_build 100 c3_cache_build
full c3 frontier 300 c3_frontier
full c3 merge 300 c3_merge
ls -la gpurun_out
