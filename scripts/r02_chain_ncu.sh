#!/bin/bash
# --set full captures of the C2 flush-chain kernels (frontier, branch,
# survivors, rank_sort, merge) at the 4th flush; run after profile_search
# exits 0 without ncu.
O=gpurun_out/chain
mkdir -p $O
python scripts/profile_search.py --config c2 --searches 2 > $O/plain.log 2>&1 || exit 1
for k in frontier_kernel branch_kernel survivors_kernel rank_sort_kernel merge_kernel cache_build_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:"^$k|::$k" --launch-skip ${SKIP:-3} -c 1 \
    -o $O/c2_$k -f python scripts/profile_search.py --config c2 --searches 2 > $O/$k.log 2>&1
done
ls $O
