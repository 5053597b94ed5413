#!/bin/bash
# --set full capture of one C2 flush probe launch (and the cube kernel) for the
# probe-efficiency work; run only after profile_search exits 0 without ncu.
O=gpurun_out/probe
mkdir -p $O
python scripts/profile_search.py --config c2 --searches 2 > $O/plain.log 2>&1 || exit 1
full() {
  ncu --set full --clock-control none --import-source on -k regex:$1 --launch-skip $2 -c 1 \
    -o $O/$3 -f python scripts/profile_search.py --config c2 --searches 2 > /dev/null 2>&1
}
full cache_probe ${SKIP:-9} c2_cache_probe
full score_cube8 ${SKIP:-9} c2_cube8
ls $O
