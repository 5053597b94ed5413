#!/bin/bash
# launch list of one C2 search (second of two) -> gpurun_out/c2_launches.csv
cfg=${1:-c2}
python scripts/profile_search.py --config $cfg --searches 2 > gpurun_out/${cfg}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${cfg}_launches.csv \
  python scripts/profile_search.py --config $cfg --searches 2 > gpurun_out/${cfg}_ncu.log 2>&1
tail -1 gpurun_out/${cfg}_plain.log
