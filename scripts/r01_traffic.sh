#!/bin/bash
# DRAM traffic + duration of every launch: C2 (2 searches) and a C3 window, warm caches
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --cache-control none --csv --log-file gpurun_out/c2_traffic.csv \
  python scripts/profile_search.py --config c2 --searches 2 > gpurun_out/c2_traffic.log 2>&1
ncu --metrics $M --clock-control none --cache-control none --csv --launch-skip 3000 --launch-count 400 \
  --log-file gpurun_out/c3_traffic.csv python scripts/profile_search.py --config c3 --searches 1 > gpurun_out/c3_traffic.log 2>&1
python bench.py > gpurun_out/bench_c2_v5.json 2> gpurun_out/bench_c2_v5.err
python bench.py --config c3 --steps 3 --no-cpu-baseline > gpurun_out/bench_c3_v5.json 2> gpurun_out/bench_c3_v5.err
