#!/bin/bash
# Round-2 evidence: GPU tests, the default bench line, then ONE ncu session:
# the C2 launch list with DRAM traffic and a --set full capture of the
# dominant kernel (root_colpad_kernel) and the flush kernels.
O=gpurun_out/r02
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; echo "bench rc=$?" >> $O/bench_c2.err
python scripts/profile_search.py --config c2 --searches 2 > $O/plain.log 2>&1 && {
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --csv --log-file $O/c2_traffic.csv \
  python scripts/profile_search.py --config c2 --searches 2 > /dev/null 2>&1
full() {
  ncu --set full --clock-control none --import-source on -k regex:$1 --launch-skip $2 -c 1 \
    -o $O/$3 -f python scripts/profile_search.py --config c2 --searches 2 > /dev/null 2>&1
}
full root_colpad 1 c2_root_colpad
full cache_probe 9 c2_cache_probe
full score_cube8 9 c2_cube8
}
ls $O
