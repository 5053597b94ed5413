#!/bin/bash
# Round-1 evidence refresh: GPU tests, benches (C2 default, C3, C4, reference arm),
# C5 sweep, launch list with DRAM traffic, ncu --set full of the top kernels.
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
python bench.py --config c3 --steps 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
python bench.py --config c4 --steps 3 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
python bench.py --config c1 --steps 5 --no-cpu-baseline > $O/bench_c1.json 2> $O/bench_c1.err
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 python scripts/sweep_c5.py > $O/sweep_c5.json 2> $O/sweep_c5.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --cache-control none --csv --log-file $O/c2_traffic.csv \
  python scripts/profile_search.py --config c2 --searches 2 > /dev/null 2>&1
ncu --metrics $M --clock-control none --cache-control none --csv --launch-skip 3000 --launch-count 400 \
  --log-file $O/c3_traffic.csv python scripts/profile_search.py --config c3 --searches 1 > /dev/null 2>&1
full() {
  ncu --set full --clock-control none --import-source on -k regex:$2 --launch-skip $3 -c 1 \
    -o $O/$4 -f python scripts/profile_search.py --config $1 --searches 1 > /dev/null 2>&1
}
full c2 root_colpad 0 c2_root_colpad
full c2 cache_probe 2 c2_cache_probe
full c2 score_cube8 3 c2_cube8
full c3 cache_probe 300 c3_cache_probe
full c3 merge 300 c3_merge
BBS_DEBUG_PHASES=1 python scripts/profile_search.py --config c2 --searches 2 > $O/c2_phases.log 2>&1
BBS_DEBUG_PHASES=1 python scripts/profile_search.py --config c3 --searches 2 > $O/c3_phases.log 2>&1
ls $O
