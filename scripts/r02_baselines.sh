#!/bin/bash
# Round-2 baselines of the secondary configs + per-phase epoch timings.
O=gpurun_out/r02c
mkdir -p $O
python bench.py --config c3 --steps 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
python bench.py --config c1 --steps 5 --no-cpu-baseline > $O/bench_c1.json 2> $O/bench_c1.err
python bench.py --config c4 --steps 3 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
BBS_DEBUG_PHASES=1 python scripts/profile_search.py --config c2 --searches 2 > $O/c2_phases.log 2>&1
BBS_DEBUG_PHASES=1 python scripts/profile_search.py --config c3 --searches 1 > $O/c3_phases.log 2>&1
ls $O
