#!/bin/bash
# Round-2 evidence refresh: GPU tests, bench lines (C2 default, C1, C3, C4,
# reference arm), C2 launch list with DRAM traffic, ncu --set full of the
# dominant C2 kernel and the C3 speculative-round kernels.
O=gpurun_out/${EVID:-r02x}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
python __graft_entry__.py > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
python bench.py --config c1 --steps 5 --no-cpu-baseline > $O/bench_c1.json 2> $O/bench_c1.err
python bench.py --config c3 --steps 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
python bench.py --config c4 --steps 3 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
BBS_COBATCH=1 BBS_GROUPS=4 python bench.py --config c4 --steps 3 --no-cpu-baseline > $O/bench_c4_cobatch.json 2> $O/bench_c4_cobatch.err
for cb in 0 1; do BBS_COBATCH=$cb BBS_GROUPS=4 C4_N=64 C4_SHARES=0 C4_CONCS=8,16,32 python scripts/c4_probe.py > $O/c4_probe_cobatch$cb.log 2>&1; done
python bench.py --impl reference --steps 3 > $O/bench_reference.json 2> $O/bench_reference.err
BBS_DEBUG_PHASES=1 python scripts/profile_search.py --config c2 --searches 2 > $O/c2_phases.log 2>&1
BBS_DEBUG_PHASES=1 python scripts/profile_search.py --config c3 --searches 1 > $O/c3_phases.log 2>&1
python scripts/profile_search.py --config c2 --searches 2 > $O/plain.log 2>&1 && {
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --csv --log-file $O/c2_traffic.csv \
  python scripts/profile_search.py --config c2 --searches 2 > /dev/null 2>&1
ncu --metrics $M --clock-control none --csv --launch-skip 150 --launch-count 300 --log-file $O/c3_traffic.csv \
  python scripts/profile_search.py --config c3 --searches 1 > /dev/null 2>&1
full() {
  ncu --set full --clock-control none --import-source on -k regex:$2 --launch-skip $3 -c 1 \
    -o $O/$1_$2 -f python scripts/profile_search.py --config $1 --searches 2 > /dev/null 2>&1
}
full c2 root_colpad 1
full c2 cache_probe 9
full c2 cache_build 0
full c3 frontier_auto 40
full c3 survivors_auto 40
full c3 cache_probe 60
full c3 merge_auto 40
full c2 root_select 0
}
ls $O
