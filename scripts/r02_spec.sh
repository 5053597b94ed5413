#!/bin/bash
# Speculative rounds: parity (GPU suite) and A/B timing vs one epoch per round.
O=gpurun_out/r02d
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for k in 1 4 8 16; do
  BBS_SPEC=$k python scripts/profile_search.py --config c2 --searches 6 > $O/c2_spec$k.log 2>&1
  BBS_SPEC=$k python scripts/profile_search.py --config c3 --searches 2 > $O/c3_spec$k.log 2>&1
done
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
tail -2 $O/pytest_gpu.log
grep -h "search [0-9]" $O/c*_spec*.log | cut -c1-120
