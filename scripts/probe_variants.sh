mkdir -p gpurun_out
# A/B builds of the probe's block shape (BBS_PROBE_T threads, BBS_PROBE_B min CTAs per SM)
for v in ${VARIANTS:-"1024 1" "512 2" "256 3"}; do set -- $v
  rm -f paper_2310_10023_b200/csrc/build/epoch_cache.o
  make -s -C paper_2310_10023_b200/csrc EXTRA="-DBBS_PROBE_T=$1 -DBBS_PROBE_B=$2" > /dev/null 2>&1 || echo build fail
  grep -A2 cache_probe paper_2310_10023_b200/csrc/build/epoch_cache.ptxas.log | grep -o "Used [0-9]* registers\|[0-9]* bytes spill stores" | tr '\n' ' '
  echo "== $1 $2"
  for i in 1 2; do
    python scripts/profile_search.py --config c2 --searches 4 2>&1 | tail -1 | cut -c1-100
    python scripts/profile_search.py --config c3 --searches 3 2>&1 | tail -1 | cut -c1-100
  done
done
