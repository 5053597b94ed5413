mkdir -p gpurun_out
for v in "256 3" "512 2" "1024 1" "512 1"; do set -- $v
  rm -f paper_2310_10023_b200/csrc/build/epoch_cache.o
  make -s -C paper_2310_10023_b200/csrc EXTRA="-DBBS_PROBE_T=$1 -DBBS_PROBE_B=$2" > /dev/null 2>&1 || echo build fail
  grep -A2 cache_probe paper_2310_10023_b200/csrc/build/epoch_cache.ptxas.log | grep -o "Used [0-9]* registers\|[0-9]* bytes spill stores" | tr '\n' ' '
  echo "== $1 $2"
  python scripts/profile_search.py --config c2 --searches 4 2>&1 | grep "search 3" | cut -c1-100
  python scripts/profile_search.py --config c3 --searches 2 2>&1 | grep "search 1" | cut -c1-100
done
