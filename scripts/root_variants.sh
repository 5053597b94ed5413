for v in 8 2 1; do
  rm -f paper_2310_10023_b200/csrc/build/score.o
  make -s -C paper_2310_10023_b200/csrc EXTRA="-DBBS_ROOT_BUCKETS=$v" > /dev/null 2>&1 || echo build fail
  echo "== buckets $v"
  python scripts/profile_search.py --config c2 --searches 4 2>&1 | grep "search 3" | cut -c1-100
  python scripts/profile_search.py --config c3 --searches 2 2>&1 | grep "search 1" | cut -c1-100
done
