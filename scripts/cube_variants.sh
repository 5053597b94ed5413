for v in 1024 2048 512 1024; do
  rm -f paper_2310_10023_b200/csrc/build/score.o
  make -s -C paper_2310_10023_b200/csrc EXTRA="-DBBS_CUBE_TILE=$v" > /dev/null 2>&1 || echo build fail
  echo "== tile $v"
  python scripts/profile_search.py --config c2 --searches 5 2>&1 | grep "search [34]" | cut -c1-100
  python scripts/profile_search.py --config c1 --searches 4 2>&1 | grep "search 3" | cut -c1-100
done
