# A/B builds of the cube kernel's CTAs per SM (BBS_CUBE_MINB, also its cache-mode grid)
for v in 4 5 6; do
  rm -f paper_2310_10023_b200/csrc/build/score.o
  make -s -C paper_2310_10023_b200/csrc EXTRA="-DBBS_CUBE_MINB=$v" > /dev/null 2>&1 || echo build fail
  grep -A3 "Compiling entry.*score_cube8_kernelILb1" paper_2310_10023_b200/csrc/build/score.ptxas.log | grep -o "Used [0-9]* registers\|[0-9]* bytes spill stores" | tr '\n' ' '
  echo "== minb $v"
  for i in 1 2; do for c in c2 c3 c1; do python scripts/profile_search.py --config $c --searches 4 2>/dev/null | tail -1 | cut -c1-80; done; done
done
