# A/B of root_colpad_kernel variants (prebuilt under variants/): min blocks
# per SM 1/3/4 (__launch_bounds__), odd vs even staged-window pitch.
for r in 1 2 3; do
for v in "mb1 BBS_EVEN_PITCH=1" "mb1 X=1" "mb3 X=1" "mb4 X=1"; do
  set -- $v
  cp variants/libbbs_b200_$1.so paper_2310_10023_b200/libbbs_b200.so
  for c in ${CONFIGS:-c2 c3}; do
    echo -n "$c [$v] "; env $2 timeout 300 python bench.py --config $c --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); l=d['latency_ms']; print(round(l['localization_total'],4), round(l['initial_nodes'],4))"
  done
done; done
