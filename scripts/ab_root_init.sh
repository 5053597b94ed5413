# A/B of the root-survivor queue init: device (default) vs host CUB path
# (BBS_ROOT_INIT=host); X=1 is the default.
for r in 1 2 3; do
for v in "BBS_ROOT_INIT=host" "X=1" "BBS_ROOT_INIT=device"; do
for c in ${CONFIGS:-c2 c3}; do
  echo -n "$c [$v] "; env $v timeout 300 python bench.py --config $c --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); l=d['latency_ms']; print(round(l['localization_total'],4), round(l['initial_nodes'],4))"
done; done; done
