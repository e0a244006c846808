#!/bin/bash
# A/B of the working tree against a HEAD build copied to _ab_old/ (same box, alternating runs)
#   bash tools/dev/ab.sh [reps]
reps=${1:-3}
for i in $(seq $reps); do
  for v in new old; do
    d=.; [ $v = old ] && d=_ab_old
    (cd $d && python bench.py --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v', round(d['ms_per_step'],3), round(1e3*d['e2e']['value']**-1*0+d['e2e']['value'],1))")
  done
done
for v in new old; do
  d=.; [ $v = old ] && d=_ab_old
  echo "== $v stages (HG_STREAMS=1)"; (cd $d && HG_STREAMS=1 python tests/tools/stage_probe.py 1 --no-parity 2>&1 | tail -14)
done
