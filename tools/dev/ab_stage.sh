#!/bin/bash
# stage probe of several trees: bash tools/dev/ab_stage.sh CFG DIR...
cfg=$1; shift
for d in "$@"; do
  echo "== $d"; (cd $d && HG_STREAMS=1 python tests/tools/stage_probe.py $cfg --no-parity 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], 'jacobi', d['stages']['jacobi'], {k:v for k,v in d['debug'].items() if k.startswith('jacobi')}); r=d['debug']['jac_round_cyc']; print('round0 phases', [r[i+1]-r[i] for i in range(5)], 'round1', [r[i+9]-r[i+8] for i in range(5)])")
done
