#!/bin/bash
# Quick A/B on the GPU box: the bench line without the NEXT rows / CPU baseline (parity kept), stage table.
#   tools/quick.sh [tag] [extra bench args]
tag=${1:-q}; shift
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 --no-cg --no-r2 --no-weights --no-schur --nested-levels 0 --no-tf32-peak "$@" \
  > gpurun_out/quick_$tag.json 2> gpurun_out/quick_$tag.err
echo "bench rc=$?"
python - <<PY
import json
d=json.load(open('gpurun_out/quick_$tag.json'))
print('ms_per_step', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],3), 'parity', d['parity'].get('F_rel_fro'), d['parity'].get('sigma_rel_max'), d['parity'].get('ok'))
for k,v in sorted(d['stages'].items(), key=lambda x:-x[1]['ms_per_step']):
    print(f"  {k:14s} {v['ms_per_step']:.3f} ms  {v['launches_per_step']:.0f}")
PY
