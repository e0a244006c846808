python -m pytest tests -m gpu -x -q 2>&1 | tail -1
HG_JACOBI_CTA=256 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for m in 512 256; do
  HG_JACOBI_CTA=$m HG_STREAMS=1 python tests/tools/stage_probe.py 4 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cta $m probe jacobi', d['stages']['jacobi'], d['F_rel'], d['sigma_rel'], d['debug']['jacobi_total_sweeps'])"
  HG_JACOBI_CTA=$m python bench.py --steps 30 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cta $m bench:', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3), d['parity']['ok'])"
done
