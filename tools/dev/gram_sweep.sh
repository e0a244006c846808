python -m pytest tests -m gpu -x -q 2>&1 | tail -1
HG_GRAM_FULL=1 HG_BN_GRAM=256 python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('full 256:', round(d['ms_per_step'],3), d['parity']['ok'])"
python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lower 128:', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3), d['parity']['F_rel_fro'], d['parity']['ok'])"
HG_BN_GRAM=64 python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lower 64:', round(d['ms_per_step'],3), d['parity']['ok'])"
