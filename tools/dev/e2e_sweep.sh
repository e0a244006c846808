python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for cfg in "2 0" "2 1" "3 0" "4 0" "4 1"; do
  set -- $cfg
  HG_STREAMS=$1 HG_STREAM_PRIO=$2 python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('parts $1 prio $2:', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3))"
done
