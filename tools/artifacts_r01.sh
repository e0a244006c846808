#!/bin/bash
# Round-1 artifacts on the GPU box: bench line, one-step launch list with DRAM bytes.
set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
L=$(HG_STREAMS=1 python tools/step_once.py --warmup 2 | awk '{print $2}')
echo "launches per step: $L"
HG_STREAMS=1 ncu -k regex:"gemm_tf32|k_" -s $((2 * L)) -c $L --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
    --log-file gpurun_out/launches.csv python tools/step_once.py --warmup 2 > gpurun_out/ncu_launches.log 2>&1
echo "ncu rc=$?"
