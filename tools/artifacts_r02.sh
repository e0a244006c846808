#!/bin/bash
# Round-2 artifacts on the GPU box: bench line, one-step launch list with DRAM bytes, full-set
# captures of the top kernels.  Each ncu pass runs only after the same command exited 0 without ncu.
#   tools/artifacts_r02.sh [bench|list|full|all]
set -u
what=${1:-all}
mkdir -p gpurun_out
if [[ $what == bench || $what == all ]]; then
  python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
  tail -c 600 gpurun_out/bench.err
fi
if [[ $what == list || $what == all ]]; then
  out=$(HG_STREAMS=1 python tools/step_once.py --warmup 2); rc=$?
  echo "step_once rc=$rc: $out"
  L=$(echo "$out" | awk '{print $2}')
  if [[ $rc == 0 ]]; then
    HG_STREAMS=1 ncu -k regex:"gemm_|k_" -s $((2 * L)) -c $L --clock-control none \
      --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
      --log-file gpurun_out/launches.csv python tools/step_once.py --warmup 2 > gpurun_out/ncu_launches.log 2>&1
    echo "ncu list rc=$?"
  fi
fi
if [[ $what == full || $what == all ]]; then
  # one steady-state launch of each top kernel (third step; demangled names carry the template arguments:
  # <(int)256, (bool)1, (bool)1> = 3xF16 power product on twins, <128, 1, 1> = 3xF16 Gram, <256, 0, 0> = 3xTF32
  # Q-formation; k_apply_fused = the fused Eq. 15 kernel);
  # SPECS="name:regex:skip ..." selects a subset
  out=$(HG_STREAMS=1 python tools/step_once.py --warmup 2); rc=$?
  echo "step_once rc=$rc: $out"
  [[ $rc == 0 ]] || exit 1
  DEFAULT_SPECS="gemm_power_f16:gemm_tc_kernel<.int.256,..bool.1,..bool.1>:18 gemm_gram_f16:gemm_tc_kernel<.int.128,..bool.1,..bool.1>:20 \
gemm_qform_tf32:gemm_tc_kernel<.int.256,..bool.0,..bool.0>:34 cholinv2:k_cholinv2:24 sytrd:k_sytrd:2 jacobi:k_jacobi_blk:2 \
rows3:k_assemble_rows3:2 trideig:k_trideig:2 orgtr:k_orgtr:2 apply_fused:k_apply_fused:2"
  for spec in ${SPECS:-$DEFAULT_SPECS}; do
    IFS=: read name rx skip <<< "$spec"
    HG_STREAMS=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k regex:"$rx" -s $skip -c 1 -f -o gpurun_out/r02_${name}_full python tools/step_once.py --warmup 2 \
      > gpurun_out/ncu_${name}.log 2>&1
    echo "ncu full $name rc=$?"
  done
fi
