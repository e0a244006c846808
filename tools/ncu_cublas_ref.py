"""Reference point for ncu's tensor-pipe counter: one cuBLAS bf16 GEMM (8192^3, the MEASURED_PEAKS shape) and one
fp32-with-TF32 GEMM, to be captured with
    ncu --metrics sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,\
sm__inst_executed_pipe_tensor.sum,gpu__time_duration.sum -k regex:"gemm|cutlass|nvjet" python tools/ncu_cublas_ref.py
so the same counter read on this repo's tcgen05 kernels can be scaled."""
import torch
torch.backends.cuda.matmul.allow_tf32 = True
n = 8192
a = torch.randn(n, n, device="cuda", dtype=torch.bfloat16)
b = torch.randn(n, n, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    c = a @ b
torch.cuda.synchronize()
a32, b32 = a.float(), b.float()
for _ in range(3):
    c32 = a32 @ b32
torch.cuda.synchronize()
print("done")
