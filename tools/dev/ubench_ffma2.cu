// FFMA vs FFMA2 (fma.rn.f32x2) issue throughput: 16 warps per SM, 8 independent chains each.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/dev/ubench_ffma2.cu -o /tmp/uf2 && /tmp/uf2
#include <cstdio>
__device__ __forceinline__ unsigned long long f2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
template <int MODE>
__global__ void k(float* out, long long* cyc, int n) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 0.001f + i;
  const float x = 0.999f, y = 0.001f;
  __syncthreads();
  long long t0 = clock64();
  if (MODE == 0) {
    for (int it = 0; it < n; ++it)
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], x, y);
  } else {
    unsigned long long p[8], xx, yy;
    float2 xf = make_float2(x, x), yf = make_float2(y, y);
    xx = *reinterpret_cast<unsigned long long*>(&xf);
    yy = *reinterpret_cast<unsigned long long*>(&yf);
    for (int i = 0; i < 8; ++i) { float2 v = make_float2(a[2 * i], a[2 * i + 1]); p[i] = *reinterpret_cast<unsigned long long*>(&v); }
    for (int it = 0; it < n; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) p[i] = f2(p[i], xx, yy);
    for (int i = 0; i < 8; ++i) { float2 v = *reinterpret_cast<float2*>(&p[i]); a[2 * i] = v.x; a[2 * i + 1] = v.y; }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 148 * 512 * 4); cudaMalloc(&c, 8);
  const int n = 4096;
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) k<0><<<148, 512>>>(o, c, n); else k<1><<<148, 512>>>(o, c, n);
    }
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    const double fma_per_sm_cycle = 512.0 * 16 * n / h;
    printf("%s: %lld cycles, %.1f fp32 FMA per SM-cycle\n", mode ? "FFMA2" : "FFMA ", h, fma_per_sm_cycle);
  }
  return 0;
}
