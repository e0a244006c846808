// Micro-benchmark: 32x32 tile POTRF variants (one warp), clock64 of the first and second call.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int TS = 32, LDT = 36;

__device__ __noinline__ void potrf_unrolled(float* T, int lane) {
  float a[TS];
#pragma unroll
  for (int t = 0; t < TS; ++t) a[t] = T[lane * LDT + t];
#pragma unroll
  for (int c = 0; c < TS; ++c) {
    float d = __shfl_sync(0xffffffffu, a[c], c);
    float inv = rsqrtf(d);
    inv = inv * fmaf(-0.5f * d * inv, inv, 1.5f);
    const float s = d * inv;
    if (lane == c) a[c] = s;
    if (lane > c) a[c] *= inv;
#pragma unroll 31
    for (int l = c + 1; l < TS; ++l) {
      const float v = __shfl_sync(0xffffffffu, a[c], l);
      if (lane >= l) a[l] = fmaf(-a[c], v, a[l]);
    }
  }
#pragma unroll
  for (int t = 0; t < TS; ++t) T[lane * LDT + t] = a[t];
  __syncwarp();
}

// compact: column loop at runtime, the pivot column of every lane staged in shared memory
__device__ __noinline__ void potrf_smem(float* T, int lane) {
  float a[TS];
#pragma unroll
  for (int t = 0; t < TS; ++t) a[t] = T[lane * LDT + t];
  __shared__ float colbuf[2][TS];
#pragma unroll 1
  for (int c = 0; c < TS; ++c) {
    // a[c] with a runtime c: select chain (compile-time register indices)
    float ac = a[0];
#pragma unroll
    for (int j = 1; j < TS; ++j) ac = (c == j) ? a[j] : ac;
    const float d = __shfl_sync(0xffffffffu, ac, c);
    float inv = rsqrtf(d);
    inv = inv * fmaf(-0.5f * d * inv, inv, 1.5f);
    const float lc = lane == c ? d * inv : (lane > c ? ac * inv : ac);
    colbuf[c & 1][lane] = lc;
    __syncwarp();
#pragma unroll
    for (int j = 0; j < TS; ++j) {
      const float v = colbuf[c & 1][j];                 // L[j][c] (broadcast)
      const float upd = (j > c && lane >= j) ? fmaf(-lc, v, a[j]) : a[j];
      a[j] = (j == c) ? lc : upd;
    }
  }
#pragma unroll
  for (int t = 0; t < TS; ++t) T[lane * LDT + t] = a[t];
  __syncwarp();
}

__global__ void bench(int variant, long long* out, float* res) {
  __shared__ float T[TS * LDT];
  const int lane = threadIdx.x;
  for (int rep = 0; rep < 2; ++rep) {
    for (int j = 0; j < TS; ++j) T[lane * LDT + j] = (lane == j ? 40.f : 0.f) + 1.0f / (1 + lane + j);
    __syncwarp();
    long long t0 = clock64();
    if (variant == 0) potrf_unrolled(T, lane); else potrf_smem(T, lane);
    long long t1 = clock64();
    if (lane == 0) out[rep] = t1 - t0;
  }
  for (int j = 0; j < TS; ++j) res[lane * TS + j] = T[lane * LDT + j];
}

int main() {
  long long* d; float* r; cudaMalloc(&d, 16); cudaMalloc(&r, 4 * 1024);
  float h0[1024], h1[1024];
  for (int v = 0; v < 2; ++v) {
    bench<<<1, 32>>>(v, d, r);
    long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(v ? h1 : h0, r, 4096, cudaMemcpyDeviceToHost);
    printf("variant %d: first %lld cycles, second %lld cycles\n", v, h[0], h[1]);
  }
  float md = 0; for (int i = 0; i < 32; ++i) for (int j = 0; j <= i; ++j) { float e = h0[i*32+j] - h1[i*32+j]; md = fmaxf(md, fabsf(e)); }
  printf("max |L_unrolled - L_smem| (lower) = %g\n", md);
}
