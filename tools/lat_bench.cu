// Dependent-issue latencies on B200 (one warp, clock64 around a chain of N
// dependent instructions): DFMA, DADD, DMMA m8n8k4 (accumulator chain), SHFL
// (64-bit = 2 SHFL), LDS.64, sqrt(double), rcp Newton, bar.sync of 256 threads.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/lat_bench tools/lat_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
constexpr int N = 256;
__global__ void k(double* out, long long* t, double seed) {
  __shared__ double sm[2048];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = (double)((i * 7 + 1) % 2048 / 8 * 8 + (i & 7)) ;
  __syncthreads();
  double x = seed + lane, y = seed * 0.5, z = 1.0 + 1e-9 * lane;
  long long t0, t1;
  if (warp == 0) {
    // DFMA chain
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < N; ++i) x = fma(x, z, y);
    t1 = clock64(); if (lane == 0) t[0] = t1 - t0;
    // DADD chain
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < N; ++i) x = x + y;
    t1 = clock64(); if (lane == 0) t[1] = t1 - t0;
    // DMMA accumulator chain
    double d0 = x, d1 = y;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < N; ++i) dmma(d0, d1, z, y);
    t1 = clock64(); if (lane == 0) t[2] = t1 - t0;
    x += d0 + d1;
    // DMMA, 4 independent chains
    double e0 = x, e1 = y, f0 = y, f1 = x, g0 = z, g1 = z;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < N / 4; ++i) { dmma(d0, d1, z, y); dmma(e0, e1, z, y); dmma(f0, f1, z, y); dmma(g0, g1, z, y); }
    t1 = clock64(); if (lane == 0) t[3] = t1 - t0;
    x += d0 + d1 + e0 + e1 + f0 + f1 + g0 + g1;
    // 64-bit shuffle chain
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < N; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1 + (i & 15));
    t1 = clock64(); if (lane == 0) t[4] = t1 - t0;
    // shuffle + add (butterfly stage)
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < N; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1 + (i & 15));
    t1 = clock64(); if (lane == 0) t[5] = t1 - t0;
    // LDS pointer chase (64-bit)
    int idx = lane;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < N; ++i) idx = (int)sm[idx] & 2047;
    t1 = clock64(); if (lane == 0) t[6] = t1 - t0;
    x += idx;
    // sqrt chain
    x = fabs(x) + 2.0;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = sqrt(x) + 3.0;
    t1 = clock64(); if (lane == 0) t[7] = t1 - t0;
    // division chain
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = 1.0 / x + 3.0;
    t1 = clock64(); if (lane == 0) t[8] = t1 - t0;
    // independent DFMA issue rate (8 chains)
    double a0 = x, a1 = x + 1, a2 = x + 2, a3 = x + 3, a4 = x + 4, a5 = x + 5, a6 = x + 6, a7 = x + 7;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < N / 8; ++i) {
      a0 = fma(a0, z, y); a1 = fma(a1, z, y); a2 = fma(a2, z, y); a3 = fma(a3, z, y);
      a4 = fma(a4, z, y); a5 = fma(a5, z, y); a6 = fma(a6, z, y); a7 = fma(a7, z, y);
    }
    t1 = clock64(); if (lane == 0) t[9] = t1 - t0;
    x += a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  }
  __syncthreads();
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < 64; ++i) __syncthreads();
  t1 = clock64(); if (threadIdx.x == 0) t[10] = (t1 - t0) * (N / 64);
  // named barrier among 4 warps
  if (warp < 4) {
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < 64; ++i) asm volatile("bar.sync 1, 128;\n" ::: "memory");
    t1 = clock64(); if (threadIdx.x == 0) t[11] = (t1 - t0) * (N / 64);
  }
  out[threadIdx.x] = x;
}
int main() {
  double* out; long long* t;
  cudaMalloc(&out, 256 * 8); cudaMalloc(&t, 16 * 8);
  for (int rep = 0; rep < 2; ++rep) k<<<1, 256>>>(out, t, 1.000001);
  long long h[16];
  cudaMemcpy(h, t, 16 * 8, cudaMemcpyDeviceToHost);
  const char* names[] = {"DFMA dependent", "DADD dependent", "DMMA dependent (accumulator)", "DMMA 4 chains (per instr)",
                         "SHFL.64 dependent", "SHFL.64 + DADD (butterfly stage)", "LDS.64 dependent", "sqrt(double)+DADD",
                         "1/x (double)+DADD", "DFMA 8 independent chains (per instr)", "__syncthreads (256 thr)", "bar.sync 1,128"};
  for (int i = 0; i < 12; ++i) printf("%-40s %.1f cycles\n", names[i], (double)h[i] / N);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
