// FP64 pipe microbenchmarks for B200 (sm_100a): DFMA, DMMA (mma.sync f64 shapes),
// DFMA+DMMA issued from the same warps, and exp() variants.  These numbers are the
// roofline denominators for the FP64-bound online-solve kernels (MEASURED_PEAKS.json
// has no FP64 entry).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peaks fp64_peaks.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1234.5) out[0] = s;
}

__device__ __forceinline__ void mma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void mma1688(double* d, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
__device__ __forceinline__ void mma16816(double* d, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

__global__ void k_dmma884(double* out, int iters) {
  double d[8][2];
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
#pragma unroll
  for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) mma884(d[i][0], d[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
  if (s == 1234.5) out[0] = s;
}

__global__ void k_dmma1688(double* out, int iters) {
  double d[4][4], a[4], b[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) { a[i] = threadIdx.x * 1e-3 + i; }
  b[0] = 1.0; b[1] = 0.5;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) d[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) mma1688(d[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += d[i][0] + d[i][1] + d[i][2] + d[i][3];
  if (s == 1234.5) out[0] = s;
}

__global__ void k_dmma16816(double* out, int iters) {
  double d[4][4], a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 1e-3 + i; }
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 / (i + 1);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) d[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) mma16816(d[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += d[i][0] + d[i][1] + d[i][2] + d[i][3];
  if (s == 1234.5) out[0] = s;
}

// Mixed: every iteration issues 4 m16n8k8 DMMA (4*2048 flops/warp) and `nf` DFMA per thread.
template <int NF>
__global__ void k_mixed(double* out, int iters, double fa, double fb) {
  double d[4][4], a[4], b[2], x[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = threadIdx.x * 1e-3 + i;
  b[0] = 1.0; b[1] = 0.5;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) d[i][j] = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) mma1688(d[i], a, b);
#pragma unroll
    for (int u = 0; u < NF / 8; ++u)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], fa, fb);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += d[i][0] + d[i][1] + d[i][2] + d[i][3];
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1234.5) out[0] = s;
}

__global__ void k_exp(double* out, int iters, double step) {
  double x = -(threadIdx.x + blockIdx.x * 7) * 1e-4, s = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) { s += exp(x); x -= step; }
  }
  if (s == 1234.5) out[0] = s;
}

static float time_it(void (*launch)(void*), void* arg, int reps = 5) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  launch(arg);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a);
    launch(arg);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

struct Cfg { double* out; int blocks, threads, iters; };
static void L_dfma(void* p) { Cfg* c = (Cfg*)p; k_dfma<<<c->blocks, c->threads>>>(c->out, c->iters, 0.999999, 1e-7); }
static void L_884(void* p) { Cfg* c = (Cfg*)p; k_dmma884<<<c->blocks, c->threads>>>(c->out, c->iters); }
static void L_1688(void* p) { Cfg* c = (Cfg*)p; k_dmma1688<<<c->blocks, c->threads>>>(c->out, c->iters); }
static void L_16816(void* p) { Cfg* c = (Cfg*)p; k_dmma16816<<<c->blocks, c->threads>>>(c->out, c->iters); }
static void L_mix16(void* p) { Cfg* c = (Cfg*)p; k_mixed<16><<<c->blocks, c->threads>>>(c->out, c->iters, 0.999999, 1e-7); }
static void L_mix32(void* p) { Cfg* c = (Cfg*)p; k_mixed<32><<<c->blocks, c->threads>>>(c->out, c->iters, 0.999999, 1e-7); }
static void L_mix64(void* p) { Cfg* c = (Cfg*)p; k_mixed<64><<<c->blocks, c->threads>>>(c->out, c->iters, 0.999999, 1e-7); }
static void L_exp(void* p) { Cfg* c = (Cfg*)p; k_exp<<<c->blocks, c->threads>>>(c->out, c->iters, 1e-6); }

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_mhz_attr\": %.0f}\n", prop.name, sms, clk_khz / 1e3);
  double* out; CK(cudaMalloc(&out, 64));
  for (int occ : {4, 8}) {
    Cfg c{out, sms * occ, 256, 4096};
    double t = time_it(L_dfma, &c);
    double flops = 2.0 * 64 * c.iters * (double)c.blocks * c.threads;
    printf("{\"test\": \"dfma\", \"blocks_per_sm\": %d, \"ms\": %.4f, \"tflops\": %.2f}\n", occ, t, flops / t / 1e9);
  }
  for (int occ : {2, 4, 8}) {
    Cfg c{out, sms * occ, 256, 2048};
    double t = time_it(L_884, &c);
    double flops = 8.0 * 512 * c.iters * (double)c.blocks * (c.threads / 32);
    printf("{\"test\": \"dmma_m8n8k4\", \"blocks_per_sm\": %d, \"ms\": %.4f, \"tflops\": %.2f}\n", occ, t, flops / t / 1e9);
    t = time_it(L_1688, &c);
    flops = 4.0 * 2048 * c.iters * (double)c.blocks * (c.threads / 32);
    printf("{\"test\": \"dmma_m16n8k8\", \"blocks_per_sm\": %d, \"ms\": %.4f, \"tflops\": %.2f}\n", occ, t, flops / t / 1e9);
    t = time_it(L_16816, &c);
    flops = 4.0 * 4096 * c.iters * (double)c.blocks * (c.threads / 32);
    printf("{\"test\": \"dmma_m16n8k16\", \"blocks_per_sm\": %d, \"ms\": %.4f, \"tflops\": %.2f}\n", occ, t, flops / t / 1e9);
  }
  {
    Cfg c{out, sms * 4, 256, 2048};
    void (*ls[3])(void*) = {L_mix16, L_mix32, L_mix64};
    int nfs[3] = {16, 32, 64};
    for (int k = 0; k < 3; ++k) {
      double t = time_it(ls[k], &c);
      double mflops = 4.0 * 2048 * c.iters * (double)c.blocks * (c.threads / 32);
      double fflops = 2.0 * nfs[k] * c.iters * (double)c.blocks * c.threads;
      printf("{\"test\": \"mixed_dmma1688_plus_dfma\", \"dfma_per_thread_per_4mma\": %d, \"ms\": %.4f, \"dmma_tflops\": %.2f, \"dfma_tflops\": %.2f, \"total_tflops\": %.2f}\n",
             nfs[k], t, mflops / t / 1e9, fflops / t / 1e9, (mflops + fflops) / t / 1e9);
    }
  }
  {
    Cfg c{out, sms * 8, 256, 256};
    double t = time_it(L_exp, &c);
    double n = 8.0 * c.iters * (double)c.blocks * c.threads;
    printf("{\"test\": \"libdevice_exp\", \"ms\": %.4f, \"gexp_per_s\": %.2f}\n", t, n / t / 1e6);
  }
  CK(cudaGetLastError());
  return 0;
}
