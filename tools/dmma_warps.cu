// Per-warp DMMA issue limit: TFLOP/s of independent DMMA streams vs warps per
// SM sub-partition, for each FP64 mma.sync shape (8 independent accumulators
// per warp).  One CTA of 4*W warps per SM (W warps per SMSP).
#include <cstdio>
__device__ __forceinline__ void mma884(double* d, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a[0]), "d"(b[0]));
}
__device__ __forceinline__ void mma1684(double* d, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
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
template <int SHAPE, int NACC>
__global__ void k(double* out, int iters) {
  double d[NACC][4], a[8], b[4];
  for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) d[i][j] = 0;
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; ++i) b[i] = 1.0 / (i + 1);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      if (SHAPE == 0) mma884(d[i], a, b);
      else if (SHAPE == 1) mma1684(d[i], a, b);
      else if (SHAPE == 2) mma1688(d[i], a, b);
      else mma16816(d[i], a, b);
    }
  }
  double s = 0;
  for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) s += d[i][j];
  if (s == 1.2345) out[0] = s;
}
template <int SHAPE>
void run(double* out, int sms, const char* name) {
  const double fl[4] = {512, 1024, 2048, 4096};
  for (int w = 1; w <= 8; w *= 2) {
    const int iters = 2000 * 8 / (1 << SHAPE) / 2;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<SHAPE, 8><<<sms, 128 * w>>>(out, 10);
    cudaEventRecord(e0);
    k<SHAPE, 8><<<sms, 128 * w>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double flops = fl[SHAPE] * 8.0 * iters * sms * 4 * w;
    printf("{\"shape\": \"%s\", \"warps_per_smsp\": %d, \"tflops\": %.2f, \"cycles_per_mma_per_warp\": %.1f}\n", name, w,
           flops / ms / 1e9, ms * 1e-3 * 1.965e9 / (8.0 * iters));
  }
}
int main() {
  double* out; cudaMalloc(&out, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>(out, sms, "m8n8k4");
  run<1>(out, sms, "m16n8k4");
  run<2>(out, sms, "m16n8k8");
  run<3>(out, sms, "m16n8k16");
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
