// K3 inner-loop ceiling experiments (no memory staging): per k-step PW values
// e_u = f(dv, b_u) feed NT DMMA.8x8x4 each.  f is one of:
//   0 sas_exp64_t2k_fr (table in shared memory)   1 same, table value replaced by a constant
//   2 five dependent DFMAs                        3 five independent DFMAs summed pairwise
//   4 one DMUL (no exp)
#include <cstdio>
#include "../paper_2510_04825_b200/csrc/sas_common.cuh"
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int MODE>
__device__ __forceinline__ double f(double dv, double b, float bf, const double* tab_s) {
  if (MODE == 0) return sas_exp64_t2k_fr(dv, b, bf, tab_s, -1);
  if (MODE == 1) {
    const int ah = max(__double2hiint(dv), 0x38000000);
    const float af = __int_as_float((ah - 0x38000000) << 3);
    const float pf = fmaxf(af * bf, -3.0e6f);
    const float kd32 = pf + 0x1.8p23f;
    const int ki = __float_as_int(kd32) - 0x4B400000;
    const int kb = __float_as_int(0x1.8p23f - kd32);
    const double kabs = __hiloint2double((kb >> 3) + 0x38000000, kb << 29);
    const double r = fma(dv, b, kabs);
    double q = fma(r, SAS_EXP2K_A3, SAS_EXP2K_A2);
    q = fma(q, r, SAS_EXP2K_A1);
    q = q * r;
    const double tv = 1.25;
    const double res = fma(tv, q, tv);
    const int hi = __double2hiint(res) + ((ki >> 11) << 20);
    const int keep = (ki >= SAS_EXP2K_KMIN) ? -1 : 0;
    return __hiloint2double(hi & keep, __double2loint(res) & keep);
  }
  if (MODE == 2) {
    double x = fma(dv, b, 1.0);
    x = fma(x, b, 0.5); x = fma(x, b, 0.25); x = fma(x, b, 0.125); return fma(x, b, 1.0);
  }
  if (MODE == 3) {
    double x0 = fma(dv, b, 1.0), x1 = fma(dv, b, 0.5), x2 = fma(dv, b, 0.25), x3 = fma(dv, b, 0.125), x4 = dv * b;
    return (x0 + x1) + (x2 + x3) + x4;  // 4 DADD extra
  }
  return dv * b;
}
template <int MODE, int PW, int NT>
__global__ void __launch_bounds__(320, 2) k_mix(double* out, int iters, double d0) {
  __shared__ double tab_s[2048];
  for (int j = threadIdx.x; j < 2048; j += blockDim.x) tab_s[j] = -g_exp2_tab2048[j];  // negated (sas_exp64_t2k_fr)
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double b[PW]; float bf[PW];
  for (int u = 0; u < PW; ++u) { b[u] = -0.1 - 0.05 * u; bf[u] = (float)b[u]; }
  double acc[PW][NT][2];
  for (int u = 0; u < PW; ++u) for (int t = 0; t < NT; ++t) acc[u][t][0] = acc[u][t][1] = 0;
  double dv = d0 + lane * 37.0, xb[NT];
  for (int t = 0; t < NT; ++t) xb[t] = 1.0 / (t + lane + 1);
#pragma unroll 2
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < PW; ++u) {
      const double e = f<MODE>(dv, b[u], bf[u], tab_s);
#pragma unroll
      for (int t = 0; t < NT; ++t) dmma884(acc[u][t][0], acc[u][t][1], e, xb[t]);
    }
    dv += 1.0;
  }
  double s = 0;
  for (int u = 0; u < PW; ++u) for (int t = 0; t < NT; ++t) s += acc[u][t][0] + acc[u][t][1];
  if (s == 12345.0) out[0] = s;
}
template <int MODE>
void run(const char* name, double* out) {
  const int iters = 4000;
  dim3 grid(148 * 2 * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k_mix<MODE, 4, 3><<<grid, 320>>>(out, 10, 0.5);
  cudaEventRecord(a);
  k_mix<MODE, 4, 3><<<grid, 320>>>(out, iters, 0.5);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double dmma = 512.0 * 3 * 4 * (double)iters * grid.x * 10;
  printf("{\"mode\": \"%s\", \"ms\": %.3f, \"dmma_tflops\": %.2f}\n", name, ms, dmma / ms / 1e9);
}
int main() {
  double* out; cudaMalloc(&out, 64);
  run<0>("exp_fr", out);
  run<1>("exp_fr_no_table", out);
  run<2>("5 dependent DFMA", out);
  run<3>("5 indep DFMA + 4 DADD", out);
  run<4>("1 DMUL", out);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
