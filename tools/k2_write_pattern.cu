// Store-pattern microbenchmark for k_wy_stencil_rows (K2): pure stores, no arithmetic,
// with K2's address pattern.  A CTA owns RB selected rows x PB parameter values and
// writes RB x 8 bytes contiguous per (parameter value, column) into column-major
// [P][cpad][ld] blocks.  Question: is the 2.4 TB/s of K2's output stream a property of
// the 64-byte segments (RB = 8), i.e. would 128 / 256-byte segments (RB = 16 / 32) or a
// CTA that owns whole blocks run nearer the 7.36 TB/s of a plain fill?
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/k2_write_pattern tools/k2_write_pattern.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int RB>
__global__ void __launch_bounds__(256) k_pattern(double* __restrict__ out, int P, int s, int ld, int cpad, int PB) {
  constexpr int CG = 256 / RB;          // column groups of 4 per pass
  const int tid = threadIdx.x;
  const int i = tid % RB, cg = tid / RB;
  const int row = blockIdx.x * RB + i;
  const long p0 = (long)blockIdx.y * PB;
  if (row >= ld) return;
  for (int j0 = 4 * cg; j0 < cpad; j0 += 4 * CG) {
    double* ob = out + (p0 * cpad + j0) * (long)ld + row;
    for (int pl = 0; pl < PB && p0 + pl < P; ++pl) {
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) ob[cc * ld] = (double)(pl + cc);
      ob += (long)cpad * ld;
    }
  }
}

// whole blocks per CTA: 16-byte stores, fully contiguous
__global__ void __launch_bounds__(256) k_blocks(double2* __restrict__ out, int P, long blk2, int PB) {
  const long p0 = (long)blockIdx.x * PB;
  for (int pl = 0; pl < PB && p0 + pl < P; ++pl) {
    double2* ob = out + (p0 + pl) * blk2;
    for (long e = threadIdx.x; e < blk2; e += 256) ob[e] = make_double2(1.0, 2.0);
  }
}

template <typename F>
static float time_ms(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9f;
  for (int it = 0; it < 8; ++it) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  const int s = 200, ld = 200, cpad = 56, P = 17974;
  const size_t bytes = (size_t)P * cpad * ld * sizeof(double);
  double* out;
  cudaMalloc(&out, bytes);
  auto rep = [&](const char* name, float ms) {
    printf("{\"pattern\": \"%s\", \"ms\": %.4f, \"write_gbs\": %.1f}\n", name, ms, bytes / ms / 1e6);
  };
  rep("memset", time_ms([&] { cudaMemsetAsync(out, 0, bytes); }));
  rep("RB=8 PB=32 (K2 today)", time_ms([&] { k_pattern<8><<<dim3((s + 7) / 8, (P + 31) / 32), 256>>>(out, P, s, ld, cpad, 32); }));
  rep("RB=16 PB=32", time_ms([&] { k_pattern<16><<<dim3((s + 15) / 16, (P + 31) / 32), 256>>>(out, P, s, ld, cpad, 32); }));
  rep("RB=32 PB=32", time_ms([&] { k_pattern<32><<<dim3((s + 31) / 32, (P + 31) / 32), 256>>>(out, P, s, ld, cpad, 32); }));
  rep("RB=32 PB=8", time_ms([&] { k_pattern<32><<<dim3((s + 31) / 32, (P + 7) / 8), 256>>>(out, P, s, ld, cpad, 8); }));
  rep("RB=8 PB=8", time_ms([&] { k_pattern<8><<<dim3((s + 7) / 8, (P + 7) / 8), 256>>>(out, P, s, ld, cpad, 8); }));
  rep("whole blocks, PB=4", time_ms([&] { k_blocks<<<(P + 3) / 4, 256>>>((double2*)out, P, (long)cpad * ld / 2, 4); }));
  rep("whole blocks, PB=1", time_ms([&] { k_blocks<<<P, 256>>>((double2*)out, P, (long)cpad * ld / 2, 1); }));
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
