// K3: Gaussian-kernel row contraction for a batch of bandwidths p.
//
//   M_p[i][j] = sum_l E_p(i,l) X[l][j],
//   E_p(i,l)  = exp(-(D[i][l] * inv_p)) (+ ridge if l == S_i),  inv_p = 1/(2 p p)
//
// This is what the reference computes per p with the dense detour
//   online._sampled_rows -> rows_dense -> row_fn -> @ basis.basis
// (online.py:57-65, systems.py:151-162, _kernels.py:38-50 for the 1-D rbf_rows;
// the ridge is added to the kernel entry before the product, as `out[k, i] += lam`
// in _kernels.py:49).  D = squared distances of the s selected points to all n
// points (p-independent, built once per plan by k_gauss_dist), so only the exp
// and the contraction are per p.
//
// GEMM view per CTA: rows (p, i) for PW parameter values x all s rows, columns
// = basis columns (8*NT >= r), K = n.  One warp owns an 8-row group i0..i0+7
// for PW parameters; per k-step of 4 each lane evaluates PW exps (A-fragment
// element of mma.m8n8k4: row lane/4, col lane%4) and issues PW*NT DMMA
// (mma.sync.m8n8k4.f64, SASS DMMA.8x8x4 — the only FP64 tensor shape on sm_100a;
// FP64 has no tcgen05 kind).  D and X tiles are staged in shared memory with
// cp.async (double-buffered) and reused by all PW parameters of the CTA.
#pragma once
#include "sas_common.cuh"

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// D[i][l] = sum_k (x_{S_i,k} - x_{l,k})^2, sequential over k, no FMA
// (the harness row oracle's order; see oracle/systems_ref.py gauss rows).
__global__ void k_gauss_dist(const double* __restrict__ pts, const int64_t* __restrict__ S,
                             int64_t n, int d, int s, double* __restrict__ D) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)s * n) return;
  int i = (int)(idx / n);
  int64_t l = idx - (int64_t)i * n;
  const double* xi = pts + S[i] * d;
  const double* xl = pts + l * d;
  double acc = 0.0;
  for (int k = 0; k < d; ++k) {
    double df = __dsub_rn(xi[k], xl[k]);
    acc = __dadd_rn(acc, __dmul_rn(df, df));
  }
  D[idx] = acc;
}

constexpr int kGaussKC = 32;            // K chunk staged per pipeline stage
constexpr int kGaussLD = kGaussKC + 4;  // padded row stride (conflict-free fragments)

template <int NT, int PW>
__host__ __device__ constexpr size_t gauss_smem_bytes(int s_pad) {
  return (size_t)2 * (s_pad + 8 * NT) * kGaussLD * sizeof(double);
}

// grid.x = ceil(P / PW); block = 32 * (s_pad / 8)
template <int NT, int PW>
__global__ void __launch_bounds__(384) k_gauss_rows(const double* __restrict__ D,   // s x n
                                                    const double* __restrict__ X,   // n x r
                                                    const int64_t* __restrict__ S,  // s
                                                    const double* __restrict__ params,  // P
                                                    int64_t P, int s, int64_t n, int r,
                                                    double ridge,
                                                    double* __restrict__ Mout) {  // P x s x r
  extern __shared__ __align__(16) double gsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const int s_pad = nwarps * 8;
  const int XR = 8 * NT;
  double* Ds[2] = {gsm, gsm + (size_t)(s_pad + XR) * kGaussLD};
  double* Xs[2] = {gsm + (size_t)s_pad * kGaussLD, gsm + (size_t)(s_pad + XR) * kGaussLD + (size_t)s_pad * kGaussLD};

  const int64_t pbase = (int64_t)blockIdx.x * PW;
  double inv[PW];
#pragma unroll
  for (int u = 0; u < PW; ++u) {
    int64_t p = pbase + u;
    double sg = (p < P) ? params[p] : 1.0;
    inv[u] = 1.0 / (2.0 * sg * sg);  // reference: inv = 1.0 / (2.0 * sigma * sigma)
  }
  const int row = warp * 8 + (lane >> 2);   // A-fragment row = selected row i
  const int kq = lane & 3;                  // A-fragment col within the k-step
  const int64_t srow = (row < s) ? S[row] : -1;
  const ExpTab tab = exp_tab_load(lane);

  double acc[PW][NT][2];
#pragma unroll
  for (int u = 0; u < PW; ++u)
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[u][t][0] = acc[u][t][1] = 0.0;

  const int64_t nchunks = (n + kGaussKC - 1) / kGaussKC;
  auto stage = [&](int64_t ch, int b) {
    const int64_t l0 = ch * kGaussKC;
    // D tile: s_pad x KC
    for (int e = threadIdx.x; e < s_pad * kGaussKC; e += blockDim.x) {
      int i = e / kGaussKC, kk = e - i * kGaussKC;
      int64_t l = l0 + kk;
      bool ok = (i < s) && (l < n);
      cp_async8(&Ds[b][i * kGaussLD + kk], ok ? (const void*)(D + (int64_t)i * n + l) : (const void*)D, ok);
    }
    // X tile transposed: Xs[col][kk]
    for (int e = threadIdx.x; e < XR * kGaussKC; e += blockDim.x) {
      int kk = e / XR, c = e - kk * XR;
      int64_t l = l0 + kk;
      bool ok = (c < r) && (l < n);
      cp_async8(&Xs[b][c * kGaussLD + kk], ok ? (const void*)(X + l * r + c) : (const void*)X, ok);
    }
    cp_async_commit();
  };

  stage(0, 0);
  for (int64_t ch = 0; ch < nchunks; ++ch) {
    const int b = (int)(ch & 1);
    if (ch + 1 < nchunks) {
      stage(ch + 1, b ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* dsb = Ds[b];
    const double* xsb = Xs[b];
    const int64_t l0 = ch * kGaussKC;
#pragma unroll 2
    for (int kk = 0; kk < kGaussKC; kk += 4) {
      const double dv = dsb[row * kGaussLD + kk + kq];
      double bf[NT];
#pragma unroll
      for (int t = 0; t < NT; ++t) bf[t] = xsb[(t * 8 + (lane >> 2)) * kGaussLD + kk + kq];
      const bool diag = (l0 + kk + kq) == srow;
#pragma unroll
      for (int u = 0; u < PW; ++u) {
        double e = sas_exp64(-(dv * inv[u]), tab);
        if (diag) e = e + ridge;
#pragma unroll
        for (int t = 0; t < NT; ++t) dmma884(acc[u][t][0], acc[u][t][1], e, bf[t]);
      }
    }
    __syncthreads();
  }
  // C fragment: lane holds C[lane/4][2*(lane%4) + {0,1}]
  const int crow = warp * 8 + (lane >> 2);
#pragma unroll
  for (int u = 0; u < PW; ++u) {
    const int64_t p = pbase + u;
    if (p >= P || crow >= s) continue;
    double* out = Mout + (p * s + crow) * (int64_t)r;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int c0 = t * 8 + 2 * (lane & 3);
      if (c0 < r) out[c0] = acc[u][t][0];
      if (c0 + 1 < r) out[c0 + 1] = acc[u][t][1];
    }
  }
}
