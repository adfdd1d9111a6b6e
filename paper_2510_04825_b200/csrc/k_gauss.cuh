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
                             int64_t n, int d, int s, int64_t ld, double* __restrict__ D) {
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
  D[(int64_t)i * ld + l] = acc;
}

constexpr int kGaussKC = 32;            // K chunk staged per pipeline stage
constexpr int kGaussLD = kGaussKC + 4;  // padded smem row stride (conflict-free fragments)
constexpr int kGaussStages = 3;         // cp.async pipeline depth
constexpr int kGaussMaxWarps = 10;      // row groups (8 rows each) per CTA -> 320 threads
// parameter values per CTA: keep PW*NT*2 accumulator doubles <= 24 (2 CTAs/SM)
template <int NT>
__host__ __device__ constexpr int gauss_pw() { return NT <= 3 ? 4 : (NT == 4 ? 3 : (NT <= 6 ? 2 : 1)); }

// Row blocking of the s selected rows: gy CTAs along grid.y with rows_cta rows each.
__host__ __device__ inline void gauss_row_blocks(int s, int* gy, int* rows_cta) {
  const int s_pad = ((s + 7) / 8) * 8;
  *gy = (s_pad + 8 * kGaussMaxWarps - 1) / (8 * kGaussMaxWarps);
  *rows_cta = 8 * ((s_pad / 8 + *gy - 1) / *gy);
}

template <int NT>
__host__ __device__ constexpr size_t gauss_smem_bytes(int rows_cta) {
  return (size_t)kGaussStages * (rows_cta + 8 * NT) * kGaussLD * sizeof(double) + 2048 * sizeof(double);
}

// Plan-time layouts (zero padded so the main loop needs no predicates):
//   Dp  [gy*rows_cta][n_pad]  row blocks of rows_cta (gauss_row_blocks), n_pad = KC*ceil(n/KC)
//   XT  [8*NT][n_pad]    X transposed, basis columns >= r are zero
// Padding is exact: a padded l contributes exp(-0)*0 = 0, padded rows are not stored.
__global__ void k_gauss_pack_xt(const double* __restrict__ X, int64_t n, int r, int64_t n_pad, int rows,
                                double* __restrict__ XT) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)rows * n_pad) return;
  int c = (int)(idx / n_pad);
  int64_t l = idx - (int64_t)c * n_pad;
  XT[idx] = (c < r && l < n) ? X[l * r + c] : 0.0;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}

// grid = (ceil(P / PW), ceil(s_pad / (8*kGaussMaxWarps))); block = 32 * (row groups of this block)
template <int NT, int PW, int MINB, bool SMEM_TAB>
__global__ void __launch_bounds__(32 * kGaussMaxWarps, MINB)
k_gauss_rows(const double* __restrict__ Dp,     // s_pad x n_pad
             const double* __restrict__ XT,     // 8NT x n_pad
             const int64_t* __restrict__ S,     // s
             const double* __restrict__ params, // P
             int64_t P, int s, int64_t n_pad, int r, double ridge,
             double* __restrict__ Mout) {       // P x s x r
  constexpr int XR = 8 * NT;
  extern __shared__ __align__(16) double gsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const int rows_cta = nwarps * 8;
  const int row0 = blockIdx.y * rows_cta;  // first selected row of this CTA
  const size_t stage_elems = (size_t)(rows_cta + XR) * kGaussLD;

  const int64_t pbase = (int64_t)blockIdx.x * PW;
  double ninv[PW];
#pragma unroll
  for (int u = 0; u < PW; ++u) {
    const int64_t p = pbase + u;
    const double sg = (p < P) ? params[p] : 1.0;
    ninv[u] = -(1.0 / (2.0 * sg * sg));  // reference: inv = 1.0 / (2.0 * sigma * sigma)
  }
  const int lrow = warp * 8 + (lane >> 2);  // A-fragment row within the CTA
  const int kq = lane & 3;                  // A-fragment column within the k-step
  const int grow = row0 + lrow;
  const int64_t srow = (grow < s) ? S[grow] : -1;
  double* tab_s = gsm + (size_t)kGaussStages * stage_elems;
  if (SMEM_TAB)
    for (int j = threadIdx.x; j < 2048; j += blockDim.x) tab_s[j] = g_exp2_tab2048[j];
  ExpTab tab{0.0, 0.0};
  if (!SMEM_TAB) tab = exp_tab_load(lane);

  double acc[PW][NT][2];
#pragma unroll
  for (int u = 0; u < PW; ++u)
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[u][t][0] = acc[u][t][1] = 0.0;

  const int64_t nchunks = n_pad / kGaussKC;
  constexpr int kChunk16 = kGaussKC / 2;  // 16-byte pieces per row per stage
  auto stage = [&](int64_t ch, int b) {
    double* base = gsm + (size_t)b * stage_elems;
    const int64_t l0 = ch * kGaussKC;
    const int tot = (rows_cta + XR) * kChunk16;
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
      const int row = e / kChunk16, q = e - row * kChunk16;
      const double* src = (row < rows_cta) ? Dp + (int64_t)(row0 + row) * n_pad + l0 + 2 * q
                                           : XT + (int64_t)(row - rows_cta) * n_pad + l0 + 2 * q;
      cp_async16(base + row * kGaussLD + 2 * q, src);
    }
  };

#pragma unroll
  for (int b = 0; b < kGaussStages - 1; ++b) {
    if (b < nchunks) stage(b, b);
    cp_async_commit();
  }
  for (int64_t ch = 0; ch < nchunks; ++ch) {
    cp_async_wait<kGaussStages - 2>();
    __syncthreads();
    {
      const int64_t nx = ch + kGaussStages - 1;
      if (nx < nchunks) stage(nx, (int)(nx % kGaussStages));
      cp_async_commit();
    }
    const double* dsb = gsm + (size_t)(ch % kGaussStages) * stage_elems;
    const double* xsb = dsb + (size_t)rows_cta * kGaussLD;
    const int64_t l0 = ch * kGaussKC;
    const int dcol = (srow >= l0 && srow < l0 + kGaussKC) ? (int)(srow - l0) : -1;
#pragma unroll 1
    for (int kk = 0; kk < kGaussKC; kk += 4) {
      const double dv = dsb[lrow * kGaussLD + kk + kq];
      double bf[NT];
#pragma unroll
      for (int t = 0; t < NT; ++t) bf[t] = xsb[(t * 8 + (lane >> 2)) * kGaussLD + kk + kq];
      const bool diag = (kk + kq) == dcol;
#pragma unroll
      for (int u = 0; u < PW; ++u) {
        double e = SMEM_TAB ? sas_exp64_t2k(dv * ninv[u], tab_s) : sas_exp64(dv * ninv[u], tab);
        if (diag) e = e + ridge;
#pragma unroll
        for (int t = 0; t < NT; ++t) dmma884(acc[u][t][0], acc[u][t][1], e, bf[t]);
      }
    }
  }
  cp_async_wait<0>();
  // C fragment: lane holds C[lane/4][2*(lane%4) + {0,1}]
  if (grow < s) {
#pragma unroll
    for (int u = 0; u < PW; ++u) {
      const int64_t p = pbase + u;
      if (p >= P) continue;
      double* out = Mout + (p * s + grow) * (int64_t)r;
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const int c0 = t * 8 + 2 * (lane & 3);
        if (c0 < r) out[c0] = acc[u][t][0];
        if (c0 + 1 < r) out[c0 + 1] = acc[u][t][1];
      }
    }
  }
}
