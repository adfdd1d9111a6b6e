// K4, column-owner layout for the large real shapes (configs 3 and 5).
// Same algorithm and outputs as k_lsq_mw (Householder QR of [W M | W t],
// reference linalg.py:89-113 via online.py:105-134), laid out so that a
// Householder step needs one CTA barrier and no cross-warp reduction:
//
//   row i    -> lane i mod 32, register slot u = i / 32 (every warp holds all rows)
//   column j -> warp j mod W,  register slot c = j / W  (cyclic over the warps)
//
// Step k applies reflector k (v, tau published in shared memory) to the
// columns j > k a warp owns: one dot product per column over the warp's rows,
// the NA dot products of a warp summed over its 32 lanes by a halving
// exchange (reduce-scatter) and the weights broadcast back, then the rank-1
// update in registers.  The owner of column k+1 applies reflector k to that
// column in the same pass and immediately forms reflector k+1 (look-ahead),
// so the next step can start after a single barrier.  The pivot slot of step
// k = kw + W*C0 is the template parameter C0: finished column slots drop out
// of the unrolled code.  All sums run in a fixed order (deterministic results).
#pragma once
#include "k_lsq_mw.cuh"

// Sum N per-lane values (N a power of two <= 8) over the 32 lanes of a warp.
// The halving exchanges (xor 16, 8, 4 for N = 8) leave lane l with a partial
// of value l >> (5 - log2 N); a butterfly over the remaining lane bits
// completes it.  Returns the total of value (lane >> (5 - log2 N)).
template <int N>
__device__ __forceinline__ double warp_reduce_scatter(double (&x)[N], int lane) {
  constexpr int LOGN = (N >= 8) ? 3 : (N >= 4) ? 2 : (N >= 2) ? 1 : 0;
#pragma unroll
  for (int lvl = 0; lvl < LOGN; ++lvl) {
    const int m = 16 >> lvl;
    const int h = N >> (lvl + 1);
    const bool up = (lane & m) != 0;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const double send = up ? x[i] : x[i + h];
      const double keep = up ? x[i + h] : x[i];
      x[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
    }
  }
  double v = x[0];
#pragma unroll
  for (int m = 16 >> LOGN; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  return v;
}

__host__ __device__ constexpr int cw_pow2(int n) { return n <= 1 ? 1 : n <= 2 ? 2 : n <= 4 ? 4 : 8; }
__host__ __device__ constexpr int cw_log2(int n) { return n >= 8 ? 3 : n >= 4 ? 2 : n >= 2 ? 1 : 0; }

struct CwShared {
  double* vbuf;   // 2 x 32*RA reflector vectors
  double* scal;   // 2 x {tau, beta}
  double* rdiag;  // R_kk
  double* nrm_s;  // |R_kk|
};

// Reflector k from column slot C of the calling warp (rows >= k):
//   |x| = sqrt(sum x_i^2), beta = -sign(x_k) |x|, tau = 1 / (|x| (|x| + |x_k|)),
//   v = x below k, x_k - beta on k, 0 above   (the formulas of k_lsq_mw)
template <int RA, int NCW, int C>
__device__ __forceinline__ void cw_reflector(const double (&A)[RA][NCW], int k, int lane, const CwShared& sh) {
  const int buf = k & 1;
  double ss = 0.0;
#pragma unroll
  for (int u = 0; u < RA; ++u) {
    const double x = (lane + 32 * u >= k) ? A[u][C] : 0.0;
    ss = fma(x, x, ss);
  }
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, m);
  const int uk = k >> 5;
  double al = 0.0;
#pragma unroll
  for (int u = 0; u < RA; ++u)
    if (u == uk) al = A[u][C];
  const double alpha = __shfl_sync(0xffffffffu, al, k & 31);
  const double nrm = sqrt(ss);
  const double aa = fabs(alpha);
  double beta = 0.0, tau = 0.0;
  if (nrm != 0.0) {
    beta = (aa == 0.0) ? -nrm : copysign(nrm, -alpha);  // -sign(x_k) |x| exactly (no reciprocal)
    tau = rcp_nr(nrm * (nrm + aa));
  }
  double* vb = sh.vbuf + buf * 32 * RA;
#pragma unroll
  for (int u = 0; u < RA; ++u) {
    const int i = lane + 32 * u;
    vb[i] = (i > k) ? A[u][C] : (i == k ? alpha - beta : 0.0);
  }
  if (lane == 0) {
    sh.scal[2 * buf] = tau;
    sh.scal[2 * buf + 1] = beta;
    sh.rdiag[k] = beta;
    sh.nrm_s[k] = nrm;
  }
}

template <int RA, int NCW, int W, int C0>
struct CwStep {
  static __device__ __forceinline__ void run(double (&A)[RA][NCW], int k, int kw, int warp, int lane, int r,
                                             const CwShared& sh) {
    constexpr int NA = NCW - C0;
    // columns in groups of at most 8, one reduce-scatter each
    constexpr int NA1 = NA < 8 ? NA : 8, NA2 = NA - NA1;
    constexpr int N21 = cw_pow2(NA1), N22 = cw_pow2(NA2 > 0 ? NA2 : 1);
    constexpr int SH1 = 5 - cw_log2(N21), SH2 = 5 - cw_log2(N22);
    const int buf = k & 1;
    const double* vb = sh.vbuf + buf * 32 * RA;
    const double tau = sh.scal[2 * buf];
    double v[RA];
#pragma unroll
    for (int u = 0; u < RA; ++u) v[u] = vb[lane + 32 * u];
    double d1[N21];
#pragma unroll
    for (int c = 0; c < N21; ++c) {
      double acc = 0.0;
      if (c < NA1) {
#pragma unroll
        for (int u = 0; u < RA; ++u) acc = fma(v[u], A[u][C0 + c], acc);
      }
      d1[c] = acc;
    }
    const double wl1 = tau * warp_reduce_scatter<N21>(d1, lane);
    double wl2 = 0.0;
    if constexpr (NA2 > 0) {
      double d2[N22];
#pragma unroll
      for (int c = 0; c < N22; ++c) {
        double acc = 0.0;
        if (c < NA2) {
#pragma unroll
          for (int u = 0; u < RA; ++u) acc = fma(v[u], A[u][C0 + NA1 + c], acc);
        }
        d2[c] = acc;
      }
      wl2 = tau * warp_reduce_scatter<N22>(d2, lane);
    }
    const bool pivot_done = warp <= kw;  // slot C0 holds column warp + W*C0 <= k
#pragma unroll
    for (int c = 0; c < NA; ++c) {
      double w;
      if (c < NA1)  // resolved at compile time (c is an unrolled index)
        w = __shfl_sync(0xffffffffu, wl1, c << SH1);
      else
        w = __shfl_sync(0xffffffffu, wl2, (c - NA1) << SH2);
      if (c == 0 && pivot_done) w = 0.0;
#pragma unroll
      for (int u = 0; u < RA; ++u) A[u][C0 + c] = fma(-v[u], w, A[u][C0 + c]);
    }
    // look-ahead: the owner of column k+1 forms reflector k+1
    if (k + 1 < r) {
      if (kw + 1 < W) {
        if (warp == kw + 1) cw_reflector<RA, NCW, C0>(A, k + 1, lane, sh);
      } else if constexpr (C0 + 1 < NCW) {
        if (warp == 0) cw_reflector<RA, NCW, C0 + 1>(A, k + 1, lane, sh);
      }
    }
    __syncthreads();
  }
};

template <int RA, int NCW, int W, int C0>
struct CwColumns {
  static __device__ __forceinline__ void run(double (&A)[RA][NCW], int warp, int lane, int r, const CwShared& sh) {
    if (C0 * W >= r) return;
#pragma unroll 1
    for (int kw = 0; kw < W; ++kw) {
      const int k = kw + W * C0;
      if (k >= r) return;
      CwStep<RA, NCW, W, C0>::run(A, k, kw, warp, lane, r, sh);
    }
    if constexpr (C0 + 1 < NCW) CwColumns<RA, NCW, W, C0 + 1>::run(A, warp, lane, r, sh);
  }
};

__host__ __device__ inline size_t lsq_cw_smem_bytes(int s, int r, int RA, size_t scratch, bool park = false) {
  const int ldm = r + 1;
  // Ms (s x ldm), R/y (r x ldm; aliases Ms when parked), c, R_kk, 2 reflector
  // vectors, 2 x {tau, beta}
  size_t n = (size_t)s * ldm + (park ? 0 : (size_t)r * ldm) + 2 * (size_t)r + 2 * 32 * (size_t)RA + 4;
  size_t bytes = (n * sizeof(double) + 15) / 16 * 16;
  return bytes + kLsqRedDoubles * sizeof(double) + (scratch + 15) / 16 * 16;
}

// PARK: the unweighted M (needed only by the explicit sampled residual at the
// end) is copied to this CTA's global (L2) slot mglob after the load into
// registers, and R reuses its shared-memory buffer: two CTAs per SM for the
// 200 x 51 shape (lsq_cw_smem_bytes(..., park = true)).
template <int RA, int NCW, int W, class Asm, int MINB = 1, bool PARK = false>
__global__ void __launch_bounds__(32 * W, MINB) k_lsq_cw(LsqArgs<double> a, Asm as, size_t scratch_bytes,
                                                         double* __restrict__ mglob = nullptr) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = a.s, r = a.r, ldm = r + 1;
  double* Ms = reinterpret_cast<double*>(smem_raw);
  double* Rs = PARK ? Ms : Ms + (size_t)s * ldm;
  double* cvec = Ms + (size_t)s * ldm + (PARK ? 0 : (size_t)r * ldm);
  CwShared sh;
  sh.rdiag = cvec + r;
  sh.vbuf = sh.rdiag + r;
  sh.scal = sh.vbuf + 2 * 32 * RA;
  const size_t core =
      ((size_t)s * ldm + (PARK ? 0 : (size_t)r * ldm) + 2 * (size_t)r + 2 * 32 * (size_t)RA + 4) * sizeof(double);
  double* mg = PARK ? mglob + (size_t)blockIdx.x * s * ldm : Ms;
  double* red = reinterpret_cast<double*>(smem_raw + (core + 15) / 16 * 16);  // residual partials (<= 16)
  sh.nrm_s = red + 16;
  double* rinfo = sh.nrm_s + 64;
  unsigned char* scratch = smem_raw + (core + 15) / 16 * 16 + kLsqRedDoubles * sizeof(double);
  (void)scratch_bytes;
  const CtaGroup grp;

  for (int64_t p = blockIdx.x; p < a.P; p += gridDim.x) {
    as(grp, p, Ms, ldm, s, r, scratch);
    for (int i = threadIdx.x; i < s; i += blockDim.x) Ms[i * ldm + r] = a.t[p * a.t_stride + i];
    __syncthreads();

    double A[RA][NCW];
    bool bad = false;
#pragma unroll
    for (int u = 0; u < RA; ++u) {
      const int i = lane + 32 * u;
      const double wi = (i < s && a.w) ? a.w[i] : 1.0;
#pragma unroll
      for (int c = 0; c < NCW; ++c) {
        const int j = warp + W * c;
        double m = 0.0;
        if (i < s && j <= r) {
          m = Ms[i * ldm + j];
          if (j < r && !isfinite(m)) bad = true;
          if (a.w) m *= wi;
        }
        A[u][c] = m;
      }
    }
    if (PARK)
      for (int idx = threadIdx.x; idx < s * ldm; idx += blockDim.x) mg[idx] = Ms[idx];
    if (__syncthreads_or(bad)) {
      lsq_nonfinite<double>(a, p);
      continue;
    }
    if (warp == 0) cw_reflector<RA, NCW, 0>(A, 0, lane, sh);
    __syncthreads();
    CwColumns<RA, NCW, W, 0>::run(A, warp, lane, r, sh);

    // strict upper R and y to shared memory
#pragma unroll
    for (int u = 0; u < RA; ++u) {
      const int i = lane + 32 * u;
#pragma unroll
      for (int c = 0; c < NCW; ++c) {
        const int j = warp + W * c;
        if (i < r && j > i && j <= r) Rs[i * ldm + j] = A[u][c];
      }
    }
    lsq_finish<double>(a, p, mg, ldm, Rs, cvec, sh.rdiag, sh.nrm_s, rinfo, red, W);
  }
}
