// K4: batched weighted least squares, W warps cooperating on one parameter
// value (W = 1 for small problems).  Replaces linalg.solve_ls
// (reference linalg.py:89-113) as called from online.solve_online
// (online.py:105-134):
//
//   M_w = diag(w) M, t_w = diag(w) t           (linalg.py:102-105)
//   Householder QR of [M_w | t_w]              (np.linalg.qr, linalg.py:106)
//   rank test  min|R_ii| < 1e-12 max|R_ii|      (linalg.py:107-112)
//   c = R^{-1} (Q^H t_w)[:r]                    (solve_triangular, linalg.py:113)
//   sampled residual ||w * (M c - t)||          (online.py:121-124, recomputed
//                                                explicitly from the unweighted M)
//   output value  (c^H X) c                     (online.py:125-127)
//
// Layout: lane = a + RG*b (a < RG row groups, b < CG = 32/RG column groups);
// the global row group of a lane is w*RG + a, so row i lives in row group
// i mod (W*RG), slot u = i / (W*RG); column j (the rhs is column r) in column
// group j mod CG, slot v = j / CG.  The augmented matrix sits in registers
// A[RA][CB]; the unweighted M(p) stays in shared memory for the residual.
//
// Householder step k, Gram-row formulation (one reduction per column):
//   x_i = M_ik            shuffle from column group k mod CG of the same rows
//   g_j = sum_i conj(x_i) M_ij    own rows, butterfly over the warp's RG row
//                         groups, warp partials in shared memory; after a
//                         barrier one thread per column sums the W partials in
//                         warp order (a second barrier publishes the totals)
//   |x| = sqrt(g_kk), beta = -e^{i arg M_kk} |x|, tau = 2 / v^H v
//   M_ij -= tau v_i (g_j - conj(beta) M_kj)      for j > k
// The column loop is split as k = bk + CG*vk with the slot vk unrolled; W is a
// template parameter and W*RG a multiple of CG, so the register slots of
// column k and of row k are compile-time indices and finished column and row
// slots drop out of the unrolled code.  Reductions are in a fixed order:
// results do not depend on the grid, the batch or the number of GPUs.
//
// The assembler functor fills shared memory with the unweighted M(p):
//   AsmGlobal  - M precomputed by another kernel (Gaussian kernel rows, K3)
//   AsmAffine  - M = sum_k f_k(p) B_k with numpy's operation order (K1)
//   AsmStencil - edge-form stencil rows with exp-affine coefficients (K2)
#pragma once
#include "k_lsq.cuh"

template <typename T>
__device__ __forceinline__ T shfl_t(T v, int src);
template <>
__device__ __forceinline__ double shfl_t<double>(double v, int src) {
  return __shfl_sync(0xffffffffu, v, src);
}
template <>
__device__ __forceinline__ cplx shfl_t<cplx>(cplx v, int src) {
  return cplx{__shfl_sync(0xffffffffu, v.re, src), __shfl_sync(0xffffffffu, v.im, src)};
}
template <typename T>
__device__ __forceinline__ T shfl_xor_t(T v, int m);
template <>
__device__ __forceinline__ double shfl_xor_t<double>(double v, int m) {
  return __shfl_xor_sync(0xffffffffu, v, m);
}
template <>
__device__ __forceinline__ cplx shfl_xor_t<cplx>(cplx v, int m) {
  return cplx{__shfl_xor_sync(0xffffffffu, v.re, m), __shfl_xor_sync(0xffffffffu, v.im, m)};
}

// 1/x to ~1 ulp: hardware reciprocal seed (MUFU.RCP64H) + two Newton steps.
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

// shared doubles after the matrix buffers: 16 residual partials, |R_kk| per
// column (r <= 64), rank-test result (2)
constexpr int kLsqRedDoubles = 16 + 64 + 2;

template <typename T>
__host__ __device__ inline size_t lsq_mw_smem_bytes(int s, int r, int W, int CGxCB, size_t scratch) {
  const int ldm = r + 1;
  // Ms (s x ldm), R/y (r x ldm), c (r), R_kk (r),
  // 2 x [row k (CG*CB) + partials (W x CG*CB)]
  size_t n = (size_t)s * ldm + (size_t)r * ldm + 2 * (size_t)r + 2 * ((size_t)CGxCB + (size_t)W * CGxCB) +
             (size_t)CGxCB;
  size_t bytes = (n * sizeof(T) + 15) / 16 * 16;
  return bytes + kLsqRedDoubles * sizeof(double) + (scratch + 15) / 16 * 16;
}

// threads per column when the W warp partials are summed: a power of two
// <= min(W, 32) with TPC * LDP <= 32 * W
__host__ __device__ constexpr int lsq_tpc(int W, int LDP, int t = 1) {
  return (2 * t <= W && 2 * t * LDP <= 32 * W && 2 * t <= 32) ? lsq_tpc(W, LDP, 2 * t) : t;
}

// One Householder step for column k = bk + CG*VK.  With NRG = W*RG a multiple
// of CG, the pivot row k lies in row slot UK = VK / (NRG/CG) for every bk, so
// both the column slot of k and the row slot of row k are compile-time
// constants: row slots u < UK hold finished R rows (skipped), u > UK hold rows
// below the pivot, and only slot UK needs a per-lane test.
template <typename T, int RG, int RA, int CB, int W>
struct LsqStep {
  using S = Sc<T>;
  static constexpr int CG = 32 / RG;
  static constexpr int NRG = W * RG;
  static constexpr int LDP = CG * CB;  // padded row length of the shared row/partial buffers
  static_assert(NRG % CG == 0, "row groups must be a multiple of the column groups");

  template <int VK>
  static __device__ __forceinline__ void run(T (&A)[RA][CB], int k, int bk, int la, int lb, int grg, int warp,
                                             int r, T* rk_s, T* pt, T* sj_s, T* rdiag, double* nrm_s) {
    constexpr int UK = VK / (NRG / CG);
    const int gk = CG * (VK % (NRG / CG)) + bk;  // row group of row k
    // x_i = M_ik for own rows from column group bk (static slot VK)
    T xg[RA];
#pragma unroll
    for (int u = UK; u < RA; ++u) {
      const T xv = shfl_t(A[u][VK], la + RG * bk);
      xg[u] = (u > UK || grg >= gk) ? xv : S::zero();
    }
    // the owner of row k publishes it (static slot UK; the buffer is padded to CG*CB)
    if (grg == gk) {
#pragma unroll
      for (int v = VK; v < CB; ++v) rk_s[lb + CG * v] = A[UK][v];
    }
    // Gram row over rows >= k, butterfly over the RG row groups of the warp
#pragma unroll
    for (int v = VK; v < CB; ++v) {
      T acc = S::zero();
#pragma unroll
      for (int u = UK; u < RA; ++u) acc = S::fma_conj(xg[u], A[u][v], acc);
#pragma unroll
      for (int off = 1; off < RG; off <<= 1) acc = S::add(acc, shfl_xor_t(acc, off));
      if (la == 0) pt[warp * LDP + lb + CG * v] = acc;
    }
    __syncthreads();
    T sj[CB];
    T beta;
    if constexpr (W > 1) {
      // TPC threads per column sum the W warp partials (fixed order: strided
      // partial sums, then a butterfly), every group also forms g_kk and the
      // reflector scalars, and publishes w_j = tau (g_j - conj(beta) M_kj)
      constexpr int TPC = lsq_tpc(W, LDP);
      const int jc = threadIdx.x / TPC, sub = threadIdx.x % TPC;
      const int jr = jc < LDP ? jc : LDP - 1;
      T g = S::zero(), gk = S::zero();
#pragma unroll
      for (int q = 0; q < (W + TPC - 1) / TPC; ++q) {
        const int w = sub + q * TPC;
        if (w < W) {
          g = S::add(g, pt[w * LDP + jr]);
          gk = S::add(gk, pt[w * LDP + k]);
        }
      }
#pragma unroll
      for (int off = 1; off < TPC; off <<= 1) {
        g = S::add(g, shfl_xor_t(g, off));
        gk = S::add(gk, shfl_xor_t(gk, off));
      }
      if (sub == 0 && jc >= k && jc <= r) {
        const T alpha = rk_s[k];
        const double nrm = sqrt(S::re(gk));
        const double aa = S::abs(alpha);
        T bt = S::zero();
        double tau = 0.0;
        if (nrm != 0.0) {
          bt = (aa == 0.0) ? S::from(-nrm, 0.0) : S::mulr(alpha, -nrm * rcp_nr(aa));
          tau = rcp_nr(nrm * (nrm + aa));  // 2 / (v^H v)
        }
        sj_s[jc] = (jc > k) ? S::mulr(S::sub(g, S::mul(S::conj(bt), rk_s[jc])), tau) : S::zero();
        if (jc == k) {
          rdiag[k] = bt;
          nrm_s[k] = nrm;
        }
      }
      __syncthreads();
      beta = rdiag[k];
#pragma unroll
      for (int v = VK; v < CB; ++v) {
        const int j = lb + CG * v;
        sj[v] = (j <= r && (v > VK || j > k)) ? sj_s[j] : S::zero();  // columns <= k keep their values
      }
    } else {
      const double gkk = S::re(pt[k]);
      const T alpha = rk_s[k];
      const double nrm = sqrt(gkk);
      const double aa = S::abs(alpha);
      double tau;
      if (nrm == 0.0) {
        beta = S::zero();
        tau = 0.0;
      } else {
        beta = (aa == 0.0) ? S::from(-nrm, 0.0) : S::mulr(alpha, -nrm * rcp_nr(aa));
        tau = rcp_nr(nrm * (nrm + aa));  // 2 / (v^H v)
      }
      if (threadIdx.x == 0) {
        rdiag[k] = beta;
        nrm_s[k] = nrm;
      }
#pragma unroll
      for (int v = VK; v < CB; ++v) {
        const int j = lb + CG * v;
        const T w = S::mulr(S::sub(pt[j], S::mul(S::conj(beta), rk_s[j])), tau);
        sj[v] = (v > VK || j > k) ? w : S::zero();  // columns <= k keep their values
      }
    }
    // v_i: x_i below the pivot, alpha - beta on it, 0 above
    const T vdiag = S::sub(rk_s[k], beta);
#pragma unroll
    for (int u = UK; u < RA; ++u) {
      const T vi = (u == UK && grg == gk) ? vdiag : xg[u];
#pragma unroll
      for (int v = VK; v < CB; ++v) A[u][v] = S::fms(vi, sj[v], A[u][v]);
    }
  }
};

template <typename T, int RG, int RA, int CB, int W, int VK>
struct LsqColumns {
  static __device__ __forceinline__ void run(T (&A)[RA][CB], int la, int lb, int grg, int warp, int r, T* rowb,
                                             T* part, T* sj_s, T* rdiag, double* nrm_s) {
    constexpr int CG = 32 / RG;
    constexpr int LDP = CG * CB;
    if (VK * CG >= r) return;
#pragma unroll 1
    for (int bk = 0; bk < CG; ++bk) {
      const int k = bk + CG * VK;
      if (k >= r) break;
      const int buf = k & 1;
      LsqStep<T, RG, RA, CB, W>::template run<VK>(A, k, bk, la, lb, grg, warp, r, rowb + buf * LDP,
                                                  part + (size_t)buf * W * LDP, sj_s, rdiag, nrm_s);
    }
    if constexpr (VK + 1 < CB)
      LsqColumns<T, RG, RA, CB, W, VK + 1>::run(A, la, lb, grg, warp, r, rowb, part, sj_s, rdiag, nrm_s);
  }
};

// Per-parameter outcome when M(p) has non-finite entries (linalg.py:36-37).
template <typename T>
__device__ __forceinline__ void lsq_nonfinite(const LsqArgs<T>& a, int64_t p) {
  using S = Sc<T>;
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  for (int j = threadIdx.x; j < a.r; j += blockDim.x) a.coef[p * a.r + j] = S::from(qnan, 0.0);
  if (threadIdx.x == 0) {
    a.status[p] = 2;
    a.sres[p] = qnan;
    if (a.badcol) a.badcol[p] = -1;
    if (a.outv) { a.outv[2 * p] = qnan; a.outv[2 * p + 1] = qnan; }
  }
  __syncthreads();
}

// After the factorisation (strict upper R and y = (Q^H t_w)[:r] in Rs, R_kk
// in rdiag, |R_kk| in nrm_s): rank test, back substitution, sampled residual
// and output value for parameter p.  All threads of the CTA call it.
template <typename T>
__device__ __forceinline__ void lsq_finish(const LsqArgs<T>& a, int64_t p, const T* Ms, int ldm, const T* Rs,
                                           T* cvec, const T* rdiag, const double* nrm_s, double* rinfo,
                                           double* red, int W) {
  using S = Sc<T>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = a.s, r = a.r;
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  if (warp == 0) {
    // rank test on |R_kk| (linalg.py:107-112): the first column of the minimum
    double mx = 0.0, mn = DBL_MAX;
    int am = 0x7fffffff;
    for (int j = lane; j < r; j += 32) {
      const double d = nrm_s[j];
      mx = fmax(mx, d);
      if (d < mn) { mn = d; am = j; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      const double pm = __shfl_xor_sync(0xffffffffu, mn, off);
      const int pa = __shfl_xor_sync(0xffffffffu, am, off);
      if (pm < mn || (pm == mn && pa < am)) { mn = pm; am = pa; }
    }
    if (lane == 0) {
      rinfo[0] = (r > 0 && mn < 1e-12 * fmax(mx, DBL_MIN)) ? 1.0 : 0.0;
      rinfo[1] = (double)(am == 0x7fffffff ? 0 : am);
    }
  }
  __syncthreads();
  const bool rankdef = rinfo[0] != 0.0;
  const int amin = (int)rinfo[1];
  if (warp == 0) {
    if (!rankdef) {
      // reciprocals of the diagonal in parallel, then a column sweep
      const T one = S::from(1.0, 0.0);
      const T rinv0 = (lane < r) ? S::div(one, rdiag[lane]) : S::zero();
      const T rinv1 = (lane + 32 < r) ? S::div(one, rdiag[lane + 32]) : S::zero();
      T y0 = (lane < r) ? Rs[lane * ldm + r] : S::zero();
      T y1 = (lane + 32 < r) ? Rs[(lane + 32) * ldm + r] : S::zero();
      for (int k = r - 1; k >= 0; --k) {
        const bool lo = k < 32;
        T ck = S::mul(lo ? y0 : y1, lo ? rinv0 : rinv1);
        ck = shfl_t(ck, k & 31);
        if (lane == 0) cvec[k] = ck;
        if (lane < k) y0 = S::fms(Rs[lane * ldm + k], ck, y0);
        if (lane + 32 < k) y1 = S::fms(Rs[(lane + 32) * ldm + k], ck, y1);
      }
    } else {
      for (int j = lane; j < r; j += 32) cvec[j] = S::from(qnan, 0.0);
    }
  }
  __syncthreads();
  // sampled residual ||w (M c - t)|| from the unweighted M (online.py:121-124)
  double ss = 0.0;
  for (int i = threadIdx.x; i < s; i += blockDim.x) {
    // four interleaved partial sums (j mod 4), combined in a fixed order: the
    // row loads (from L2 when M is parked) overlap instead of one chain
    T a4[4] = {S::zero(), S::zero(), S::zero(), S::zero()};
    const T* mrow = Ms + i * ldm;
    int j = 0;
    for (; j + 4 <= r; j += 4) {
#pragma unroll
      for (int t = 0; t < 4; ++t) a4[t] = S::add(a4[t], S::mul(mrow[j + t], cvec[j + t]));
    }
#pragma unroll
    for (int t = 0; t < 3; ++t)
      if (j + t < r) a4[t] = S::add(a4[t], S::mul(mrow[j + t], cvec[j + t]));
    const T acc = S::add(S::add(a4[0], a4[1]), S::add(a4[2], a4[3]));
    T res = S::sub(acc, Ms[i * ldm + r]);
    if (a.w) res = S::mulr(res, a.w[i]);
    ss += S::abs2(res);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
  if (lane == 0) red[warp] = ss;
  for (int j = threadIdx.x; j < r; j += blockDim.x) a.coef[p * r + j] = cvec[j];
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < W; ++w) tot += red[w];
    a.sres[p] = rankdef ? qnan : sqrt(tot);
    a.status[p] = rankdef ? 1 : 0;
    if (a.badcol) a.badcol[p] = rankdef ? amin : -1;
    if (a.outv) {
      T o = S::zero();
      if (a.proj)
        for (int j = 0; j < r; ++j) o = S::add(o, S::mul(a.proj[j], cvec[j]));
      a.outv[2 * p] = S::re(o);
      a.outv[2 * p + 1] = S::im(o);
    }
  }
  __syncthreads();
}

template <typename T, int RG, int RA, int CB, int W, class Asm>
__global__ void __launch_bounds__(32 * W) k_lsq_mw(LsqArgs<T> a, Asm as, size_t scratch_bytes) {
  using S = Sc<T>;
  constexpr int CG = 32 / RG;
  constexpr int LDP = CG * CB;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = a.s, r = a.r, ldm = r + 1;
  const int la = lane % RG, lb = lane / RG;
  const int grg = warp * RG + la;  // global row group
  constexpr int nrg = W * RG;
  T* Ms = reinterpret_cast<T*>(smem_raw);
  T* Rs = Ms + (size_t)s * ldm;
  T* cvec = Rs + (size_t)r * ldm;
  T* rdiag = cvec + r;                // R_kk (beta) per column
  T* rowb = rdiag + r;                // 2 x LDP
  T* part = rowb + 2 * LDP;           // 2 x W x LDP
  T* sj_s = part + 2 * W * LDP;       // LDP reflector weights w_j
  const size_t core =
      ((size_t)s * ldm + (size_t)r * ldm + 2 * (size_t)r + 2 * ((size_t)LDP + (size_t)W * LDP) + LDP) * sizeof(T);
  double* red = reinterpret_cast<double*>(smem_raw + (core + 15) / 16 * 16);  // W residual partials (<= 16)
  double* nrm_s = red + 16;                                                    // |R_kk|
  double* rinfo = nrm_s + 64;                                                  // rank deficient, column
  unsigned char* scratch = smem_raw + (core + 15) / 16 * 16 + kLsqRedDoubles * sizeof(double);
  (void)scratch_bytes;
  const CtaGroup grp;

  for (int64_t p = blockIdx.x; p < a.P; p += gridDim.x) {
    as(grp, p, Ms, ldm, s, r, scratch);
    for (int i = threadIdx.x; i < s; i += blockDim.x) Ms[i * ldm + r] = a.t[p * a.t_stride + i];
    __syncthreads();

    T A[RA][CB];
    bool bad = false;
#pragma unroll
    for (int u = 0; u < RA; ++u) {
      const int i = grg + nrg * u;
      const double wi = (i < s && a.w) ? a.w[i] : 1.0;
#pragma unroll
      for (int v = 0; v < CB; ++v) {
        const int j = lb + CG * v;
        if (i < s && j <= r) {
          const T m = Ms[i * ldm + j];
          if (j < r && !S::finite(m)) bad = true;
          A[u][v] = a.w ? S::mulr(m, wi) : m;
        } else {
          A[u][v] = S::zero();
        }
      }
    }
    if (__syncthreads_or(bad)) {
      lsq_nonfinite<T>(a, p);
      continue;
    }

    LsqColumns<T, RG, RA, CB, W, 0>::run(A, la, lb, grg, warp, r, rowb, part, sj_s, rdiag, nrm_s);

    // R (strict upper part from registers, diagonal = beta) and y to shared memory
#pragma unroll
    for (int u = 0; u < RA; ++u) {
      const int i = grg + nrg * u;
#pragma unroll
      for (int v = 0; v < CB; ++v) {
        const int j = lb + CG * v;
        if (i < r && j > i && j <= r) Rs[i * ldm + j] = A[u][v];
      }
    }
    lsq_finish<T>(a, p, Ms, ldm, Rs, cvec, rdiag, nrm_s, rinfo, red, W);
  }
}
