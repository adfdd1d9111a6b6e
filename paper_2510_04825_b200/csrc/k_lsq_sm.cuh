// K4, shared-memory-resident Householder QR for the large shapes (configs 3,
// 4 and 5).  Same algorithm and outputs as k_lsq_mw / k_lsq_cw (Householder QR
// of [W M | W t], reference linalg.py:89-113 via online.py:105-134):
//
//   M_w = diag(w) M, t_w = diag(w) t                      (linalg.py:102-105)
//   H_k = I - tau_k v_k v_k^H, beta_k = -e^{i arg x_k} |x|, tau_k = 1/(|x|(|x| + |x_k|))
//   rank test min|R_kk| < 1e-12 max|R_kk|, c = R^{-1} y   (linalg.py:107-113)
//   sampled residual ||w (M c - t)|| from the unweighted M (online.py:121-124)
//
// Why shared memory: the register-resident kernels hold [M_w | t_w] in the
// registers of the warps that factor it, which caps the parameter values in
// flight at two per SM for 200 x 51 (20.4 K registers each) and leaves every
// Householder step a latency chain on 3 warps per SMSP (~2.5 K cycles per
// step, profiles/r01_k4_lsq_cw_config5_ncu.json).  Here the augmented matrix
// lives column-major in shared memory (one CTA per parameter value, two CTAs
// per SM at 200 x 51, four at 160 x 41), so a CTA can run 12-16 warps that
// share each step's columns:
//
//   warp 0        column k+1: dot, update, then forms reflector k+1 from it
//                 (look-ahead) and publishes tau, the head of v and R_kk;
//   warps 1..W-1  columns k+2 .. r round robin, two at a time: each lane holds
//                 rows lane + 32u (u < RA) of the column in registers, the dot
//                 with v is one butterfly over the warp, the rank-1 update is
//                 in registers, rows >= k go back to shared memory;
//   one __syncthreads per step.
//
// v_k is column k itself below the diagonal (left in place by step k-1) with
// its head alpha - beta kept in shared memory; R ends up in the upper
// triangle of the column-major matrix, y = (Q^H t_w)[:r] in column r.  The
// unweighted M | t is copied to this CTA's L2 slot for the explicit residual.
// All reductions run in a fixed order (results do not depend on the batch).
#pragma once
#include "k_lsq_cw.cuh"

template <typename T>
__device__ __forceinline__ T warp_allreduce(T v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = Sc<T>::add(v, shfl_xor_t(v, off));
  return v;
}
__device__ __forceinline__ double warp_allreduce_d(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

struct SmShared {
  void* vk;        // 2 x T: head of v (alpha - beta), double-buffered by step parity
  double* tau;     // 2
  void* rdiag;     // r x T: R_kk = beta_k
  double* nrm;     // r: |R_kk|
};

// Reflector kk from the column values y (rows >= kk count; rows < kk ignored).
template <typename T, int RA>
__device__ __forceinline__ void sm_reflector(const T (&y)[RA], int kk, int s, int lane, const SmShared& sh) {
  using S = Sc<T>;
  double ss = 0.0;
#pragma unroll
  for (int u = 0; u < RA; ++u) {
    const int i = lane + 32 * u;
    ss += (i >= kk) ? S::abs2(y[u]) : 0.0;   // rows >= s are zero padding
  }
  ss = warp_allreduce_d(ss);
  T al = S::zero();
#pragma unroll
  for (int u = 0; u < RA; ++u)
    if (u == (kk >> 5)) al = y[u];
  const T alpha = shfl_t(al, kk & 31);
  const double nrm = sqrt(ss);
  const double aa = S::abs(alpha);
  T beta = S::zero();
  double tau = 0.0;
  if (nrm != 0.0) {
    if constexpr (std::is_same<T, double>::value) {
      beta = (aa == 0.0) ? -nrm : copysign(nrm, -alpha);   // -sign(x_k) |x|
    } else {
      beta = (aa == 0.0) ? S::from(-nrm, 0.0) : S::mulr(alpha, -nrm / aa);   // -e^{i arg x_k} |x|
    }
    tau = rcp_nr(nrm * (nrm + aa));
  }
  if (lane == 0) {
    const int buf = kk & 1;
    reinterpret_cast<T*>(sh.vk)[buf] = S::sub(alpha, beta);
    sh.tau[buf] = tau;
    reinterpret_cast<T*>(sh.rdiag)[kk] = beta;
    sh.nrm[kk] = nrm;
  }
}

// Apply reflector k (v, tau) to NC columns held in registers.  v is zero on
// rows < k and on the padding rows >= s, so every slot takes part without a
// per-row test: those rows contribute 0 to the dot and are left unchanged.
template <typename T, int RA, int NC>
__device__ __forceinline__ void sm_apply(T (&y)[NC][RA], const T (&v)[RA], double tau) {
  using S = Sc<T>;
  T d[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) d[c] = S::zero();
#pragma unroll
  for (int u = 0; u < RA; ++u) {
#pragma unroll
    for (int c = 0; c < NC; ++c) d[c] = S::fma_conj(v[u], y[c][u], d[c]);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int c = 0; c < NC; ++c) d[c] = S::add(d[c], shfl_xor_t(d[c], off));
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const T w = S::mulr(d[c], tau);
#pragma unroll
    for (int u = 0; u < RA; ++u) y[c][u] = S::fms(v[u], w, y[c][u]);
  }
}

// columns are padded to 32 RA rows (zeros below s): plain loads and stores
template <typename T, int RA>
__device__ __forceinline__ void sm_load_col(T (&y)[RA], const T* col, int lane) {
#pragma unroll
  for (int u = 0; u < RA; ++u) y[u] = col[lane + 32 * u];
}
template <typename T, int RA>
__device__ __forceinline__ void sm_store_col(const T (&y)[RA], T* col, int lane) {
#pragma unroll
  for (int u = 0; u < RA; ++u) col[lane + 32 * u] = y[u];
}

// column stride: 32 RA rows (zero padding below s), odd so that the
// assembler's row-major walk writes conflict-free into the column-major matrix
__host__ __device__ inline int lsq_sm_lda(int RA) { return 32 * RA + 1; }

template <typename T>
__host__ __device__ inline size_t lsq_sm_smem_bytes(int RA, int r, size_t scratch) {
  const size_t n = (size_t)lsq_sm_lda(RA) * (r + 1) + 2 * (size_t)r + 2;  // A, c, R_kk, v heads
  size_t bytes = (n * sizeof(T) + 15) / 16 * 16;
  bytes += (2 + 64 + 32 + 2) * sizeof(double);                            // tau, |R_kk|, partials, rank info
  return bytes + (scratch + 15) / 16 * 16;
}

// Rank test, back substitution, sampled residual and output value from the
// column-major factorisation (R_ij = A[j lda + i], i < j; y_i = A[r lda + i])
// and the unweighted column-major M | t in mg (column stride ldg).
template <typename T>
__device__ __forceinline__ void sm_finish(const LsqArgs<T>& a, int64_t p, const T* A, int lda, const T* mg,
                                          T* cvec, const T* rdiag, const double* nrm_s, double* rinfo,
                                          double* red, int ldg) {
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
    const bool rankdef = r > 0 && mn < 1e-12 * fmax(mx, DBL_MIN);
    if (lane == 0) {
      rinfo[0] = rankdef ? 1.0 : 0.0;
      rinfo[1] = (double)(am == 0x7fffffff ? 0 : am);
    }
    if (!rankdef) {
      // reciprocals of the diagonal in parallel, then a column sweep (R column k
      // is contiguous: lane i reads R_ik)
      const T one = S::from(1.0, 0.0);
      const T rinv0 = (lane < r) ? S::div(one, rdiag[lane]) : S::zero();
      const T rinv1 = (lane + 32 < r) ? S::div(one, rdiag[lane + 32]) : S::zero();
      T y0 = (lane < r) ? A[(size_t)r * lda + lane] : S::zero();
      T y1 = (lane + 32 < r) ? A[(size_t)r * lda + lane + 32] : S::zero();
      for (int k = r - 1; k >= 0; --k) {
        const bool lo = k < 32;
        T ck = S::mul(lo ? y0 : y1, lo ? rinv0 : rinv1);
        ck = shfl_t(ck, k & 31);
        if (lane == 0) cvec[k] = ck;
        const T* rk = A + (size_t)k * lda;
        if (lane < k) y0 = S::fms(rk[lane], ck, y0);
        if (lane + 32 < k) y1 = S::fms(rk[lane + 32], ck, y1);
      }
    } else {
      for (int j = lane; j < r; j += 32) cvec[j] = S::from(qnan, 0.0);
    }
  }
  __syncthreads();
  const bool rankdef = rinfo[0] != 0.0;
  // sampled residual ||w (M c - t)|| from the unweighted M (online.py:121-124):
  // one row per thread, coalesced column-major loads from the L2 slot
  double ss = 0.0;
  for (int i = threadIdx.x; i < s; i += blockDim.x) {
    T a4[4] = {S::zero(), S::zero(), S::zero(), S::zero()};
    int j = 0;
    for (; j + 4 <= r; j += 4) {
#pragma unroll
      for (int t = 0; t < 4; ++t) a4[t] = S::add(a4[t], S::mul(mg[(size_t)(j + t) * ldg + i], cvec[j + t]));
    }
#pragma unroll
    for (int t = 0; t < 3; ++t)
      if (j + t < r) a4[t] = S::add(a4[t], S::mul(mg[(size_t)(j + t) * ldg + i], cvec[j + t]));
    const T acc = S::add(S::add(a4[0], a4[1]), S::add(a4[2], a4[3]));
    T res = S::sub(acc, mg[(size_t)r * ldg + i]);
    if (a.w) res = S::mulr(res, a.w[i]);
    ss += S::abs2(res);
  }
  ss = warp_allreduce_d(ss);
  if (lane == 0) red[warp] = ss;
  for (int j = threadIdx.x; j < r; j += blockDim.x) a.coef[p * r + j] = cvec[j];
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
    a.sres[p] = rankdef ? qnan : sqrt(tot);
    a.status[p] = rankdef ? 1 : 0;
    if (a.badcol) a.badcol[p] = rankdef ? (int)rinfo[1] : -1;
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

// One CTA per parameter value (persistent over p), W warps, s <= 32 RA rows.
template <typename T, int RA, int W, class Asm, int MINB>
__global__ void __launch_bounds__(32 * W, MINB) k_lsq_sm(LsqArgs<T> a, Asm as, T* __restrict__ mglob) {
  using S = Sc<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = a.s, r = a.r, n = r + 1, lda = lsq_sm_lda(RA);
  T* A = reinterpret_cast<T*>(smem_raw);
  T* cvec = A + (size_t)lda * n;
  T* rdiag = cvec + r;
  T* vk_s = rdiag + r;
  const size_t tb = (((size_t)lda * n + 2 * (size_t)r + 2) * sizeof(T) + 15) / 16 * 16;
  double* tau_s = reinterpret_cast<double*>(smem_raw + tb);
  double* nrm_s = tau_s + 2;
  double* red = nrm_s + 64;
  double* rinfo = red + 32;
  unsigned char* scratch = smem_raw + tb + (2 + 64 + 32 + 2) * sizeof(double);
  SmShared sh{vk_s, tau_s, rdiag, nrm_s};
  T* mg = mglob + (size_t)blockIdx.x * s * n;
  const CtaGroup grp;
  for (int idx = threadIdx.x; idx < lda * n; idx += blockDim.x) A[idx] = S::zero();  // rows >= s stay zero
  __syncthreads();
#ifdef SAS_SM_PROF
  long long tp[4] = {0, 0, 0, 0}, t0 = clock64(), t1;
#define SM_PROF_MARK(ph) do { t1 = clock64(); tp[ph] += t1 - t0; t0 = t1; } while (0)
#else
#define SM_PROF_MARK(ph) do {} while (0)
#endif

  for (int64_t p = blockIdx.x; p < a.P; p += gridDim.x) {
    as(grp, p, A, 1, s, r, scratch, lda);   // column-major: entry (i, j) at A[i + j lda]
    for (int i = threadIdx.x; i < s; i += blockDim.x) A[(size_t)r * lda + i] = a.t[p * a.t_stride + i];
    __syncthreads();
    SM_PROF_MARK(0);
    // unweighted M | t to the L2 slot (residual), weights in place, non-finite test (linalg.py:36-37)
    bool bad = false;
    for (int j = warp; j < n; j += W) {
      T* col = A + (size_t)j * lda;
      T* gcol = mg + (size_t)j * s;
      for (int i = lane; i < s; i += 32) {
        const T m = col[i];
        gcol[i] = m;
        if (j < r && !S::finite(m)) bad = true;
        if (a.w) col[i] = S::mulr(m, a.w[i]);
      }
    }
    if (__syncthreads_or(bad)) {
      lsq_nonfinite<T>(a, p);
      continue;
    }
    SM_PROF_MARK(1);
    if (warp == 0) {
      T y[RA];
      sm_load_col<T, RA>(y, A, lane);
      sm_reflector<T, RA>(y, 0, s, lane, sh);
    }
    __syncthreads();
    for (int k = 0; k < r; ++k) {
      const int buf = k & 1;
      const double tau = tau_s[buf];
      const T vhead = vk_s[buf];
      const T* colk = A + (size_t)k * lda;
      T v[RA];
#pragma unroll
      for (int u = 0; u < RA; ++u) {
        const int i = lane + 32 * u;
        const T x = colk[i];
        v[u] = (i > k) ? x : (i == k ? vhead : S::zero());
      }
      if (warp == 0) {
        // column k+1 first, then reflector k+1 from it (look-ahead)
        T y[1][RA];
        T* col = A + (size_t)(k + 1) * lda;
        sm_load_col<T, RA>(y[0], col, lane);
        sm_apply<T, RA, 1>(y, v, tau);
        sm_store_col<T, RA>(y[0], col, lane);
        if (k + 1 < r) sm_reflector<T, RA>(y[0], k + 1, s, lane, sh);
      } else {
        int j = k + 1 + warp;
        for (; j + (W - 1) <= r; j += 2 * (W - 1)) {
          T y[2][RA];
          T* c0 = A + (size_t)j * lda;
          T* c1 = A + (size_t)(j + W - 1) * lda;
          sm_load_col<T, RA>(y[0], c0, lane);
          sm_load_col<T, RA>(y[1], c1, lane);
          sm_apply<T, RA, 2>(y, v, tau);
          sm_store_col<T, RA>(y[0], c0, lane);
          sm_store_col<T, RA>(y[1], c1, lane);
        }
        if (j <= r) {
          T y[1][RA];
          T* c0 = A + (size_t)j * lda;
          sm_load_col<T, RA>(y[0], c0, lane);
          sm_apply<T, RA, 1>(y, v, tau);
          sm_store_col<T, RA>(y[0], c0, lane);
        }
      }
      __syncthreads();
    }
    SM_PROF_MARK(2);
    sm_finish<T>(a, p, A, lda, mg, cvec, rdiag, nrm_s, rinfo, red, s);
    SM_PROF_MARK(3);
  }
#ifdef SAS_SM_PROF
  if (threadIdx.x == 0 && blockIdx.x < 4)
    printf("sm_prof block %d: assemble %lld copy/weights %lld qr %lld finish %lld cycles (all p of the CTA)\n",
           blockIdx.x, tp[0], tp[1], tp[2], tp[3]);
#endif
}
