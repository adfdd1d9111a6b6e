// K4w: batched weighted least squares with ONE WARP per parameter value, for
// problems whose augmented matrix [M_w | t_w] fits in a warp's registers
// (s <= 8*RA rows, r+1 <= 4*CB columns).  Same contract and arithmetic steps as
// k_lsq (linalg.solve_ls, linalg.py:89-113, called from online.py:105-134);
// the difference is the data layout, chosen so that no __syncthreads is needed
// and many parameter values are in flight per SM:
//
//   lane = a + 8 b  (a = row group 0..7, b = column group 0..3)
//   lane (a, b) holds rows {a + 8u} x columns {b + 4v} in registers A[u][v].
//
// Householder step k (the Gram-row formulation of k_lsq):
//   x_i = M_ik for the lane's rows      <- shuffle from lane (a, k mod 4)
//   partial g_j = sum_i conj(x_i) M_ij  (own rows, own columns)
//   g_j summed over the 8 row groups    <- xor-shuffle butterfly (1, 2, 4), every
//                                          lane ends with the totals of its columns
//   |x| = sqrt(g_kk), alpha = M_kk, row k values M_kj   <- shuffles
//   w_j = g_j - conj(beta) M_kj, M_ij -= tau v_i w_j
// The butterfly adds in a fixed order, so results are deterministic.
#pragma once
#include "k_lsq.cuh"

template <typename T>
__host__ __device__ inline size_t lsq_warp_smem_per_warp(int s, int r, size_t scratch) {
  const int ldm = r + 1;
  size_t n = (size_t)s * ldm + (size_t)r * ldm + r;
  size_t bytes = n * sizeof(T);
  bytes = (bytes + 15) / 16 * 16;
  return bytes + (scratch + 15) / 16 * 16;
}

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

template <typename T, int RA, int CB, class Asm>
__global__ void __launch_bounds__(128) k_lsq_warp(LsqArgs<T> a, Asm as, size_t scratch_bytes) {
  using S = Sc<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  const int s = a.s, r = a.r, ldm = r + 1;
  const int la = lane & 7, lb = lane >> 3;
  const size_t per_warp = lsq_warp_smem_per_warp<T>(s, r, scratch_bytes);
  unsigned char* base = smem_raw + wib * per_warp;
  T* Ms = reinterpret_cast<T*>(base);
  T* Rs = Ms + (size_t)s * ldm;
  T* cvec = Rs + (size_t)r * ldm;
  unsigned char* scratch = base + ((((size_t)s * ldm + (size_t)r * ldm + r) * sizeof(T) + 15) / 16 * 16);
  const WarpGroup grp;
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);

  for (int64_t p = (int64_t)blockIdx.x * nw + wib; p < a.P; p += (int64_t)gridDim.x * nw) {
    as(grp, p, Ms, ldm, s, r, scratch);
    for (int i = lane; i < s; i += 32) Ms[i * ldm + r] = a.t[p * a.t_stride + i];
    __syncwarp();

    T A[RA][CB];
    bool bad = false;
#pragma unroll
    for (int u = 0; u < RA; ++u) {
      const int i = la + 8 * u;
      const double wi = (i < s && a.w) ? a.w[i] : 1.0;
#pragma unroll
      for (int v = 0; v < CB; ++v) {
        const int j = lb + 4 * v;
        if (i < s && j <= r) {
          const T m = Ms[i * ldm + j];
          if (j < r && !S::finite(m)) bad = true;
          A[u][v] = a.w ? S::mulr(m, wi) : m;
        } else {
          A[u][v] = S::zero();
        }
      }
    }
    if (__any_sync(0xffffffffu, bad)) {
      for (int j = lane; j < r; j += 32) a.coef[p * r + j] = S::from(qnan, 0.0);
      if (lane == 0) {
        a.status[p] = 2;
        a.sres[p] = qnan;
        if (a.badcol) a.badcol[p] = -1;
        if (a.outv) { a.outv[2 * p] = qnan; a.outv[2 * p + 1] = qnan; }
      }
      __syncwarp();
      continue;
    }

    double dmax = 0.0, dmin = DBL_MAX;
    int amin = 0;
    for (int k = 0; k < r; ++k) {
      const int ak = k & 7, uk = k >> 3, bk = k & 3, vk = k >> 2;
      // x_i = M_ik for this lane's rows: column k lives in column group bk, slot vk
      T x[RA];
#pragma unroll
      for (int u = 0; u < RA; ++u) {
        T mine = A[u][0];
#pragma unroll
        for (int v = 1; v < CB; ++v)
          if (v == vk) mine = A[u][v];
        x[u] = shfl_t(mine, la + 8 * bk);
      }
      // row k of this lane's columns (row group ak, slot uk)
      T rk[CB];
#pragma unroll
      for (int v = 0; v < CB; ++v) {
        T mine = A[0][v];
#pragma unroll
        for (int u = 1; u < RA; ++u)
          if (u == uk) mine = A[u][v];
        rk[v] = shfl_t(mine, ak + 8 * lb);
      }
      // partial Gram row over own rows i >= k, then butterfly over row groups
      T gj[CB];
#pragma unroll
      for (int v = 0; v < CB; ++v) {
        T acc = S::zero();
#pragma unroll
        for (int u = 0; u < RA; ++u) {
          const int i = la + 8 * u;
          if (i >= k && i < s) acc = S::fma_conj(x[u], A[u][v], acc);
        }
        acc = S::add(acc, shfl_xor_t(acc, 1));
        acc = S::add(acc, shfl_xor_t(acc, 2));
        acc = S::add(acc, shfl_xor_t(acc, 4));
        gj[v] = acc;
      }
      // g_kk and alpha = M_kk from column group bk
      T gsel = gj[0], asel = rk[0];
#pragma unroll
      for (int v = 1; v < CB; ++v)
        if (v == vk) { gsel = gj[v]; asel = rk[v]; }
      const double gkk = S::re(shfl_t(gsel, 8 * bk));
      const T alpha = shfl_t(asel, 8 * bk);
      const double nrm = sqrt(gkk);
      const double aa = S::abs(alpha);
      T beta;
      double tau;
      if (nrm == 0.0) {
        beta = S::zero();
        tau = 0.0;
      } else {
        beta = (aa == 0.0) ? S::from(-nrm, 0.0) : S::mulr(alpha, -nrm / aa);
        tau = 1.0 / (nrm * (nrm + aa));  // 2 / (v^H v)
      }
      dmax = fmax(dmax, nrm);
      if (nrm < dmin) { dmin = nrm; amin = k; }
      T sj[CB];
#pragma unroll
      for (int v = 0; v < CB; ++v) {
        const int j = lb + 4 * v;
        sj[v] = (j > k && j <= r) ? S::mulr(S::sub(gj[v], S::mul(S::conj(beta), rk[v])), tau) : S::zero();
      }
      const T vk_diag = S::sub(alpha, beta);
#pragma unroll
      for (int u = 0; u < RA; ++u) {
        const int i = la + 8 * u;
        if (i >= k && i < s) {
          const T vi = (i == k) ? vk_diag : x[u];
#pragma unroll
          for (int v = 0; v < CB; ++v) {
            const int j = lb + 4 * v;
            if (j > k && j <= r) A[u][v] = S::fms(vi, sj[v], A[u][v]);
            else if (j == k && i == k) A[u][v] = beta;
          }
        }
      }
    }

    // R (upper r x r) and y = (Q^H t_w)[:r] to shared memory
#pragma unroll
    for (int u = 0; u < RA; ++u) {
      const int i = la + 8 * u;
#pragma unroll
      for (int v = 0; v < CB; ++v) {
        const int j = lb + 4 * v;
        if (i < r && j >= i && j <= r) Rs[i * ldm + j] = A[u][v];
      }
    }
    __syncwarp();
    const bool rankdef = (r > 0) && (dmin < 1e-12 * fmax(dmax, DBL_MIN));
    if (!rankdef) {
      // column-oriented back substitution, lane i holds y_i (r <= 63 -> 2 slots)
      T y0 = (lane < r) ? Rs[lane * ldm + r] : S::zero();
      T y1 = (lane + 32 < r) ? Rs[(lane + 32) * ldm + r] : S::zero();
      for (int k = r - 1; k >= 0; --k) {
        const T yk = shfl_t(k < 32 ? y0 : y1, k & 31);
        const T ck = S::div(yk, Rs[k * ldm + k]);
        if (lane == 0) cvec[k] = ck;
        if (lane < k) y0 = S::fms(Rs[lane * ldm + k], ck, y0);
        if (lane + 32 < k) y1 = S::fms(Rs[(lane + 32) * ldm + k], ck, y1);
      }
    } else {
      for (int j = lane; j < r; j += 32) cvec[j] = S::from(qnan, 0.0);
    }
    __syncwarp();
    // sampled residual ||w (M c - t)|| from the unweighted M (online.py:121-124)
    double ss = 0.0;
    for (int i = lane; i < s; i += 32) {
      T acc = S::zero();
      for (int j = 0; j < r; ++j) acc = S::add(acc, S::mul(Ms[i * ldm + j], cvec[j]));
      T res = S::sub(acc, Ms[i * ldm + r]);
      if (a.w) res = S::mulr(res, a.w[i]);
      ss += S::abs2(res);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    for (int j = lane; j < r; j += 32) a.coef[p * r + j] = cvec[j];
    if (lane == 0) {
      a.sres[p] = rankdef ? qnan : sqrt(ss);
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
    __syncwarp();
  }
}
