// K4m: batched weighted least squares, W warps cooperating on one parameter
// value, for matrices too large for one warp's registers (configs 3, 4, 5:
// 160x41, 120x9 complex, 200x51).  Same contract as k_lsq / k_lsq_warp
// (linalg.solve_ls, linalg.py:89-113, called from online.py:105-134).
//
// Layout: lane = a + RG*b (a < RG row groups, b < CG = 32/RG column groups).
// Global row group of a lane = w*RG + a (w = warp), so row i belongs to
// (row group i mod (W*RG), slot u = i / (W*RG)); column j to (b = j mod CG,
// slot v = j / CG).  Registers A[RA][CB].
//
// Householder step k (Gram-row formulation):
//   x_i = M_ik for own rows           <- shuffle inside the warp (column group k mod CG)
//   partial g_j over own rows, butterfly over the RG row groups of the warp
//   warp partials and row k go to shared memory (double-buffered), ONE
//   __syncthreads, every thread sums the W partials of its columns in warp
//   order (deterministic), forms beta/tau and updates its rows.
#pragma once
#include "k_lsq_warp.cuh"

template <typename T>
__host__ __device__ inline size_t lsq_mw_smem_bytes(int s, int r, int W, size_t scratch) {
  const int ldm = r + 1;
  // Ms (s x ldm), R/y (r x ldm), c (r), 2 x [row k (ldm) + partials (W x ldm)]
  size_t n = (size_t)s * ldm + (size_t)r * ldm + r + 2 * ((size_t)ldm + (size_t)W * ldm);
  size_t bytes = (n * sizeof(T) + 15) / 16 * 16;
  return bytes + 128 + (scratch + 15) / 16 * 16;
}

template <typename T, int RG, int RA, int CB, class Asm>
__global__ void __launch_bounds__(256) k_lsq_mw(LsqArgs<T> a, Asm as, size_t scratch_bytes) {
  using S = Sc<T>;
  constexpr int CG = 32 / RG;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int W = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = a.s, r = a.r, ldm = r + 1;
  const int la = lane % RG, lb = lane / RG;
  const int grg = warp * RG + la;  // global row group
  const int NRG = W * RG;
  T* Ms = reinterpret_cast<T*>(smem_raw);
  T* Rs = Ms + (size_t)s * ldm;
  T* cvec = Rs + (size_t)r * ldm;
  T* rowb = cvec + r;                 // 2 x ldm
  T* part = rowb + 2 * ldm;           // 2 x W x ldm
  const size_t core = ((size_t)s * ldm + (size_t)r * ldm + r + 2 * ((size_t)ldm + (size_t)W * ldm)) * sizeof(T);
  double* red = reinterpret_cast<double*>(smem_raw + (core + 15) / 16 * 16);  // W doubles (<= 8)
  unsigned char* scratch = smem_raw + (core + 15) / 16 * 16 + 64 * 2;
  (void)scratch_bytes;
  const CtaGroup grp;
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);

  for (int64_t p = blockIdx.x; p < a.P; p += gridDim.x) {
    as(grp, p, Ms, ldm, s, r, scratch);
    for (int i = threadIdx.x; i < s; i += blockDim.x) Ms[i * ldm + r] = a.t[p * a.t_stride + i];
    __syncthreads();

    T A[RA][CB];
    bool bad = false;
#pragma unroll
    for (int u = 0; u < RA; ++u) {
      const int i = grg + NRG * u;
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
      for (int j = threadIdx.x; j < r; j += blockDim.x) a.coef[p * r + j] = S::from(qnan, 0.0);
      if (threadIdx.x == 0) {
        a.status[p] = 2;
        a.sres[p] = qnan;
        if (a.badcol) a.badcol[p] = -1;
        if (a.outv) { a.outv[2 * p] = qnan; a.outv[2 * p + 1] = qnan; }
      }
      __syncthreads();
      continue;
    }

    double dmax = 0.0, dmin = DBL_MAX;
    int amin = 0;
    for (int k = 0; k < r; ++k) {
      const int buf = k & 1;
      T* rk_s = rowb + buf * ldm;
      T* pt = part + (size_t)buf * W * ldm;
      const int bk = k % CG, vk = k / CG;
      const int gk = k % NRG, uk = k / NRG;
      // x_i = M_ik for own rows (column group bk of this warp, slot vk)
      T x[RA];
#pragma unroll
      for (int u = 0; u < RA; ++u) {
        T mine = A[u][0];
#pragma unroll
        for (int v = 1; v < CB; ++v)
          if (v == vk) mine = A[u][v];
        x[u] = shfl_t(mine, la + RG * bk);
      }
      // the owner of row k publishes it (columns >= k)
      if (grg == gk) {
#pragma unroll
        for (int u = 0; u < RA; ++u)
          if (u == uk) {
#pragma unroll
            for (int v = 0; v < CB; ++v) {
              const int j = lb + CG * v;
              if (j >= k && j <= r) rk_s[j] = A[u][v];
            }
          }
      }
      // partial Gram row: own rows, butterfly over the warp's row groups
#pragma unroll
      for (int v = 0; v < CB; ++v) {
        T acc = S::zero();
#pragma unroll
        for (int u = 0; u < RA; ++u) {
          const int i = grg + NRG * u;
          if (i >= k && i < s) acc = S::fma_conj(x[u], A[u][v], acc);
        }
#pragma unroll
        for (int off = 1; off < RG; off <<= 1) acc = S::add(acc, shfl_xor_t(acc, off));
        const int j = lb + CG * v;
        if (la == 0 && j >= k && j <= r) pt[warp * ldm + j] = acc;
      }
      __syncthreads();
      double gkk = 0.0;
      for (int w = 0; w < W; ++w) gkk += S::re(pt[w * ldm + k]);
      const T alpha = rk_s[k];
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
        const int j = lb + CG * v;
        sj[v] = S::zero();
        if (j > k && j <= r) {
          T g = S::zero();
          for (int w = 0; w < W; ++w) g = S::add(g, pt[w * ldm + j]);
          sj[v] = S::mulr(S::sub(g, S::mul(S::conj(beta), rk_s[j])), tau);
        }
      }
      const T vdiag = S::sub(alpha, beta);
#pragma unroll
      for (int u = 0; u < RA; ++u) {
        const int i = grg + NRG * u;
        if (i >= k && i < s) {
          const T vi = (i == k) ? vdiag : x[u];
#pragma unroll
          for (int v = 0; v < CB; ++v) {
            const int j = lb + CG * v;
            if (j > k && j <= r) A[u][v] = S::fms(vi, sj[v], A[u][v]);
            else if (j == k && i == k) A[u][v] = beta;
          }
        }
      }
    }

    // R and y to shared memory, back substitution by warp 0
#pragma unroll
    for (int u = 0; u < RA; ++u) {
      const int i = grg + NRG * u;
#pragma unroll
      for (int v = 0; v < CB; ++v) {
        const int j = lb + CG * v;
        if (i < r && j >= i && j <= r) Rs[i * ldm + j] = A[u][v];
      }
    }
    __syncthreads();
    const bool rankdef = (r > 0) && (dmin < 1e-12 * fmax(dmax, DBL_MIN));
    if (warp == 0) {
      if (!rankdef) {
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
    }
    __syncthreads();
    double ss = 0.0;
    for (int i = threadIdx.x; i < s; i += blockDim.x) {
      T acc = S::zero();
      for (int j = 0; j < r; ++j) acc = S::add(acc, S::mul(Ms[i * ldm + j], cvec[j]));
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
}
