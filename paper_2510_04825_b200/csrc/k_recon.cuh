// K5/K6: reconstruction x = X c (OnlineSolution.lift, online.py:50-54) and the
// full-residual checker ||A(p) x - b|| / max(||b||, 1e-300) (cli.py:285, 344-351)
// evaluated without materialising x: each thread recomputes the x entries of a
// row's stencil neighbourhood from X and c.
#pragma once
#include "sas_common.cuh"

constexpr int kLiftPT = 8;  // parameter values per CTA

// grid = (ceil(n/256), ceil(P/kLiftPT)); block 256
template <typename T>
__global__ void __launch_bounds__(256) k_lift(const T* __restrict__ X, int64_t n, int r,
                                              const T* __restrict__ coef, int64_t P,
                                              T* __restrict__ x) {
  using S = Sc<T>;
  __shared__ T cs[kLiftPT][64];
  const int64_t p0 = (int64_t)blockIdx.y * kLiftPT;
  for (int e = threadIdx.x; e < kLiftPT * r; e += blockDim.x) {
    int u = e / r, j = e - u * r;
    cs[u][j] = (p0 + u < P) ? coef[(p0 + u) * r + j] : S::zero();
  }
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  T acc[kLiftPT];
#pragma unroll
  for (int u = 0; u < kLiftPT; ++u) acc[u] = S::zero();
  const T* xr = X + i * r;
  for (int j = 0; j < r; ++j) {
    const T v = xr[j];
#pragma unroll
    for (int u = 0; u < kLiftPT; ++u) acc[u] = S::add(acc[u], S::mul(v, cs[u][j]));
  }
#pragma unroll
  for (int u = 0; u < kLiftPT; ++u)
    if (p0 + u < P) x[(p0 + u) * n + i] = acc[u];
}

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
  return t;  // valid on thread 0
}

// Stencil residual for ONE parameter value per blockIdx.y; grid.x strides over rows.
// Partial sums of |A x - b|^2 and |b|^2 per CTA go to part[(p * gridDim.x + bx) * 2].
// Coefficients c_e(p) = exp(sum_k p_k phi[row][e][k]) / hh as in the online rows.
__global__ void __launch_bounds__(256) k_resid_stencil(const double* __restrict__ X, int64_t n, int r,
                                                       const int64_t* __restrict__ nbr,   // n x E
                                                       const double* __restrict__ phi,    // n x E x dp
                                                       int E, int dp, double hh,
                                                       const double* __restrict__ b,      // n
                                                       const double* __restrict__ params, // P x dp
                                                       const double* __restrict__ coef,   // P x r
                                                       double* __restrict__ part) {
  __shared__ double cs[64];
  __shared__ double red[32];
  const int64_t p = blockIdx.y;
  for (int j = threadIdx.x; j < r; j += blockDim.x) cs[j] = coef[p * r + j];
  __syncthreads();
  const double* pp = params + p * dp;
  double rr = 0.0, bb = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double xi = 0.0;
    for (int j = 0; j < r; ++j) xi = fma(X[i * r + j], cs[j], xi);
    double diag = 0.0, off = 0.0;
    for (int e = 0; e < E; ++e) {
      const double* ph = phi + (i * E + e) * dp;
      double arg = dmul_exact(pp[0], ph[0]);
      for (int k = 1; k < dp; ++k) arg = dadd_exact(arg, dmul_exact(pp[k], ph[k]));
      const double c = exp(arg) / hh;
      diag = dadd_exact(diag, c);
      const int64_t m = nbr[i * E + e];
      if (m >= 0) {
        double xm = 0.0;
        for (int j = 0; j < r; ++j) xm = fma(X[m * r + j], cs[j], xm);
        off = fma(-c, xm, off);
      }
    }
    const double ax = fma(diag, xi, off);
    const double res = ax - b[i];
    rr = fma(res, res, rr);
    bb = fma(b[i], b[i], bb);
  }
  double trr = block_sum(rr, red);
  double tbb = block_sum(bb, red);
  if (threadIdx.x == 0) {
    part[(p * gridDim.x + blockIdx.x) * 2] = trr;
    part[(p * gridDim.x + blockIdx.x) * 2 + 1] = tbb;
  }
}

// Affine residual: sum_k f_k(p) A_k x - b with CSR A_k, for one p per blockIdx.y.
template <typename T>
__global__ void __launch_bounds__(256) k_resid_affine(const T* __restrict__ X, int64_t n, int r, int K,
                                                      const int64_t* const* __restrict__ rp,
                                                      const int64_t* const* __restrict__ ci,
                                                      const T* const* __restrict__ va,
                                                      const T* __restrict__ fcoef,  // P x K
                                                      const T* __restrict__ b,
                                                      const T* __restrict__ coef,   // P x r
                                                      double* __restrict__ part) {
  using S = Sc<T>;
  __shared__ T cs[64];
  __shared__ double red[32];
  const int64_t p = blockIdx.y;
  for (int j = threadIdx.x; j < r; j += blockDim.x) cs[j] = coef[p * r + j];
  __syncthreads();
  double rr = 0.0, bb = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    T ax = S::zero();
    for (int k = 0; k < K; ++k) {
      T rowacc = S::zero();
      for (int64_t q = rp[k][i]; q < rp[k][i + 1]; ++q) {
        const int64_t m = ci[k][q];
        T xm = S::zero();
        for (int j = 0; j < r; ++j) xm = S::add(xm, S::mul(X[m * r + j], cs[j]));
        rowacc = S::add(rowacc, S::mul(va[k][q], xm));
      }
      ax = S::add(ax, S::mul(fcoef[p * K + k], rowacc));
    }
    const T res = S::sub(ax, b[i]);
    rr += S::abs2(res);
    bb += S::abs2(b[i]);
  }
  double trr = block_sum(rr, red);
  double tbb = block_sum(bb, red);
  if (threadIdx.x == 0) {
    part[(p * gridDim.x + blockIdx.x) * 2] = trr;
    part[(p * gridDim.x + blockIdx.x) * 2 + 1] = tbb;
  }
}

// Gaussian-kernel residual: (K_p + ridge I) x - b with kernel entries
// re-evaluated on the fly (n^2 exps per p; used on a small subset of p).
__global__ void __launch_bounds__(256) k_resid_gauss(const double* __restrict__ X, int64_t n, int r,
                                                     const double* __restrict__ pts, int d,
                                                     double ridge, const double* __restrict__ b,
                                                     const double* __restrict__ params,
                                                     const double* __restrict__ xfull,  // P x n (lifted)
                                                     double* __restrict__ part) {
  __shared__ double red[32];
  const int64_t p = blockIdx.y;
  const double sg = params[p];
  const double inv = 1.0 / (2.0 * sg * sg);
  const double* x = xfull + p * n;
  double rr = 0.0, bb = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double* xi = pts + i * d;
    double acc = 0.0;
    for (int64_t l = 0; l < n; ++l) {
      const double* xl = pts + l * d;
      double dd = 0.0;
      for (int k = 0; k < d; ++k) {
        double df = __dsub_rn(xi[k], xl[k]);
        dd = __dadd_rn(dd, __dmul_rn(df, df));
      }
      double kv = exp(-(dd * inv));
      if (l == i) kv += ridge;
      acc = fma(kv, x[l], acc);
    }
    const double res = acc - b[i];
    rr = fma(res, res, rr);
    bb = fma(b[i], b[i], bb);
  }
  double trr = block_sum(rr, red);
  double tbb = block_sum(bb, red);
  if (threadIdx.x == 0) {
    part[(p * gridDim.x + blockIdx.x) * 2] = trr;
    part[(p * gridDim.x + blockIdx.x) * 2 + 1] = tbb;
  }
}

// relres[p] = sqrt(sum rr) / max(sqrt(sum bb), 1e-300), fixed-order sum over CTAs.
__global__ void k_resid_finish(const double* __restrict__ part, int nb, int64_t P, double* __restrict__ relres) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= P) return;
  double rr = 0.0, bb = 0.0;
  for (int q = 0; q < nb; ++q) {
    rr += part[(p * nb + q) * 2];
    bb += part[(p * nb + q) * 2 + 1];
  }
  relres[p] = sqrt(rr) / fmax(sqrt(bb), 1e-300);
}
