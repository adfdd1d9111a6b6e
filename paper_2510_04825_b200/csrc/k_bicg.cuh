// Offline snapshot solves for the large affine systems (config 4's complex,
// non-symmetric transfer-function sweep): Jacobi-preconditioned BiCGSTAB on a
// CSR matrix A(p) = sum_k f_k(p) A_k.  Replaces the reference's SuperLU
// full_solve (systems.py:187-222), impractical at n = 1e6, with the same
// residual guard applied by the caller.
//
// Five fused kernels per iteration, no host round trip between them:
//   k_bicg_p     rho = <rhat, r> (from the previous kernel's CTA partials),
//                beta = (rho / rho_old)(alpha / omega), p = r + beta (p - omega v), phat = p / d
//   k_bicg_spmv  v = A phat, partials of <rhat, v>
//   k_bicg_s     alpha = rho / <rhat, v>, s = r - alpha v, shat = s / d
//   k_bicg_spmv  t = A shat, partials of <t, s> and <t, t>
//   k_bicg_x     omega = <t, s> / <t, t>, x += alpha phat + omega shat, r = s - omega t,
//                partials of <rhat, r>, |r|^2, |x|^2
// Every CTA re-sums the partials in index order (fixed-order reductions: the
// iterates do not depend on timing).  The scalars live in two device slots
// (iteration parity); block 0 publishes the new ones for the next kernel.
#pragma once
#include "k_cg.cuh"

template <typename T>
struct BicgScal {
  T rho, alpha, omega;
};

__device__ __forceinline__ double bicg_cmul(double a, double b) { return a * b; }   // conj(a) b
__device__ __forceinline__ cplx bicg_cmul(cplx a, cplx b) {
  return cplx{fma(a.re, b.re, a.im * b.im), fma(a.re, b.im, -(a.im * b.re))};
}
__device__ __forceinline__ double bicg_re(double a) { return a; }
__device__ __forceinline__ double bicg_re(cplx a) { return a.re; }
__device__ __forceinline__ double bicg_im(double) { return 0.0; }
__device__ __forceinline__ double bicg_im(cplx a) { return a.im; }
__device__ __forceinline__ void bicg_make(double& t, double re, double) { t = re; }
__device__ __forceinline__ void bicg_make(cplx& t, double re, double im) { t = cplx{re, im}; }

constexpr int kBicgPart = 6;   // per CTA: dot1 (re, im), dot2 (re, im), |.|^2, |.|^2

template <typename T>
__device__ __forceinline__ T bicg_sum_dot(const double* __restrict__ part, int nb, int slot, double* red, double* bc) {
  const double re = cg_sum_partials(part + slot, nb, kBicgPart, red, bc);
  __syncthreads();
  double im = 0.0;
  if (!std::is_same<T, double>::value) {
    im = cg_sum_partials(part + slot + 1, nb, kBicgPart, red, bc);
    __syncthreads();
  }
  T t;
  bicg_make(t, re, im);
  return t;
}

template <typename T>
__device__ __forceinline__ void bicg_store_part(double* __restrict__ part, T d1, T d2, double a, double b,
                                                double* red) {
  const double v[6] = {bicg_re(d1), bicg_im(d1), bicg_re(d2), bicg_im(d2), a, b};
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    const double t = cg_block_sum(v[q], red);
    if (threadIdx.x == 0) part[(size_t)blockIdx.x * kBicgPart + q] = t;
  }
}

// x = 0, r = rhat = b, p = v = 0; partials (<rhat, r>, -, |r|^2, 0)
template <typename T>
__global__ void __launch_bounds__(kCgThreads) k_bicg_init(int64_t n, const T* __restrict__ b, T* __restrict__ x,
                                                          T* __restrict__ r, T* __restrict__ rhat, T* __restrict__ p,
                                                          T* __restrict__ v, double* __restrict__ part,
                                                          BicgScal<T>* __restrict__ scal) {
  using S = Sc<T>;
  __shared__ double red[32];
  double rr = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const T bi = b[i];
    x[i] = S::zero();
    r[i] = bi;
    rhat[i] = bi;
    p[i] = S::zero();
    v[i] = S::zero();
    rr += S::abs2(bi);
  }
  T d1;
  bicg_make(d1, rr, 0.0);   // <b, b>
  bicg_store_part<T>(part, d1, S::zero(), rr, 0.0, red);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    T one;
    bicg_make(one, 1.0, 0.0);
    scal[0] = scal[1] = BicgScal<T>{one, one, one};
  }
}

template <typename T>
__global__ void __launch_bounds__(kCgThreads) k_bicg_p(int64_t n, const T* __restrict__ d, const T* __restrict__ r,
                                                       const T* __restrict__ v, T* __restrict__ p,
                                                       T* __restrict__ phat, const double* __restrict__ part_x,
                                                       const BicgScal<T>* __restrict__ prev,
                                                       BicgScal<T>* __restrict__ cur) {
  using S = Sc<T>;
  __shared__ double red[32];
  __shared__ double bc;
  const T rho = bicg_sum_dot<T>(part_x, gridDim.x, 0, red, &bc);
  const BicgScal<T> o = *prev;
  const T beta = S::mul(S::div(rho, o.rho), S::div(o.alpha, o.omega));
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const T pi = S::add(r[i], S::mul(beta, S::sub(p[i], S::mul(o.omega, v[i]))));
    p[i] = pi;
    phat[i] = S::div(pi, d[i]);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cur->rho = rho;
}

// MODE 0: y = A xin, dot1 = <u, y>                      (u = rhat)
// MODE 1: y = A xin, dot1 = <y, u>, |y|^2 in slot 4     (u = s)
// MODE 2: no store,  |u - A xin|^2 in slot 4, |xin|^2 in slot 5   (u = b: the true residual)
template <typename T, int MODE>
__global__ void __launch_bounds__(kCgThreads) k_bicg_spmv(int64_t n, const int32_t* __restrict__ rp,
                                                          const int32_t* __restrict__ ci, const T* __restrict__ va,
                                                          const T* __restrict__ xin, const T* __restrict__ u,
                                                          T* __restrict__ y, double* __restrict__ part) {
  using S = Sc<T>;
  __shared__ double red[32];
  T d1 = S::zero();
  double a = 0.0, b2 = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    T acc = S::zero();
    const int q1 = rp[i + 1];
    for (int q = rp[i]; q < q1; ++q) acc = S::add(acc, S::mul(va[q], xin[ci[q]]));
    if (MODE == 0) {
      y[i] = acc;
      d1 = S::add(d1, bicg_cmul(u[i], acc));
    } else if (MODE == 1) {
      y[i] = acc;
      d1 = S::add(d1, bicg_cmul(acc, u[i]));
      a += S::abs2(acc);
    } else {
      a += S::abs2(S::sub(u[i], acc));
      b2 += S::abs2(xin[i]);
    }
  }
  bicg_store_part<T>(part, d1, S::zero(), a, b2, red);
}

template <typename T>
__global__ void __launch_bounds__(kCgThreads) k_bicg_s(int64_t n, const T* __restrict__ d, const T* __restrict__ r,
                                                       const T* __restrict__ v, T* __restrict__ s,
                                                       T* __restrict__ shat, const double* __restrict__ part_v,
                                                       BicgScal<T>* __restrict__ cur) {
  using S = Sc<T>;
  __shared__ double red[32];
  __shared__ double bc;
  const T rv = bicg_sum_dot<T>(part_v, gridDim.x, 0, red, &bc);
  const T alpha = S::div(cur->rho, rv);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const T si = S::sub(r[i], S::mul(alpha, v[i]));
    s[i] = si;
    shat[i] = S::div(si, d[i]);
  }
  __syncthreads();   // every thread has read cur->rho
  if (blockIdx.x == 0 && threadIdx.x == 0) cur->alpha = alpha;
}

template <typename T>
__global__ void __launch_bounds__(kCgThreads) k_bicg_x(int64_t n, const T* __restrict__ rhat,
                                                       const T* __restrict__ phat, const T* __restrict__ shat,
                                                       const T* __restrict__ s, const T* __restrict__ t,
                                                       T* __restrict__ x, T* __restrict__ r,
                                                       const double* __restrict__ part_t, BicgScal<T>* __restrict__ cur,
                                                       double* __restrict__ part_x) {
  using S = Sc<T>;
  __shared__ double red[32];
  __shared__ double bc;
  const T ts = bicg_sum_dot<T>(part_t, gridDim.x, 0, red, &bc);
  const double tt = cg_sum_partials(part_t + 4, gridDim.x, kBicgPart, red, &bc);
  __syncthreads();
  const T omega = S::mulr(ts, 1.0 / tt);
  const T alpha = cur->alpha;
  T d1 = S::zero();
  double rr = 0.0, xx = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const T xi = S::add(x[i], S::add(S::mul(alpha, phat[i]), S::mul(omega, shat[i])));
    x[i] = xi;
    const T ri = S::sub(s[i], S::mul(omega, t[i]));
    r[i] = ri;
    d1 = S::add(d1, bicg_cmul(rhat[i], ri));
    rr += S::abs2(ri);
    xx += S::abs2(xi);
  }
  bicg_store_part<T>(part_x, d1, S::zero(), rr, xx, red);
  if (blockIdx.x == 0 && threadIdx.x == 0) cur->omega = omega;
}
