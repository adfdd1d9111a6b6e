// K4: batched weighted least squares, one CTA (warp-group of W warps) per
// parameter value p.  Replaces linalg.solve_ls (reference linalg.py:89-113)
// called from online.solve_online (online.py:105-134):
//
//   M_w = diag(w) M, t_w = diag(w) t           (linalg.py:102-105)
//   Householder QR of [M_w | t_w]              (np.linalg.qr, linalg.py:106)
//   rank test  min|R_ii| < 1e-12 max|R_ii|      (linalg.py:107-112)
//   c = R^{-1} (Q^H t_w)[:r]                    (solve_triangular, linalg.py:113)
//   sampled residual ||w * (M c - t)||          (online.py:121-124, recomputed
//                                                explicitly from the unweighted M)
//   output value  (c^H X) c                     (online.py:125-127)
//
// Layout: the unweighted M(p) (s x r) and t sit in shared memory (column r of
// Ms).  Thread (warp w, lane l) keeps rows {w + W q} x columns {l + 32 c} of the
// weighted augmented matrix in registers (RPT x NC).  Householder step k needs
// ONE cross-thread reduction: the Gram row g_j = sum_{i>=k} conj(M_ik) M_ij for
// all j >= k (including the rhs column) gives |x| = sqrt(g_kk) and
// v^H M_j = g_j - conj(beta) M_kj at once; W per-warp partial rows are summed in
// a fixed order (deterministic, so results do not depend on the launch or the
// GPU count).  Two __syncthreads per column step; column k and row k are
// double-buffered.
//
// The assembler functor fills Ms with the unweighted M(p), entry (i, j) at
// Ms[i * ldm + j * ldc] (ldc = 1: row-major; k_lsq_sm passes ldm = 1 and
// ldc = its column stride for a column-major matrix):
//   AsmGlobal  - M precomputed by another kernel (Gaussian kernel rows, K3)
//   AsmAffine  - M = sum_k f_k(p) B_k with numpy's operation order (K1)
//   AsmStencil - edge-form stencil rows with exp-affine coefficients (K2)
#pragma once
#include <cfloat>
#include "sas_common.cuh"

template <typename T>
struct LsqArgs {
  int s, r;
  int64_t P;
  const double* w;    // s or nullptr
  const T* t;         // s (t_stride == 0) or P x s
  int64_t t_stride;
  const T* proj;      // r or nullptr
  T* coef;            // P x r
  double* sres;       // P
  double* outv;       // P x 2 or nullptr
  int32_t* status;    // P
  int32_t* badcol;    // P or nullptr
};

// Parameter value p as a complex number (params are P x dp, optionally complex).
struct ParamView {
  const double* params;
  int dp;
  int pcomplex;
  __device__ __forceinline__ cplx get(int64_t p, int k) const {
    if (pcomplex) {
      const double* q = params + (p * dp + k) * 2;
      return cplx{q[0], q[1]};
    }
    return cplx{params[p * dp + k], 0.0};
  }
};

// Cooperative group the assembler runs on: the whole CTA (k_lsq) or one warp
// (k_lsq_warp, one parameter value per warp).
struct CtaGroup {
  __device__ __forceinline__ int rank() const { return threadIdx.x; }
  __device__ __forceinline__ int size() const { return blockDim.x; }
  __device__ __forceinline__ void sync() const { __syncthreads(); }
};
struct WarpGroup {
  __device__ __forceinline__ int rank() const { return threadIdx.x & 31; }
  __device__ __forceinline__ int size() const { return 32; }
  __device__ __forceinline__ void sync() const { __syncwarp(); }
};

// (i, j) walk over an s x r matrix in row-major order, stepping `step` entries
// per iteration without a division per element.
struct RowMajorWalk {
  int i, j, di, dj, r;
  __device__ __forceinline__ RowMajorWalk(int start, int step, int r_) : r(r_) {
    i = start / r_;
    j = start - i * r_;
    di = step / r_;
    dj = step - di * r_;
  }
  __device__ __forceinline__ void next() {
    i += di;
    j += dj;
    if (j >= r) { j -= r; ++i; }
  }
};

// ---------------------------------------------------------------------------
template <typename T>
struct AsmGlobal {
  const T* M;          // nsplit x P x s x r: split-K partial products (K3), summed in split order
  int nsplit = 1;
  int64_t split = 0;   // elements between partials
  static constexpr size_t scratch_bytes(int, int) { return 0; }
  template <class Grp>
  __device__ __forceinline__ void operator()(const Grp& g, int64_t p, T* Ms, int ldm, int s, int r,
                                             unsigned char*, int ldc = 1) const {
    const T* src = M + p * (int64_t)s * r;
    RowMajorWalk wk(g.rank(), g.size(), r);
    if (nsplit == 2) {  // K3's split-K partials: loads of 4 entries issued before their adds
      constexpr int U = 4;
      const int total = s * r, step = g.size();
      for (int base = g.rank(); base < total; base += U * step) {
        T v0[U], v1[U];
#pragma unroll
        for (int t = 0; t < U; ++t) {
          const int idx = base + t * step;
          v0[t] = idx < total ? src[idx] : T{};
          v1[t] = idx < total ? src[idx + split] : T{};
        }
#pragma unroll
        for (int t = 0; t < U; ++t) {
          if (base + t * step < total) Ms[wk.i * ldm + wk.j * ldc] = v0[t] + v1[t];
          wk.next();
        }
      }
      return;
    }
    for (int idx = g.rank(); idx < s * r; idx += g.size(), wk.next()) {
      T v = src[idx];
      for (int z = 1; z < nsplit; ++z) v = v + src[idx + z * split];
      Ms[wk.i * ldm + wk.j * ldc] = v;
    }
  }
};

// Affine coefficient f_k(p) with the reference's scalar semantics
// (systems.py:91-100: Python complex arithmetic; cmath.exp for "c*exp(a*p)").
template <typename T>
struct AffineCoef;

template <>
struct AffineCoef<double> {
  static __device__ __forceinline__ double eval(int kind, cplx scale, cplx rate, cplx pv,
                                                const double* tab) {
    switch (kind) {
      case 0: return scale.re;
      case 1: return dmul_exact(scale.re, pv.re);
      case 2: return dmul_exact(scale.re, exp(dmul_exact(rate.re, pv.re)));
      default: return tab[0];
    }
  }
};

template <>
struct AffineCoef<cplx> {
  static __device__ __forceinline__ cplx eval(int kind, cplx scale, cplx rate, cplx pv,
                                              const double* tab) {
    switch (kind) {
      case 0: return scale;
      case 1: return cmul_exact(scale, pv);
      case 2: {
        cplx z = cmul_exact(rate, pv);
        double m = exp(z.re);
        double sn, cs;
        sincos(z.im, &sn, &cs);
        return cmul_exact(scale, cplx{m * cs, m * sn});
      }
      default: return cplx{tab[0], tab[1]};
    }
  }
};

template <typename T>
struct AsmAffine {
  int K;
  const T* blocks;            // K x s x r
  const int32_t* kind;        // K
  const double* scale;        // K x 2
  const double* rate;         // K x 2
  ParamView pv;
  const double* coef_table;   // P x K x 2 or nullptr
  static constexpr size_t scratch_bytes(int, int) { return 16 * sizeof(T); }
  template <class Grp>
  __device__ __forceinline__ void operator()(const Grp& g, int64_t p, T* Ms, int ldm, int s, int r,
                                             unsigned char* scratch, int ldc = 1) const {
    T* f = reinterpret_cast<T*>(scratch);
    if (g.rank() < K) {
      int k = g.rank();
      cplx sc{scale[2 * k], scale[2 * k + 1]};
      cplx rt = rate ? cplx{rate[2 * k], rate[2 * k + 1]} : cplx{0.0, 0.0};
      const double* tab = coef_table ? coef_table + (p * K + k) * 2 : nullptr;
      f[k] = AffineCoef<T>::eval(kind[k], sc, rt, pv.get(p, 0), tab);
    }
    g.sync();
    const int64_t blk = (int64_t)s * r;
    RowMajorWalk wk(g.rank(), g.size(), r);
    for (int idx = g.rank(); idx < s * r; idx += g.size(), wk.next()) {
      // m = f0*B0; m = m + fk*Bk  (online.py:110-112, numpy elementwise order)
      T m = Sc<T>::mul_exact(f[0], blocks[idx]);
      for (int k = 1; k < K; ++k) m = Sc<T>::add_exact(m, Sc<T>::mul_exact(f[k], blocks[k * blk + idx]));
      Ms[wk.i * ldm + wk.j * ldc] = m;
    }
  }
};

// Edge-form stencil rows (real).  Row i of A(p) for node S_i:
//   c_e = exp(sum_k p_k phi[i][e][k]) / hh      (sequential sum, no FMA)
//   diag = sum_e c_e (edge order), off-diagonal -c_e for interior neighbours
// (the harness row oracle, oracle/online_ref.py stencil_rows).  The product
// with X accumulates the row's nonzeros in ascending column order with FMA,
// as the reference's dense rows_dense(...) @ basis does (online.py:62):
//   G[i][q] = X[node_q], gmap[i][q] = 0 (diagonal) | 1+e (edge e) | -1 (pad).
// kRows = 0: one (row, column) entry per thread, kUnroll entries' gathered
// rows in flight; kRows >= 1: one warp per selected row, kRows rows at a time,
// every lane owns column pairs (2 lane + 64 m, +1) loaded as 16-byte vectors
// (all E+1 gathered rows of kRows rows in flight per lane).  Same FMA order.
template <int kUnroll = 4, int kRows = 0>
struct AsmStencilT {
  static constexpr int kMaxEdges = 7;  // E + 1 <= 8 gathered rows per selected row
  int E, dp;
  const double* phi;    // s x E x dp
  const double* G;      // s x (E+1) x r
  const int8_t* gmap;   // s x (E+1)
  double hh;
  const double* params;  // P x dp (real)
  // per row 8 doubles: the diagonal and edge coefficients, then (rewritten in
  // place) the coefficient of each gathered row in G order (zero for padding)
  static size_t scratch_bytes(int s, int) { return (size_t)s * 8 * sizeof(double); }
  template <class Grp>
  __device__ __forceinline__ void operator()(const Grp& g, int64_t p, double* Ms, int ldm, int s, int r,
                                             unsigned char* scratch, int ldc = 1) const {
    double* cs = reinterpret_cast<double*>(scratch);
    const double* pp = params + p * dp;
    const int E1 = E + 1;
    // edge coefficients, one (row, edge) per thread and pass: the exp/division
    // chains are independent, so a thread's two unrolled passes overlap
    const int se = s * E;
#pragma unroll 2
    for (int idx = g.rank(); idx < se; idx += g.size()) {
      const int i = idx / E, e = idx - i * E;
      const double* ph = phi + (int64_t)idx * dp;
      double arg = dmul_exact(pp[0], ph[0]);
      for (int k = 1; k < dp; ++k) arg = dadd_exact(arg, dmul_exact(pp[k], ph[k]));
      cs[i * 8 + 1 + e] = exp(arg) / hh;
    }
    g.sync();
    // per row: the diagonal (edge order), then the signed coefficient of every
    // gathered row
    for (int i = g.rank(); i < s; i += g.size()) {
      double* ci = cs + i * 8;
      double d = 0.0;
      for (int e = 0; e < E; ++e) d = dadd_exact(d, ci[1 + e]);
      ci[0] = d;
      const int8_t* mp = gmap + i * E1;
      double nv[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int slot = (q < E1) ? mp[q] : -1;
        nv[q] = (slot < 0) ? 0.0 : (slot == 0 ? d : -ci[slot]);
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) ci[q] = nv[q];
    }
    g.sync();
    // M = rows @ G in ascending column order with FMA (padding slots add
    // 0 * 0); the gathered rows are L2-resident, the loads of kUnroll entries
    // are issued before their FMA chains
    if constexpr (kRows > 0) {
      if ((r & 1) == 0) {
        const int warp = g.rank() >> 5, lane = g.rank() & 31, nw = g.size() >> 5;
        for (int i0 = warp * kRows; i0 < s; i0 += nw * kRows) {
          for (int jb = 2 * lane; jb < r; jb += 64) {
            double2 gv[kRows][8];
#pragma unroll
            for (int t = 0; t < kRows; ++t) {
              const int i = i0 + t;
              const double* gr = G + ((int64_t)i * E1) * r + jb;
#pragma unroll
              for (int q = 0; q < 8; ++q)
                gv[t][q] = (i < s && q < E1) ? __ldg(reinterpret_cast<const double2*>(gr + (int64_t)q * r))
                                             : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int t = 0; t < kRows; ++t) {
              const int i = i0 + t;
              if (i >= s) break;
              const double* ci = cs + i * 8;
              double mx = 0.0, my = 0.0;
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                if (q < E1) {
                  const double c = ci[q];
                  mx = fma(c, gv[t][q].x, mx);
                  my = fma(c, gv[t][q].y, my);
                }
              }
              Ms[i * ldm + jb * ldc] = mx;
              Ms[i * ldm + (jb + 1) * ldc] = my;
            }
          }
        }
        return;
      }
    }
    const int total = s * r;
    RowMajorWalk wk(g.rank(), g.size(), r);
    for (int base = g.rank(); base < total; base += kUnroll * g.size()) {
      double gv[kUnroll][8];
      int ii[kUnroll], jj[kUnroll];
#pragma unroll
      for (int t = 0; t < kUnroll; ++t) {
        ii[t] = wk.i;
        jj[t] = wk.j;
        const bool ok = base + t * g.size() < total;
        const double* __restrict__ gr = G + ((int64_t)wk.i * E1) * r + wk.j;
#pragma unroll
        for (int q = 0; q < 8; ++q) gv[t][q] = (ok && q < E1) ? __ldg(gr + q * r) : 0.0;
        wk.next();
      }
#pragma unroll
      for (int t = 0; t < kUnroll; ++t) {
        if (base + t * g.size() < total) {
          const double2* a2 = reinterpret_cast<const double2*>(cs + ii[t] * 8);
          double m = 0.0;
#pragma unroll
          for (int q2 = 0; q2 < 4; ++q2) {
            const double2 a = a2[q2];
            if (2 * q2 < E1) m = fma(a.x, gv[t][2 * q2], m);
            if (2 * q2 + 1 < E1) m = fma(a.y, gv[t][2 * q2 + 1], m);
          }
          Ms[ii[t] * ldm + jj[t] * ldc] = m;
        }
      }
    }
  }
};
using AsmStencil = AsmStencilT<4, 2>;

// ---------------------------------------------------------------------------
template <typename T>
__host__ __device__ inline size_t lsq_smem_bytes(int s, int r, int W, int NC, size_t scratch) {
  const int ldm = r + 1, ncol = 32 * NC;
  size_t part = (size_t)2 * W * ncol;
  size_t rr = (size_t)r * ldm;
  size_t uni = part > rr ? part : rr;
  size_t n = (size_t)s * ldm + 2 * (size_t)s + 2 * (size_t)ncol + uni + ncol;
  return (n * sizeof(T) + (W + 8) * sizeof(double) + 15) / 16 * 16 + ((scratch + 15) / 16) * 16;
}

template <typename T, int NC, int RPT, class Asm>
__global__ void __launch_bounds__(512) k_lsq(LsqArgs<T> a, Asm as, size_t scratch_bytes) {
  using S = Sc<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int W = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = a.s, r = a.r, ldm = r + 1;
  constexpr int ncol = 32 * NC;
  const int nthr = blockDim.x;

  T* Ms = reinterpret_cast<T*>(smem_raw);
  T* colk = Ms + (size_t)s * ldm;
  T* rowk = colk + 2 * s;
  T* part = rowk + 2 * ncol;
  size_t partsz = (size_t)2 * W * ncol, rr = (size_t)r * ldm;
  T* cvec = part + (partsz > rr ? partsz : rr);
  double* red = reinterpret_cast<double*>(cvec + ncol);
  unsigned char* scratch = smem_raw + (reinterpret_cast<unsigned char*>(red + W + 8) - smem_raw + 15) / 16 * 16;
  (void)scratch_bytes;

  for (int64_t p = blockIdx.x; p < a.P; p += gridDim.x) {
    as(CtaGroup{}, p, Ms, ldm, s, r, scratch);
    for (int i = threadIdx.x; i < s; i += nthr) Ms[i * ldm + r] = a.t[p * a.t_stride + i];
    __syncthreads();

    T A[RPT][NC];
    bool bad = false;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int i = warp + W * q;
      const double wi = (i < s && a.w) ? a.w[i] : 1.0;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int j = lane + 32 * c;
        if (i < s && j <= r) {
          T m = Ms[i * ldm + j];
          if (j < r && !S::finite(m)) bad = true;
          A[q][c] = a.w ? S::mulr(m, wi) : m;
        } else {
          A[q][c] = S::zero();
        }
      }
    }
    if (__syncthreads_or(bad)) {
      for (int j = threadIdx.x; j < r; j += nthr) a.coef[p * r + j] = S::from(__longlong_as_double(0x7ff8000000000000ll), 0.0);
      if (threadIdx.x == 0) {
        a.status[p] = 2;
        a.sres[p] = __longlong_as_double(0x7ff8000000000000ll);
        if (a.badcol) a.badcol[p] = -1;
        if (a.outv) { a.outv[2 * p] = a.sres[p]; a.outv[2 * p + 1] = a.sres[p]; }
      }
      __syncthreads();
      continue;
    }

    double dmax = 0.0, dmin = DBL_MAX;
    int amin = 0;
    for (int k = 0; k < r; ++k) {
      const int buf = k & 1;
      T* ck = colk + buf * s;
      T* rk = rowk + buf * ncol;
      T* pt = part + (size_t)buf * W * ncol;
      const int lk = k & 31, sk = k >> 5;
      // publish column k (rows >= k) and row k (columns >= k)
      if (lane == lk) {
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
          const int i = warp + W * q;
          if (i >= k && i < s) {
#pragma unroll
            for (int c = 0; c < NC; ++c)
              if (c == sk) ck[i] = A[q][c];
          }
        }
      }
      if (warp == k % W) {
        const int qk = k / W;
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
          if (q == qk) {
#pragma unroll
            for (int c = 0; c < NC; ++c) {
              const int j = lane + 32 * c;
              if (j >= k && j <= r) rk[j] = A[q][c];
            }
          }
        }
      }
      __syncthreads();
      // per-warp partial Gram row
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int j = lane + 32 * c;
        if (j >= k && j <= r) {
          T acc = S::zero();
#pragma unroll
          for (int q = 0; q < RPT; ++q) {
            const int i = warp + W * q;
            if (i >= k && i < s) acc = S::fma_conj(ck[i], A[q][c], acc);
          }
          pt[warp * ncol + j] = acc;
        }
      }
      __syncthreads();
      // reduce (fixed order over warps) and form the reflector
      double gkk = 0.0;
      for (int w = 0; w < W; ++w) gkk += S::re(pt[w * ncol + k]);
      const T alpha = rk[k];
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
      T sj[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int j = lane + 32 * c;
        sj[c] = S::zero();
        if (j > k && j <= r) {
          T g = S::zero();
          for (int w = 0; w < W; ++w) g = S::add(g, pt[w * ncol + j]);
          T wj = S::sub(g, S::mul(S::conj(beta), rk[j]));
          sj[c] = S::mulr(wj, tau);
        }
      }
      // apply H = I - tau v v^H to the trailing columns
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const int i = warp + W * q;
        if (i >= k && i < s) {
          const T v = (i == k) ? S::sub(alpha, beta) : ck[i];
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            const int j = lane + 32 * c;
            if (j > k && j <= r) A[q][c] = S::fms(v, sj[c], A[q][c]);
            else if (j == k && i == k) A[q][c] = beta;
          }
        }
      }
    }
    __syncthreads();  // everyone is done reading part/colk/rowk of the last step

    // R (r x r upper) and y = (Q^H t_w)[:r] into shared memory (aliases part)
    T* Rs = part;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int i = warp + W * q;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int j = lane + 32 * c;
        if (i < r && j >= i && j <= r) Rs[i * ldm + j] = A[q][c];
      }
    }
    __syncthreads();
    const bool rankdef = (r > 0) && (dmin < 1e-12 * fmax(dmax, DBL_MIN));
    if (warp == 0) {
      if (!rankdef) {
        // column-oriented back substitution; lane l holds y_{l+32c}
        T y[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const int i = lane + 32 * c;
          y[c] = (i < r) ? Rs[i * ldm + r] : S::zero();
        }
        for (int k = r - 1; k >= 0; --k) {
          const int lk = k & 31, sk = k >> 5;
          T yk = S::zero();
#pragma unroll
          for (int c = 0; c < NC; ++c)
            if (c == sk) yk = y[c];
          T ckv = S::div(yk, Rs[k * ldm + k]);
          // broadcast from lane lk
          double re = __shfl_sync(0xffffffffu, S::re(ckv), lk);
          double im = __shfl_sync(0xffffffffu, S::im(ckv), lk);
          ckv = S::from(re, im);
          if (lane == 0) cvec[k] = ckv;
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            const int i = lane + 32 * c;
            if (i < k) y[c] = S::fms(Rs[i * ldm + k], ckv, y[c]);
          }
        }
      } else {
        for (int j = lane; j < r; j += 32) cvec[j] = S::from(__longlong_as_double(0x7ff8000000000000ll), 0.0);
      }
    }
    __syncthreads();

    // sampled residual ||w (M c - t)|| from the unweighted M (online.py:121-124)
    double ss = 0.0;
    for (int i = threadIdx.x; i < s; i += nthr) {
      T acc = S::zero();
      for (int j = 0; j < r; ++j) acc = S::add(acc, S::mul(Ms[i * ldm + j], cvec[j]));
      T res = S::sub(acc, Ms[i * ldm + r]);
      if (a.w) res = S::mulr(res, a.w[i]);
      ss += S::abs2(res);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    if (lane == 0) red[warp] = ss;
    for (int j = threadIdx.x; j < r; j += nthr) a.coef[p * r + j] = cvec[j];
    __syncthreads();
    if (threadIdx.x == 0) {
      double tot = 0.0;
      for (int w = 0; w < W; ++w) tot += red[w];
      a.sres[p] = rankdef ? __longlong_as_double(0x7ff8000000000000ll) : sqrt(tot);
      a.status[p] = rankdef ? 1 : 0;
      if (a.badcol) a.badcol[p] = rankdef ? amin : -1;
      if (a.outv) {
        if (a.proj) {
          T o = S::zero();
          for (int j = 0; j < r; ++j) o = S::add(o, S::mul(a.proj[j], cvec[j]));
          a.outv[2 * p] = S::re(o);
          a.outv[2 * p + 1] = S::im(o);
        } else {
          a.outv[2 * p] = 0.0;
          a.outv[2 * p + 1] = 0.0;
        }
      }
    }
    __syncthreads();
  }
}
