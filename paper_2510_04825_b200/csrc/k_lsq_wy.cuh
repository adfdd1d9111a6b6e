// K4 for the large real shapes (configs 3 and 5): blocked Householder QR in
// compact-WY form, trailing updates on the FP64 tensor path (DMMA m8n8k4).
// Same algorithm and outputs as k_lsq_sm / k_lsq_cw (Householder QR of
// [W M | W t], reference linalg.py:89-113 via online.py:105-134): the same
// reflectors H_k = I - tau_k v_k v_k^T (v_k = x - beta e_k, beta = -sign(x_k)|x|,
// tau_k = 1/(|x|(|x| + |x_k|))), applied eight at a time:
//
//   panel j (columns 8j .. 8j+7)   one warp, unblocked Householder on the panel
//                                  columns only (s x 8, registers + shared memory)
//   S1  W = V^T [V | A_trail]      DMMA, K = rows; the V^T V tile gives the
//                                  reflector cross products for S2
//   S2  Z_i = tau_i (W_i - sum_{l<i} (v_i.v_l) Z_l)   forward substitution, one
//                                  thread per trailing column (the T factor of
//                                  the compact-WY form, never formed)
//   S3  A_trail -= V Z             DMMA, K = 8, every warp a set of 8-row tiles
//
// which is H_8j+7 ... H_8j applied to the trailing columns (A_i+1 = A_i -
// tau_i v_i (v_i^T A_i) unrolled).  The unblocked kernels spend a warp
// butterfly per (column, step); here the row reduction of the trailing update
// happens inside the DMMA K dimension, and the trailing matrix is read and
// written once per 8 reflectors instead of once per reflector
// (profiles/r02_k4_tuning.txt: k_lsq_sm was bound by exactly that traffic).
//
// Layout.  [M | t] is column-major with column stride ld = 8 (mod 16) doubles,
// zero-padded to ld rows and to cpad = 8 ceil((r+1)/8) columns.  With that
// stride the 16-byte fragment loads below are conflict-free:
//   lane l reads rows 8 rt + 2 (l & 3), +1 of column 8 ct + (l >> 2)
// serves the A operand (V^T), the B operand (A_trail) of S1 - DMMA's k index is
// mapped to the even rows in the first and the odd rows in the second of the
// two instructions per 8-row tile - and the accumulator of S3 (computed as
// A^T -= Z^T V^T, so that a lane owns two consecutive rows of one column).
// V stays in place below the diagonal of its panel columns with the head
// v_kk = x_k - beta on the diagonal (R_kk = beta is kept in rdiag); the
// diagonal 8 x 8 tile is masked to its lower triangle when it is used as V.
//
// The unweighted [M | t] comes from a separate row-assembly kernel
// (k_wy_stencil_rows: K2 for a block of 32 parameter values per CTA, so the
// gathered basis rows G are read from L2 once per 32 parameter values instead
// of once per parameter value) in exactly this layout, and is brought in by ONE
// bulk async copy per parameter value (cp.async.bulk + mbarrier); the same
// global block serves the explicit sampled residual (online.py:121-124).
// Everything runs in a fixed order: results do not depend on the batch.
#pragma once
#include "k_lsq_sm.cuh"
#include "k_gauss.cuh"  // dmma884, mbarrier and bulk-copy helpers

__host__ __device__ inline int wy_ld(int s) {
  int ld = (s + 7) / 8 * 8;
  while ((ld & 15) != 8) ld += 8;
  return ld;
}
__host__ __device__ inline int wy_cpad(int r) { return (r + 1 + 7) / 8 * 8; }

// ---------------------------------------------------------------------------
// K2 as a standalone kernel: the unweighted [M(p) | t | 0] blocks (column-major,
// stride ld, cpad columns) of PB parameter values x RB selected rows per CTA.
// Arithmetic identical to AsmStencil (k_lsq.cuh): sequential no-FMA exponent
// sum, exp()/hh, diagonal in edge order, FMA chain over the gathered rows in G
// order - the blocks are bitwise what the fused assembler produces.
constexpr int kWyRB = 8;
constexpr int kWyPB = 32;

__host__ __device__ inline size_t wy_rows_smem_bytes(int E1, int r) {
  return ((size_t)kWyRB * E1 * r + 1) / 2 * 2 * sizeof(double) + (size_t)kWyPB * kWyRB * 8 * sizeof(double);
}

__global__ void __launch_bounds__(256)
k_wy_stencil_rows(int E, int dp, const double* __restrict__ phi, const double* __restrict__ G,
                  const int8_t* __restrict__ gmap, double hh, const double* __restrict__ params,
                  const double* __restrict__ t, int64_t t_stride, int64_t P, int s, int r, int ld, int cpad,
                  double* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char wy_rows_smem[];
  const int E1 = E + 1;
  double* Gs = reinterpret_cast<double*>(wy_rows_smem);
  double* cs = Gs + ((size_t)kWyRB * E1 * r + 1) / 2 * 2;
  const int tid = threadIdx.x;
  const int i0 = blockIdx.x * kWyRB;
  const int64_t p0 = (int64_t)blockIdx.y * kWyPB;
  const int np = (int)((P - p0 < kWyPB) ? (P - p0) : kWyPB);
  int nrows = s - i0;
  nrows = nrows > kWyRB ? kWyRB : (nrows < 0 ? 0 : nrows);
  const int gcount = nrows * E1 * r;
  const double* gsrc = G + (int64_t)i0 * E1 * r;
  for (int idx = tid; idx < gcount; idx += 256) Gs[idx] = __ldg(gsrc + idx);
  // edge coefficients, one (parameter value, row, edge) per thread and pass
  const int re = nrows * E, tot = np * re;
#pragma unroll 2
  for (int idx = tid; idx < tot; idx += 256) {
    const int pl = idx / re, rem = idx - pl * re;
    const int i = rem / E, e = rem - i * E;
    const double* ph = phi + ((int64_t)(i0 + i) * E + e) * dp;
    const double* pp = params + (p0 + pl) * dp;
    double arg = dmul_exact(pp[0], ph[0]);
    for (int k = 1; k < dp; ++k) arg = dadd_exact(arg, dmul_exact(pp[k], ph[k]));
    cs[(pl * kWyRB + i) * 8 + 1 + e] = exp(arg) / hh;
  }
  __syncthreads();
  // per (parameter value, row): the diagonal (edge order), then the signed
  // coefficient of every gathered row
  for (int idx = tid; idx < np * nrows; idx += 256) {
    const int pl = idx / nrows, i = idx - pl * nrows;
    double* ci = cs + (pl * kWyRB + i) * 8;
    double d = 0.0;
    for (int e = 0; e < E; ++e) d = dadd_exact(d, ci[1 + e]);
    const int8_t* mp = gmap + (i0 + i) * E1;
    double nv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int slot = (q < E1) ? mp[q] : -1;
      nv[q] = (slot < 0) ? 0.0 : (slot == 0 ? d : -ci[slot]);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) ci[q] = nv[q];
  }
  __syncthreads();
  // products: thread = (row i, column pair), the gathered rows of its two
  // columns in registers for all parameter values of the block
  const int i = tid & 7, j0 = 2 * (tid >> 3);
  if (j0 >= cpad) return;
  const int row = i0 + i;
  const bool rok = i < nrows;
  double g0[8], g1[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    g0[q] = (rok && q < E1 && j0 < r) ? Gs[(i * E1 + q) * r + j0] : 0.0;
    g1[q] = (rok && q < E1 && j0 + 1 < r) ? Gs[(i * E1 + q) * r + j0 + 1] : 0.0;
  }
  for (int pl = 0; pl < np; ++pl) {
    double m0 = 0.0, m1 = 0.0;
    if (rok) {
      const double2* c2 = reinterpret_cast<const double2*>(cs + (pl * kWyRB + i) * 8);
#pragma unroll
      for (int q2 = 0; q2 < 4; ++q2) {
        const double2 c = c2[q2];
        if (2 * q2 < E1) {
          m0 = fma(c.x, g0[2 * q2], m0);
          m1 = fma(c.x, g1[2 * q2], m1);
        }
        if (2 * q2 + 1 < E1) {
          m0 = fma(c.y, g0[2 * q2 + 1], m0);
          m1 = fma(c.y, g1[2 * q2 + 1], m1);
        }
      }
      const double tv = (j0 == r || j0 + 1 == r) ? t[(p0 + pl) * t_stride + row] : 0.0;
      if (j0 >= r) m0 = (j0 == r) ? tv : 0.0;
      if (j0 + 1 >= r) m1 = (j0 + 1 == r) ? tv : 0.0;
    }
    double* ob = out + (p0 + pl) * (int64_t)ld * cpad + row;
    ob[(int64_t)j0 * ld] = m0;
    ob[(int64_t)(j0 + 1) * ld] = m1;
  }
}

// ---------------------------------------------------------------------------
__host__ __device__ inline size_t lsq_wy_smem_bytes(int ld, int cpad) {
  // A, W partials (2 x 8 x cpad), Z (8 x cpad), weights, tau/R_kk/|R_kk|/c (64 each),
  // residual partials (32), rank info (2), mbarrier
  return ((size_t)ld * cpad + 24 * (size_t)cpad + ld + 4 * 64 + 32 + 2) * sizeof(double) + 16;
}

// Panel j: unblocked Householder on columns [8j, 8j+8) by one warp.  Lane l
// holds rows l + 32u of a column.  Reflector columns are k < r; the remaining
// panel columns (t, zero padding) are only updated.
template <int RA>
__device__ __forceinline__ void wy_panel(double* A, int ld, int s, int r, int j, int lane, double* tau_s,
                                         double* rdiag, double* nrm_s) {
  const int k0 = 8 * j, cend = k0 + 8;
  const int kend = (cend < r) ? cend : r;
  for (int k = k0; k < kend; ++k) {
    double* colk = A + (size_t)k * ld;
    double v[RA];
    double ss = 0.0;
#pragma unroll
    for (int u = 0; u < RA; ++u) {
      const int i = lane + 32 * u;
      const double x = (i < s) ? colk[i] : 0.0;
      v[u] = (i >= k) ? x : 0.0;
      ss += v[u] * v[u];
    }
    ss = warp_allreduce_d(ss);
    double al = 0.0;
#pragma unroll
    for (int u = 0; u < RA; ++u)
      if (u == (k >> 5)) al = v[u];
    const double alpha = __shfl_sync(0xffffffffu, al, k & 31);
    const double nrm = sqrt(ss);
    const double aa = fabs(alpha);
    double beta = 0.0, tau = 0.0;
    if (nrm != 0.0) {
      beta = (aa == 0.0) ? -nrm : copysign(nrm, -alpha);   // -sign(x_k) |x|
      tau = rcp_nr(nrm * (nrm + aa));
    }
    const double vhead = alpha - beta;
#pragma unroll
    for (int u = 0; u < RA; ++u)
      if (lane + 32 * u == k) {
        v[u] = vhead;
        colk[k] = vhead;   // V in place: the head on the diagonal, R_kk in rdiag
      }
    if (lane == 0) {
      tau_s[k] = tau;
      rdiag[k] = beta;
      nrm_s[k] = nrm;
    }
    for (int c = k + 1; c < cend; c += 4) {
      double y[4][RA];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double* col = A + (size_t)(c + q) * ld;
#pragma unroll
        for (int u = 0; u < RA; ++u) {
          const int i = lane + 32 * u;
          y[q][u] = (c + q < cend && i < s) ? col[i] : 0.0;
        }
      }
      sm_apply<double, RA, 4>(y, v, tau);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        double* col = A + (size_t)(c + q) * ld;
#pragma unroll
        for (int u = 0; u < RA; ++u) {
          const int i = lane + 32 * u;
          if (c + q < cend && i < s) col[i] = y[q][u];
        }
      }
    }
  }
  for (int k = kend + lane; k < cend; k += 32) tau_s[k] = 0.0;
}

#ifdef SAS_WY_PROF
#define WY_PROF_MARK(ph) do { wy_t1 = clock64(); wy_tp[ph] += wy_t1 - wy_t0; wy_t0 = wy_t1; } while (0)
#else
#define WY_PROF_MARK(ph) do {} while (0)
#endif

// One CTA of W warps per parameter value (persistent over p); s <= 32 RA rows,
// r + 1 <= 8 NTM columns.  Mg: P blocks of ld x cpad doubles (k_wy_stencil_rows).
template <int RA, int W, int MINB, int NTM>
__global__ void __launch_bounds__(32 * W, MINB)
k_lsq_wy(LsqArgs<double> a, const double* __restrict__ Mg, int ld, int cpad) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int s = a.s, r = a.r;
  const int nt = cpad >> 3, rtn = ld >> 3;
  double* A = reinterpret_cast<double*>(smem_raw);
  double* Wp = A + (size_t)ld * cpad;
  double* Zs = Wp + 16 * cpad;
  double* ws = Zs + 8 * cpad;
  double* tau_s = ws + ld;
  double* rdiag = tau_s + 64;
  double* nrm_s = rdiag + 64;
  double* cvec = nrm_s + 64;
  double* red = cvec + 64;
  double* rinfo = red + 32;
  uint64_t* bar = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(rinfo + 2) + 7) & ~(uintptr_t)7);
  for (int i = tid; i < ld; i += 32 * W) ws[i] = (i < s) ? (a.w ? a.w[i] : 1.0) : 0.0;
  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const unsigned bytes = (unsigned)((size_t)ld * cpad * sizeof(double));
  const int64_t blk = (int64_t)ld * cpad;
  const int npanel = (r + 7) >> 3;
  const int lq = lane >> 2, lr = lane & 3;
  unsigned phase = 0;
#ifdef SAS_WY_PROF
  long long wy_tp[6] = {0, 0, 0, 0, 0, 0}, wy_t0 = clock64(), wy_t1;
#endif

  for (int64_t p = blockIdx.x; p < a.P; p += gridDim.x) {
    const double* mg = Mg + p * blk;
    if (tid == 0) {
      // the previous parameter value's generic-proxy accesses to A are ordered
      // before the async-proxy write by the barrier that ended its finish
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      mbar_expect_tx(bar, bytes);
      bulk_g2s(A, mg, bytes, bar);
      if (p + gridDim.x < a.P)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(mg + (int64_t)gridDim.x * blk), "r"(bytes)
                     : "memory");
    }
    mbar_wait(bar, phase);
    phase ^= 1u;
    WY_PROF_MARK(0);
    // weights in place, non-finite test (linalg.py:36-37, 102-105)
    bool bad = false;
    {
      const int n2 = ld >> 1;
      for (int jc = warp; jc <= r; jc += W) {
        double2* col = reinterpret_cast<double2*>(A + (size_t)jc * ld);
        for (int i2 = lane; i2 < n2; i2 += 32) {
          double2 m = col[i2];
          if (jc < r && !(isfinite(m.x) && isfinite(m.y))) bad = true;
          if (a.w) {
            m.x *= ws[2 * i2];
            m.y *= ws[2 * i2 + 1];
            col[i2] = m;
          }
        }
      }
    }
    if (__syncthreads_or(bad)) {
      lsq_nonfinite<double>(a, p);
      continue;
    }
    WY_PROF_MARK(1);

    for (int j = 0; j < npanel; ++j) {
      if (warp == 0) wy_panel<RA>(A, ld, s, r, j, lane, tau_s, rdiag, nrm_s);
      __syncthreads();
      WY_PROF_MARK(2);
      const int ntrail = nt - 1 - j;
      if (ntrail <= 0) break;
      // S1: W = V^T [V | A_trail], two K halves (even / odd 8-row tiles) per column tile
      {
        const double* vcol = A + (size_t)(8 * j + lq) * ld + 2 * lr;
        const bool m0 = 2 * lr >= lq, m1 = 2 * lr + 1 >= lq;   // lower triangle of the diagonal tile
        for (int u = warp; u < 2 * (ntrail + 1); u += W) {
          const int ti = u >> 1, ks = u & 1, ct = j + ti;
          const double* acol = A + (size_t)(8 * ct + lq) * ld + 2 * lr;
          double c0a = 0.0, c1a = 0.0, c0b = 0.0, c1b = 0.0;
          int rt = j + ks;
          if (ks == 0) {
            double2 vv = *reinterpret_cast<const double2*>(vcol + 8 * rt);
            double2 av = *reinterpret_cast<const double2*>(acol + 8 * rt);
            vv.x = m0 ? vv.x : 0.0;
            vv.y = m1 ? vv.y : 0.0;
            if (ti == 0) {
              av.x = m0 ? av.x : 0.0;
              av.y = m1 ? av.y : 0.0;
            }
            dmma884(c0a, c1a, vv.x, av.x);
            dmma884(c0b, c1b, vv.y, av.y);
            rt += 2;
          }
#pragma unroll 2
          for (; rt < rtn; rt += 2) {
            const double2 vv = *reinterpret_cast<const double2*>(vcol + 8 * rt);
            const double2 av = *reinterpret_cast<const double2*>(acol + 8 * rt);
            dmma884(c0a, c1a, vv.x, av.x);
            dmma884(c0b, c1b, vv.y, av.y);
          }
          *reinterpret_cast<double2*>(Wp + (size_t)(8 * ks + lq) * cpad + 8 * ct + 2 * lr) =
              make_double2(c0a + c0b, c1a + c1b);
        }
      }
      __syncthreads();
      WY_PROF_MARK(3);
      // S2: Z_i = tau_i (W_i - sum_{l<i} (v_i . v_l) Z_l), stored negated
      if (tid < 8 * ntrail) {
        const int col = 8 * (j + 1) + tid;
        const double* g0 = Wp + 8 * j;
        const double* g1 = Wp + (size_t)8 * cpad + 8 * j;
        double z[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          double wv = Wp[(size_t)i * cpad + col] + Wp[(size_t)(8 + i) * cpad + col];
#pragma unroll
          for (int l = 0; l < i; ++l) wv = fma(-(g0[(size_t)i * cpad + l] + g1[(size_t)i * cpad + l]), z[l], wv);
          z[i] = tau_s[8 * j + i] * wv;
          Zs[(size_t)i * cpad + col] = -z[i];
        }
      }
      __syncthreads();
      // S3: A_trail -= V Z as A^T += (-Z)^T V^T, every warp its 8-row tiles
      {
        double za[NTM][2];
#pragma unroll
        for (int ti = 0; ti < NTM; ++ti) {
          const bool ok = ti < ntrail;
          const int cc = 8 * (j + 1 + ti) + lq;
          za[ti][0] = ok ? Zs[(size_t)lr * cpad + cc] : 0.0;
          za[ti][1] = ok ? Zs[(size_t)(lr + 4) * cpad + cc] : 0.0;
        }
        const double* v0 = A + (size_t)(8 * j + lr) * ld + lq;
        const double* v1 = A + (size_t)(8 * j + lr + 4) * ld + lq;
        for (int rt = j + warp; rt < rtn; rt += W) {
          double b0 = v0[8 * rt], b1 = v1[8 * rt];
          if (rt == j) {
            b0 = (lq >= lr) ? b0 : 0.0;
            b1 = (lq >= lr + 4) ? b1 : 0.0;
          }
          double* cbase = A + (size_t)(8 * (j + 1) + lq) * ld + 8 * rt + 2 * lr;
#pragma unroll
          for (int ti = 0; ti < NTM; ++ti) {
            if (ti < ntrail) {
              double2* cp = reinterpret_cast<double2*>(cbase + (size_t)8 * ti * ld);
              double2 c = *cp;
              dmma884(c.x, c.y, za[ti][0], b0);
              dmma884(c.x, c.y, za[ti][1], b1);
              *cp = c;
            }
          }
        }
      }
      __syncthreads();
      WY_PROF_MARK(4);
    }
    sm_finish<double>(a, p, A, ld, mg, cvec, rdiag, nrm_s, rinfo, red, ld);
    WY_PROF_MARK(5);
  }
#ifdef SAS_WY_PROF
  if (tid == 0 && blockIdx.x < 2)
    printf("wy_prof block %d: load %lld weights %lld panel %lld S1 %lld S2+S3 %lld finish %lld cycles (all p of the CTA)\n",
           blockIdx.x, wy_tp[0], wy_tp[1], wy_tp[2], wy_tp[3], wy_tp[4], wy_tp[5]);
#endif
}
