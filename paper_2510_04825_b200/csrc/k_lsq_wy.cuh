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
#ifndef SAS_WY_PB
#define SAS_WY_PB 32
#endif
#ifndef SAS_WY_CPT
#define SAS_WY_CPT 4
#endif
constexpr int kWyPB = SAS_WY_PB;    // parameter values per CTA
constexpr int kWyCPT = SAS_WY_CPT;  // columns per thread in the product phase (4: two p-halves of 128 threads; 2: one)
static_assert(kWyPB <= 32 && (kWyCPT == 2 || kWyCPT == 4), "k_wy_stencil_rows: 256 threads = 32 parameter values x 8 rows in the slot phase");
#ifndef SAS_WY_MINB
#define SAS_WY_MINB 1
#endif

__host__ __device__ inline size_t wy_rows_smem_bytes(int E1, int r, int dp) {
  // gathered rows (RB x E1 x r), slot coefficients [p][q/2][row] (double2), edge
  // coefficients [p][row][8], parameter values [p][dp]
  return (((size_t)kWyRB * E1 * r + 1) / 2 * 2 + 2 * (size_t)kWyPB * kWyRB * 8 + (size_t)kWyPB * dp) * sizeof(double);
}

__global__ void __launch_bounds__(256, SAS_WY_MINB)
k_wy_stencil_rows(int E, int dp, const double* __restrict__ phi, const double* __restrict__ G,
                  const int8_t* __restrict__ gmap, double hh, const double* __restrict__ params,
                  const double* __restrict__ t, int64_t t_stride, int64_t P, int s, int r, int ld, int cpad,
                  double* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char wy_rows_smem[];
  const int E1 = E + 1;
  double* Gs = reinterpret_cast<double*>(wy_rows_smem);
  double* cs = Gs + (kWyRB * E1 * r + 1) / 2 * 2;   // [pl][q / 2][row] double2: conflict-free reads below
  double* ce = cs + kWyPB * kWyRB * 8;              // [pl][row][edge] edge coefficients
  double* ps = ce + kWyPB * kWyRB * 8;              // [pl][dp]
  const int tid = threadIdx.x;
  const int i0 = blockIdx.x * kWyRB;
  const int64_t p0 = (int64_t)blockIdx.y * kWyPB;
  const int np = (int)((P - p0 < kWyPB) ? (P - p0) : kWyPB);
  int nrows = s - i0;
  nrows = nrows > kWyRB ? kWyRB : (nrows < 0 ? 0 : nrows);
  const int gcount = nrows * E1 * r;
  const double* gsrc = G + (int64_t)i0 * E1 * r;
  for (int idx = tid; idx < gcount; idx += 256) Gs[idx] = __ldg(gsrc + idx);
  for (int idx = tid; idx < np * dp; idx += 256) ps[idx] = __ldg(params + p0 * dp + idx);
  __syncthreads();
  // edge coefficients: thread = (row, edge) pair x parameter values pl = group, + groups, ...
  // (groups = 256 / pairs); phi of the pair in registers, the parameter values broadcast
  // from shared memory; four independent exp / division chains in flight per thread
  {
    const int npair = nrows * E;
    const int groups = npair > 0 ? 256 / npair : 0;
    const int pg = npair > 0 ? tid / npair : 0, pair = npair > 0 ? tid - pg * npair : 0;
    if (pg < groups) {
      const int i = pair / E, e = pair - i * E;
      const double* ph = phi + ((int64_t)(i0 + i) * E + e) * dp;
      double phr[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) phr[k] = (k < dp) ? __ldg(ph + k) : 0.0;
      double* cdst = ce + i * 8 + e;
      for (int pl = pg; pl < np; pl += 4 * groups) {
        double arg[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int pu = pl + u * groups;
          const double* pp = ps + (pu < np ? pu : pl) * dp;
          arg[u] = dmul_exact(pp[0], phr[0]);
#pragma unroll
          for (int k = 1; k < 8; ++k)
            if (k < dp) arg[u] = dadd_exact(arg[u], dmul_exact(pp[k], phr[k]));
        }
        double cv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) cv[u] = exp(arg[u]) / hh;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (pl + u * groups < np) cdst[(pl + u * groups) * kWyRB * 8] = cv[u];
      }
    }
  }
  __syncthreads();
  // per (parameter value, row): the diagonal (edge order), then the signed
  // coefficient of every gathered row
  {
    const int pl = tid >> 3, i = tid & 7;
    if (pl < np && i < nrows) {
      const double* ci = ce + (pl * kWyRB + i) * 8 - 1;   // ci[1 + e]: edge e
      double d = 0.0;
      for (int e = 0; e < E; ++e) d = dadd_exact(d, ci[1 + e]);
      const int8_t* mp = gmap + (i0 + i) * E1;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int slot = (q < E1) ? mp[q] : -1;
        cs[((pl * 4 + (q >> 1)) * kWyRB + i) * 2 + (q & 1)] = (slot < 0) ? 0.0 : (slot == 0 ? d : -ci[slot]);
      }
    }
  }
  __syncthreads();
  // products: thread = (row i, kWyCPT columns), the gathered rows of its columns in
  // registers for the parameter values pl = half, half + NH, ...
  constexpr int CPT = kWyCPT, NG = 64 / CPT, NH = 256 / (kWyRB * NG);
  const int i = tid & 7, j0 = CPT * ((tid >> 3) % NG), half = tid / (kWyRB * NG);
  if (j0 >= cpad) return;
  const int row = i0 + i;
  const bool rok = i < nrows;
  double g[CPT][8];
#pragma unroll
  for (int c = 0; c < CPT; ++c)
#pragma unroll
    for (int q = 0; q < 8; ++q) g[c][q] = (rok && q < E1 && j0 + c < r) ? Gs[(i * E1 + q) * r + j0 + c] : 0.0;
  const int tc = r - j0;   // the t column among this thread's columns (0..CPT-1), if any
  double* ob = out + ((p0 + half) * (int64_t)cpad + j0) * ld + row;
  const int64_t ostep = NH * (int64_t)cpad * ld;
  const double2* c2 = reinterpret_cast<const double2*>(cs) + half * 4 * kWyRB + i;
  const double* tp = t + (p0 + half) * t_stride + row;
#pragma unroll 2
  for (int pl = half; pl < np; pl += NH) {
    double m[CPT];
#pragma unroll
    for (int cc = 0; cc < CPT; ++cc) m[cc] = 0.0;
#pragma unroll
    for (int q2 = 0; q2 < 4; ++q2) {
      const double2 c = c2[q2 * kWyRB];
#pragma unroll
      for (int cc = 0; cc < CPT; ++cc) {
        if (2 * q2 < E1) m[cc] = fma(c.x, g[cc][2 * q2], m[cc]);
        if (2 * q2 + 1 < E1) m[cc] = fma(c.y, g[cc][2 * q2 + 1], m[cc]);
      }
    }
    if (!rok) {   // padding rows (their coefficient slots are not initialised)
#pragma unroll
      for (int cc = 0; cc < CPT; ++cc) m[cc] = 0.0;
    }
    if (tc >= 0 && tc < CPT) {
      const double tv = rok ? *tp : 0.0;
#pragma unroll
      for (int cc = 0; cc < CPT; ++cc)
        if (cc == tc) m[cc] = tv;
    }
#pragma unroll
    for (int cc = 0; cc < CPT; ++cc)
      if (j0 + cc < cpad) ob[cc * ld] = m[cc];
    ob += ostep;
    c2 += NH * 4 * kWyRB;
    tp += NH * t_stride;
  }
}

// ---------------------------------------------------------------------------
constexpr int kWyWarps = 8;        // warps 0..3 factor panels, all eight run the DMMA phases
constexpr int kWyPanelWarps = 4;

__host__ __device__ inline size_t lsq_wy_smem_bytes(int ld, int cpad) {
  // A (reused for the residual's per-warp row partials, kWyWarps x ld <= ld x cpad);
  // W partials (2 x 8 x cpad) + Z (8 x cpad); weights (ld); tau / R_kk / |R_kk| / c
  // (cpad each), residual partials (8), rank info (2), mbarrier
  return ((size_t)ld * cpad + 24 * (size_t)cpad + ld + 4 * (size_t)cpad + 8 + 2) * sizeof(double) + 16;
}

__device__ __forceinline__ void wy_bar_panel() { asm volatile("bar.sync 1, 128;\n" ::: "memory"); }

// Panel j: unblocked Householder on columns [8j, 8j+8), column-parallel over the
// four panel warps: warp g holds columns g and g+4 in registers (lane l: rows
// l + 32u).  Step k: the owner of column k forms the reflector (|x| from the
// norm carried over from the previous step) and writes the column - V in place,
// head on the diagonal - and tau to shared memory; after ONE named barrier the
// four warps read v and reflect their remaining columns, each with one warp
// reduction.  The owner of the next pivot column reduces q = |y_{k+1}[k:]|^2
// together with its dot product: the reflection preserves q, so the next norm
// below row k is q - y_{k+1,k}^2 (as exact as a direct sum unless one
// reflection removes most of the column; then it is summed directly).
// Reflector columns are k < r; the remaining panel columns (t, zero padding)
// are only updated.
template <int RA, int KK>
__device__ __forceinline__ void wy_panel_step(double (&y)[2][RA], double& ss, double* A, int ld, int s, int k0, int r,
                                              int g, int lane, const bool (&inb)[RA], double* tau_s, double* rdiag,
                                              double* nrm_s) {
  constexpr int OWN = KK & 3, SL = KK >> 2;
  const int k = k0 + KK;
  if (k >= r) return;   // uniform over the panel warps
  double* colk = A + k * ld + k0 + lane;   // row k0 + lane + 32u at colk[32u]
  if (g == OWN) {
    const double alpha = __shfl_sync(0xffffffffu, y[SL][0], KK);   // row k: lane KK, slot 0
    const double nrm = sqrt(ss);
    const double aa = fabs(alpha);
    double beta = 0.0, tau = 0.0;
    if (nrm != 0.0) {
      beta = (aa == 0.0) ? -nrm : copysign(nrm, -alpha);   // -sign(x_k) |x|
      tau = rcp_nr(fma(nrm, aa, ss));                      // 1 / (|x| (|x| + |x_k|)), |x|^2 = ss
    }
    const double vhead = alpha - beta;
    if (lane == KK) y[SL][0] = vhead;   // R above (lanes < KK), head, v below
#pragma unroll
    for (int u = 0; u < RA; ++u)
      if (inb[u]) colk[32 * u] = y[SL][u];
    if (lane == 0) {
      tau_s[k] = tau;
      rdiag[k] = beta;
      nrm_s[k] = nrm;
    }
  }
  wy_bar_panel();
  if constexpr (KK < 7) {
    constexpr int NOWN = (KK + 1) & 3, NSL = (KK + 1) >> 2;
    const bool act0 = g > KK, act1 = g + 4 > KK, nxt = g == NOWN;
    if (!act1) return;   // both of this warp's columns are finished (act0 implies act1)
    const double tau = tau_s[k];
    double v[RA];
#pragma unroll
    for (int u = 0; u < RA; ++u) v[u] = inb[u] ? colk[32 * u] : 0.0;
    if (lane < KK) v[0] = 0.0;   // rows k0 .. k-1 of column k are R entries
    double d0 = 0.0, d1 = 0.0, q = 0.0;
#pragma unroll
    for (int u = 0; u < RA; ++u) {
      d0 = fma(v[u], y[0][u], d0);
      d1 = fma(v[u], y[1][u], d1);
    }
    if (nxt) {
      const double y0 = (lane >= KK) ? y[NSL][0] : 0.0;
      q = y0 * y0;
#pragma unroll
      for (int u = 1; u < RA; ++u) q = fma(y[NSL][u], y[NSL][u], q);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        d0 += __shfl_xor_sync(0xffffffffu, d0, off);
        d1 += __shfl_xor_sync(0xffffffffu, d1, off);
        q += __shfl_xor_sync(0xffffffffu, q, off);
      }
    } else {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        d0 += __shfl_xor_sync(0xffffffffu, d0, off);
        d1 += __shfl_xor_sync(0xffffffffu, d1, off);
      }
    }
    const double w0 = act0 ? tau * d0 : 0.0, w1 = tau * d1;
#pragma unroll
    for (int u = 0; u < RA; ++u) {
      y[0][u] = fma(-w0, v[u], y[0][u]);
      y[1][u] = fma(-w1, v[u], y[1][u]);
    }
    if (nxt) {
      const double e = __shfl_sync(0xffffffffu, y[NSL][0], KK);   // row k of the next pivot column, reflected
      double ssn = fma(-e, e, q);
      if (!(ssn > 0.25 * q)) {
        const double y0 = (lane > KK) ? y[NSL][0] : 0.0;
        ssn = y0 * y0;
#pragma unroll
        for (int u = 1; u < RA; ++u) ssn = fma(y[NSL][u], y[NSL][u], ssn);
        ssn = warp_allreduce_d(ssn);
      }
      ss = ssn;
    }
  }
}

// The panel warps hold the rows at and below the panel's first row only:
// lane l, slot u = row 8j + l + 32u (rows above are finished R rows), so the
// pivot row of step KK is lane KK, slot 0 at compile time.
template <int RA>
__device__ __forceinline__ void wy_panel(double* A, int ld, int s, int r, int j, int g, int lane, double* tau_s,
                                         double* rdiag, double* nrm_s) {
  const int k0 = 8 * j;
  bool inb[RA];
#pragma unroll
  for (int u = 0; u < RA; ++u) inb[u] = k0 + lane + 32 * u < s;
  double y[2][RA];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const double* col = A + (k0 + g + 4 * c) * ld + k0 + lane;
#pragma unroll
    for (int u = 0; u < RA; ++u) y[c][u] = inb[u] ? col[32 * u] : 0.0;
  }
  double ss = 0.0;
  if (g == 0) {
#pragma unroll
    for (int u = 0; u < RA; ++u) ss = fma(y[0][u], y[0][u], ss);
    ss = warp_allreduce_d(ss);
  }
  wy_panel_step<RA, 0>(y, ss, A, ld, s, k0, r, g, lane, inb, tau_s, rdiag, nrm_s);
  wy_panel_step<RA, 1>(y, ss, A, ld, s, k0, r, g, lane, inb, tau_s, rdiag, nrm_s);
  wy_panel_step<RA, 2>(y, ss, A, ld, s, k0, r, g, lane, inb, tau_s, rdiag, nrm_s);
  wy_panel_step<RA, 3>(y, ss, A, ld, s, k0, r, g, lane, inb, tau_s, rdiag, nrm_s);
  wy_panel_step<RA, 4>(y, ss, A, ld, s, k0, r, g, lane, inb, tau_s, rdiag, nrm_s);
  wy_panel_step<RA, 5>(y, ss, A, ld, s, k0, r, g, lane, inb, tau_s, rdiag, nrm_s);
  wy_panel_step<RA, 6>(y, ss, A, ld, s, k0, r, g, lane, inb, tau_s, rdiag, nrm_s);
  wy_panel_step<RA, 7>(y, ss, A, ld, s, k0, r, g, lane, inb, tau_s, rdiag, nrm_s);
  // columns that were no pivots (t, padding: k >= r) go back updated; tau = 0 for them
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const int kc = k0 + g + 4 * c;
    if (kc >= r) {
      double* col = A + kc * ld + k0 + lane;
#pragma unroll
      for (int u = 0; u < RA; ++u)
        if (inb[u]) col[32 * u] = y[c][u];
      if (lane == 0) tau_s[kc] = 0.0;
    }
  }
}

// S3: A_trail -= V Z on column tiles [ti0, ti0 + ntile) after the panel, as
// A^T += (-Z)^T V^T, for the 8-row tiles rt = j + vw0, j + vw0 + stride, ...
template <int NTM>
__device__ __forceinline__ void wy_s3(double* A, const double* Zs, int ld, int cpad, int rtn, int j, int ti0,
                                      int ntile, int vw0, int stride, int lq, int lr) {
  if (ntile <= 0) return;
  double za[NTM][2];
#pragma unroll
  for (int ti = 0; ti < NTM; ++ti) {
    const bool ok = ti < ntile;
    const int cc = 8 * (j + 1 + ti0 + ti) + lq;
    za[ti][0] = ok ? Zs[lr * cpad + cc] : 0.0;
    za[ti][1] = ok ? Zs[(lr + 4) * cpad + cc] : 0.0;
  }
  const double* v0 = A + (8 * j + lr) * ld + lq;
  const double* v1 = v0 + 4 * ld;
  double* cb0 = A + (8 * (j + 1 + ti0) + lq) * ld + 2 * lr;
  for (int rt = j + vw0; rt < rtn; rt += stride) {
    double b0 = v0[8 * rt], b1 = v1[8 * rt];
    if (rt == j) {
      b0 = (lq >= lr) ? b0 : 0.0;
      b1 = (lq >= lr + 4) ? b1 : 0.0;
    }
    double* cbase = cb0 + 8 * rt;
#pragma unroll
    for (int ti = 0; ti < NTM; ++ti) {
      if (ti < ntile) {
        double2* cp = reinterpret_cast<double2*>(cbase + 8 * ti * ld);
        double2 c = *cp;
        dmma884(c.x, c.y, za[ti][0], b0);
        dmma884(c.x, c.y, za[ti][1], b1);
        *cp = c;
      }
    }
  }
}

// K2 inside the factorisation kernel (FUSED): the stencil rows of the NEXT
// parameter value are assembled by the warps that idle while the panel warps
// factor (one slice of row pairs per panel window) into this CTA's second
// global slot, which stays in L2; the block never makes the HBM round trip of
// the two-kernel path.  One warp per pair of selected rows: lanes 0..E-1 and
// 8..8+E-1 evaluate the edge coefficients of the two rows, every lane then
// builds the eight slot coefficients from shuffles and owns column pairs
// (2 lane + 64 m, +1) loaded as 16-byte vectors.  Arithmetic identical to
// AsmStencil (k_lsq.cuh): the blocks are bitwise what the other paths produce.
struct WyAsm {
  int E, dp;
  const double* phi;     // s x E x dp
  const double* G;       // s x (E+1) x r
  const int8_t* gmap;    // s x (E+1)
  double hh;
  const double* params;  // P x dp
  const double* t;       // s or P x s
  int64_t t_stride;
};

// Row pairs [m_lo, m_hi) of the block of parameter value p, by a group of nthr
// threads (rank tr; whole warps) synchronised by sync():
//   stage 1  edge coefficients c_e = exp(sum_k p_k phi_k) / hh, one (row, edge) per thread
//   stage 2  the eight slot coefficients of every row (diagonal in edge order)
//   stage 3  products, one warp per row pair, every lane column pairs (2 lane + 64 m, +1)
//            loaded as 16-byte vectors, the slot coefficients broadcast from shared memory
// cbuf: 16 doubles per row of the range (edge coefficients, then slot coefficients).
template <bool TWO, class Sync>
__device__ __forceinline__ void wy_asm_pairs(const WyAsm& as, int64_t p, int s, int r, int ld, double* dst, int m_lo,
                                             int m_hi, int tr, int nthr, double* cbuf, Sync sync) {
  const int E = as.E, E1 = E + 1, dp = as.dp;
  const int row0 = 2 * m_lo, nrw = 2 * (m_hi - m_lo);
  if (nrw <= 0) return;
  const double* pp = as.params + p * dp;
  double* ce = cbuf;
  double* cq = cbuf + 8 * nrw;
  for (int idx = tr; idx < nrw * E; idx += nthr) {
    const int rl = idx / E, e = idx - rl * E, row = row0 + rl;
    double c = 0.0;
    if (row < s) {
      const double* ph = as.phi + ((int64_t)row * E + e) * dp;
      double arg = dmul_exact(pp[0], ph[0]);
      for (int k = 1; k < dp; ++k) arg = dadd_exact(arg, dmul_exact(pp[k], ph[k]));
      c = exp(arg) / as.hh;
    }
    ce[rl * 8 + e] = c;
  }
  sync();
  for (int idx = tr; idx < nrw * 8; idx += nthr) {
    const int rl = idx >> 3, q = idx & 7, row = row0 + rl;
    const int slot = (q < E1 && row < s) ? as.gmap[row * E1 + q] : -1;
    double d = 0.0;
    for (int e = 0; e < E; ++e) d = dadd_exact(d, ce[rl * 8 + e]);
    cq[idx] = (slot < 0) ? 0.0 : (slot == 0 ? d : -ce[rl * 8 + slot - 1]);
  }
  sync();
  const int wi = tr >> 5, nw = nthr >> 5, lane = tr & 31;
  for (int m = m_lo + wi; m < m_hi; m += nw) {
    const int i0 = 2 * m, rl = i0 - row0;
    for (int jb = 2 * lane; jb < r; jb += 64) {
      double mres[2][2];
      const double* gr = as.G + ((int64_t)i0 * E1) * r + jb;
      if constexpr (TWO) {
        double2 gv[2][8];
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int q = 0; q < 8; ++q)
            gv[t][q] = (q < E1 && i0 + t < s) ? __ldcg(reinterpret_cast<const double2*>(gr + (int64_t)(t * E1 + q) * r))
                                              : make_double2(0.0, 0.0);
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const double2* c2 = reinterpret_cast<const double2*>(cq + (rl + t) * 8);
          double mx = 0.0, my = 0.0;
#pragma unroll
          for (int q2 = 0; q2 < 4; ++q2) {
            const double2 c = c2[q2];
            if (2 * q2 < E1) { mx = fma(c.x, gv[t][2 * q2].x, mx); my = fma(c.x, gv[t][2 * q2].y, my); }
            if (2 * q2 + 1 < E1) { mx = fma(c.y, gv[t][2 * q2 + 1].x, mx); my = fma(c.y, gv[t][2 * q2 + 1].y, my); }
          }
          mres[t][0] = mx;
          mres[t][1] = my;
        }
      } else {
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          double2 gv[8];
#pragma unroll
          for (int q = 0; q < 8; ++q)
            gv[q] = (q < E1 && i0 + t < s) ? __ldcg(reinterpret_cast<const double2*>(gr + (int64_t)(t * E1 + q) * r))
                                           : make_double2(0.0, 0.0);
          const double2* c2 = reinterpret_cast<const double2*>(cq + (rl + t) * 8);
          double mx = 0.0, my = 0.0;
#pragma unroll
          for (int q2 = 0; q2 < 4; ++q2) {
            const double2 c = c2[q2];
            if (2 * q2 < E1) { mx = fma(c.x, gv[2 * q2].x, mx); my = fma(c.x, gv[2 * q2].y, my); }
            if (2 * q2 + 1 < E1) { mx = fma(c.y, gv[2 * q2 + 1].x, mx); my = fma(c.y, gv[2 * q2 + 1].y, my); }
          }
          mres[t][0] = mx;
          mres[t][1] = my;
        }
      }
      *reinterpret_cast<double2*>(dst + (int64_t)jb * ld + i0) = make_double2(mres[0][0], mres[1][0]);
      *reinterpret_cast<double2*>(dst + (int64_t)(jb + 1) * ld + i0) = make_double2(mres[0][1], mres[1][1]);
    }
    if (lane < 2) dst[(int64_t)r * ld + i0 + lane] = (i0 + lane < s) ? as.t[p * as.t_stride + i0 + lane] : 0.0;
  }
}

struct WySyncCta { __device__ __forceinline__ void operator()() const { __syncthreads(); } };
struct WySyncUpd { __device__ __forceinline__ void operator()() const { asm volatile("bar.sync 2, 128;\n" ::: "memory"); } };

#ifdef SAS_WY_PROF
#define WY_PROF_MARK(ph) do { wy_t1 = clock64(); wy_tp[ph] += wy_t1 - wy_t0; wy_t0 = wy_t1; } while (0)
#else
#define WY_PROF_MARK(ph) do {} while (0)
#endif

// One CTA of eight warps per parameter value (persistent over p); s <= 32 RA rows,
// r + 1 <= 8 (NTM + 1) columns.  Mg: P blocks of ld x cpad doubles (k_wy_stencil_rows).
// Per panel: S1 (all warps) | S2 | S3 on the next panel's column tile (all warps) |
// warps 0..3 factor the next panel while warps 4..7 finish S3 (look-ahead).
// FUSED: Mg holds two blocks per CTA (slots), filled by the CTA itself (wy_asm_pairs).
template <int RA, int MINB, int NTM, bool FUSED>
__global__ void __launch_bounds__(32 * kWyWarps, MINB)
k_lsq_wy(LsqArgs<double> a, double* __restrict__ Mg, int ld, int cpad, WyAsm as) {
  constexpr int W = kWyWarps;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int s = a.s, r = a.r;
  const int nt = cpad >> 3, rtn = ld >> 3;
  double* A = reinterpret_cast<double*>(smem_raw);
  double* Wp = A + ld * cpad;                // 2 x 8 x cpad
  double* Zs = Wp + 16 * cpad;               // 8 x cpad
  double* ws = Zs + 8 * cpad;                // weights (1 when unweighted), ld
  double* tau_s = ws + ld;
  double* rdiag = tau_s + cpad;
  double* nrm_s = rdiag + cpad;
  double* cvec = nrm_s + cpad;
  double* red = cvec + cpad;
  double* rinfo = red + 8;
  uint64_t* bar = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(rinfo + 2) + 7) & ~(uintptr_t)7);
  const unsigned bytes = (unsigned)((size_t)ld * cpad * sizeof(double));
  const int64_t blk = (int64_t)ld * cpad;
  const int npanel = (r + 7) >> 3;
  const int lq = lane >> 2, lr = lane & 3;
  const int n2 = ld >> 1;
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  for (int i = tid; i < ld; i += 32 * W) ws[i] = (a.w && i < s) ? a.w[i] : 1.0;
  const int s2 = (s + 1) >> 1;                               // row pairs
  const int spw = (s2 + npanel - 1) / (npanel > 0 ? npanel : 1);   // row pairs per panel window
  double* slots = Mg + (int64_t)blockIdx.x * 2 * blk;       // FUSED: this CTA's two blocks
  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (FUSED && (int64_t)blockIdx.x < a.P) {
    // first block of this CTA, by all warps, in slices that fit the coefficient scratch
    for (int lo = 0; lo < s2; lo += spw) {
      wy_asm_pairs<MINB <= 2>(as, blockIdx.x, s, r, ld, slots, lo, lo + spw < s2 ? lo + spw : s2, tid, 32 * W, Wp,
                              WySyncCta{});
      __syncthreads();
    }
  }
  __syncthreads();
  if (tid == 0 && (int64_t)blockIdx.x < a.P) {
    asm volatile("fence.proxy.async;\n" ::: "memory");
    mbar_expect_tx(bar, bytes);
    bulk_g2s(A, FUSED ? slots : Mg + (int64_t)blockIdx.x * blk, bytes, bar);
  }
  unsigned phase = 0;
  int it = 0;
#ifdef SAS_WY_PROF
  long long wy_tp[8] = {0, 0, 0, 0, 0, 0, 0, 0}, wy_t0 = clock64(), wy_t1;
#endif

  for (int64_t p = blockIdx.x; p < a.P; p += gridDim.x, ++it) {
    const double* mg = FUSED ? slots + (it & 1) * blk : Mg + p * blk;
    double* mg_next = slots + ((it + 1) & 1) * blk;
    const bool has_next = p + gridDim.x < a.P;
    // the next parameter value's block: issued as soon as A is dead (after the
    // residual's row partials, which reuse A, are summed; all generic-proxy accesses to
    // A - and, FUSED, this CTA's global stores of the block - are ordered before the
    // async-proxy copy by the preceding barrier and the proxy fence)
    auto issue_next = [&]() {
      if (tid == 0 && has_next) {
        asm volatile("fence.proxy.async;\n" ::: "memory");
        mbar_expect_tx(bar, bytes);
        bulk_g2s(A, FUSED ? mg_next : mg + (int64_t)gridDim.x * blk, bytes, bar);
        if (!FUSED && p + 2 * (int64_t)gridDim.x < a.P)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(mg + 2 * (int64_t)gridDim.x * blk),
                       "r"(bytes)
                       : "memory");
      }
    };
    // FUSED: window w of the panel schedule assembles row pairs [w spw, (w+1) spw) of the next block
    auto asm_window = [&](int w) {
      if (FUSED && has_next) {
        const int lo = w * spw, hi = (lo + spw < s2) ? lo + spw : s2;
        wy_asm_pairs<MINB <= 2>(as, p + gridDim.x, s, r, ld, mg_next, lo, hi, tid - 32 * kWyPanelWarps,
                                32 * (W - kWyPanelWarps), Wp, WySyncUpd{});
      }
    };
    mbar_wait(bar, phase);
    phase ^= 1u;
    WY_PROF_MARK(0);
    // weights in place, non-finite test (linalg.py:36-37, 102-105): lane = row pairs
    // lane + 32m, warp = columns warp + W q.  Branch-free: an exponent field of all
    // ones (inf / nan) carries into the sign bit of badbits.
    bool bad = false;
    {
      double wr[8];
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int i = 2 * (lane + 32 * m);
        wr[2 * m] = (i < ld) ? ws[i] : 1.0;
        wr[2 * m + 1] = (i < ld) ? ws[i + 1] : 1.0;
      }
      unsigned badbits = 0u;
      for (int jc = warp; jc <= r; jc += W) {
        double2* col = reinterpret_cast<double2*>(A + jc * ld);
        const unsigned live = (jc < r) ? 0x7ff00000u : 0u;   // t is not tested (the reference tests M only)
        double2 mv[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) mv[m] = (lane + 32 * m < n2) ? col[lane + 32 * m] : make_double2(0.0, 0.0);
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          badbits |= (((unsigned)__double2hiint(mv[m].x) & live) + 0x00100000u) |
                     (((unsigned)__double2hiint(mv[m].y) & live) + 0x00100000u);
          if (lane + 32 * m < n2) col[lane + 32 * m] = make_double2(mv[m].x * wr[2 * m], mv[m].y * wr[2 * m + 1]);
        }
      }
      bad = (badbits >> 31) != 0u;
    }
    if (__syncthreads_or(bad)) {
      lsq_nonfinite<double>(a, p);
      if (FUSED && has_next) {   // no panel windows for this parameter value: assemble the next block now
        for (int lo = 0; lo < s2; lo += spw) {
          wy_asm_pairs<MINB <= 2>(as, p + gridDim.x, s, r, ld, mg_next, lo, lo + spw < s2 ? lo + spw : s2, tid, 32 * W,
                                  Wp, WySyncCta{});
          __syncthreads();
        }
      }
      issue_next();
      continue;
    }
    WY_PROF_MARK(1);
    if (warp < kWyPanelWarps) wy_panel<RA>(A, ld, s, r, 0, warp, lane, tau_s, rdiag, nrm_s);
    else asm_window(0);
    __syncthreads();
    WY_PROF_MARK(2);

    for (int j = 0; j < npanel; ++j) {
      const int ntrail = nt - 1 - j;
      if (ntrail <= 0) break;
      // S1: W = V^T [V | A_trail]: units (column tile, K half), K half ks = the 8-row
      // tiles j + ks, j + ks + 2, ...; the two halves are summed in S2
      {
        const double* vcol = A + (8 * j + lq) * ld + 2 * lr;
        const bool m0 = 2 * lr >= lq, m1 = 2 * lr + 1 >= lq;   // lower triangle of the diagonal tile
        for (int u = warp; u < 2 * (ntrail + 1); u += W) {
          const int ti = u >> 1, ks = u & 1;
          const double* acol = vcol + 8 * ti * ld;
          double c0a = 0.0, c1a = 0.0, c0b = 0.0, c1b = 0.0;
          int rt = j + ks;
          if (ks == 0) {
            double2 vv = *reinterpret_cast<const double2*>(vcol + 8 * rt);
            double2 av = *reinterpret_cast<const double2*>(acol + 8 * rt);
            vv.x = m0 ? vv.x : 0.0;
            vv.y = m1 ? vv.y : 0.0;
            if (ti == 0) av = vv;
            dmma884(c0a, c1a, vv.x, av.x);
            dmma884(c0b, c1b, vv.y, av.y);
            rt += 2;
          }
#pragma unroll 4
          for (; rt < rtn; rt += 2) {
            const double2 vv = *reinterpret_cast<const double2*>(vcol + 8 * rt);
            const double2 av = *reinterpret_cast<const double2*>(acol + 8 * rt);
            dmma884(c0a, c1a, vv.x, av.x);
            dmma884(c0b, c1b, vv.y, av.y);
          }
          *reinterpret_cast<double2*>(Wp + (8 * ks + lq) * cpad + 8 * (j + ti) + 2 * lr) =
              make_double2(c0a + c0b, c1a + c1b);
        }
      }
      __syncthreads();
      WY_PROF_MARK(3);
      // S2: Z_i = tau_i (W_i - sum_{l<i} (v_i . v_l) Z_l), stored negated
      if (tid < 8 * ntrail) {
        const int col = 8 * (j + 1) + tid;
        const double* b0 = Wp + 8 * j;
        const double* b1 = b0 + 8 * cpad;
        double gg[28], wv[8], tt[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          wv[i] = Wp[i * cpad + col] + Wp[(8 + i) * cpad + col];
          tt[i] = tau_s[8 * j + i];
#pragma unroll
          for (int l = 0; l < i; ++l) gg[i * (i - 1) / 2 + l] = b0[i * cpad + l] + b1[i * cpad + l];
        }
        double z[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          double x = wv[i];
#pragma unroll
          for (int l = 0; l < i; ++l) x = fma(-gg[i * (i - 1) / 2 + l], z[l], x);
          z[i] = tt[i] * x;
          Zs[i * cpad + col] = -z[i];
        }
      }
      __syncthreads();
      WY_PROF_MARK(4);
      if (j + 1 < npanel) {
        // the next panel's column tile first, then look-ahead
        wy_s3<1>(A, Zs, ld, cpad, rtn, j, 0, 1, warp, W, lq, lr);
        __syncthreads();
        WY_PROF_MARK(5);
        if (warp < kWyPanelWarps) wy_panel<RA>(A, ld, s, r, j + 1, warp, lane, tau_s, rdiag, nrm_s);
        else {
          wy_s3<NTM>(A, Zs, ld, cpad, rtn, j, 1, ntrail - 1, warp - kWyPanelWarps, W - kWyPanelWarps, lq, lr);
          asm_window(j + 1);
        }
        __syncthreads();
        WY_PROF_MARK(2);
      } else {
        wy_s3<NTM>(A, Zs, ld, cpad, rtn, j, 0, ntrail, warp, W, lq, lr);
        __syncthreads();
        WY_PROF_MARK(5);
      }
    }

    // rank test (linalg.py:107-112) and back substitution by warp 0
    if (warp == 0) {
      double mx = 0.0, mn = DBL_MAX;
      int am = 0x7fffffff;
      for (int jj = lane; jj < r; jj += 32) {
        const double d = nrm_s[jj];
        mx = fmax(mx, d);
        if (d < mn) { mn = d; am = jj; }
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
        // column sweep: lane i holds y_i and y_{i+32}; R column k is contiguous and
        // is fetched ahead of the dependent chain
        const double rinv0 = (lane < r) ? 1.0 / rdiag[lane] : 0.0;
        const double rinv1 = (lane + 32 < r) ? 1.0 / rdiag[lane + 32] : 0.0;
        double y0 = (lane < r) ? A[r * ld + lane] : 0.0;
        double y1 = (lane + 32 < r) ? A[r * ld + lane + 32] : 0.0;
        int k = r - 1;
        for (; k >= 32; --k) {          // pivots in the upper lane slot
          const double r0 = A[k * ld + lane], r1 = A[k * ld + lane + 32];
          const double ck = __shfl_sync(0xffffffffu, y1 * rinv1, k - 32);
          if (lane == 0) cvec[k] = ck;
          y0 = fma(-r0, ck, y0);
          if (lane + 32 < k) y1 = fma(-r1, ck, y1);
        }
#pragma unroll 4
        for (; k >= 0; --k) {
          const double r0 = A[k * ld + lane];
          const double ck = __shfl_sync(0xffffffffu, y0 * rinv0, k);
          if (lane == 0) cvec[k] = ck;
          if (lane < k) y0 = fma(-r0, ck, y0);
        }
      } else {
        for (int jj = lane; jj < r; jj += 32) cvec[jj] = qnan;
      }
    }
    __syncthreads();
    WY_PROF_MARK(6);
    const bool rankdef = rinfo[0] != 0.0;
    // sampled residual ||w (M c - t)|| from the unweighted block in global memory
    // (online.py:121-124): warp = columns warp + W q (t is column r with coefficient
    // -1), lane = row pairs, four columns' loads in flight; per-warp row partials
    // summed in warp order
    {
      double2 acc[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) acc[m] = make_double2(0.0, 0.0);
      for (int jb = warp; jb <= r; jb += 4 * W) {
        double2 mv[4][4];
        double cj[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int jc = jb + q * W;
          cj[q] = (jc < r) ? cvec[jc] : (jc == r ? -1.0 : 0.0);
          const double2* col = reinterpret_cast<const double2*>(mg + (jc <= r ? jc : r) * ld);
#pragma unroll
          for (int m = 0; m < 4; ++m)
            mv[q][m] = (lane + 32 * m < n2) ? __ldcg(col + lane + 32 * m) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            acc[m].x = fma(mv[q][m].x, cj[q], acc[m].x);
            acc[m].y = fma(mv[q][m].y, cj[q], acc[m].y);
          }
        }
      }
      double2* rb = reinterpret_cast<double2*>(A + warp * ld);
#pragma unroll
      for (int m = 0; m < 4; ++m)
        if (lane + 32 * m < n2) rb[lane + 32 * m] = acc[m];
    }
    for (int jj = tid; jj < r; jj += 32 * W) a.coef[p * r + jj] = cvec[jj];
    __syncthreads();
    double ss = 0.0;
    for (int i = tid; i < s; i += 32 * W) {
      double tot = A[i];
#pragma unroll
      for (int w = 1; w < W; ++w) tot += A[w * ld + i];
      tot *= ws[i];
      ss += tot * tot;
    }
    ss = warp_allreduce_d(ss);
    if (lane == 0) red[warp] = ss;
    __syncthreads();
    issue_next();
    if (tid == 0) {
      double tot = 0.0;
      for (int w = 0; w < W; ++w) tot += red[w];
      a.sres[p] = rankdef ? qnan : sqrt(tot);
      a.status[p] = rankdef ? 1 : 0;
      if (a.badcol) a.badcol[p] = rankdef ? (int)rinfo[1] : -1;
      if (a.outv) {
        double o = 0.0;
        if (a.proj)
          for (int jj = 0; jj < r; ++jj) o += a.proj[jj] * cvec[jj];
        a.outv[2 * p] = o;
        a.outv[2 * p + 1] = 0.0;
      }
    }
    __syncthreads();
    WY_PROF_MARK(7);
  }
#ifdef SAS_WY_PROF
  if (tid == 0 && blockIdx.x < 2)
    printf("wy_prof block %d: load %lld weights %lld panel(+lookahead S3) %lld S1 %lld S2 %lld S3 %lld backsub %lld "
           "residual %lld cycles (all p of the CTA)\n",
           blockIdx.x, wy_tp[0], wy_tp[1], wy_tp[2], wy_tp[3], wy_tp[4], wy_tp[5], wy_tp[6], wy_tp[7]);
#endif
}
