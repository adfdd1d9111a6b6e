// K3: Gaussian-kernel row contraction for a batch of bandwidths p.
//
//   M_p[i][j] = sum_l E_p(i,l) X[l][j],
//   E_p(i,l)  = exp(-(D[i][l] * inv_p)) (+ lam if l == S_i),  inv_p = 1/(2 sigma^2)
//   p = sigma with a plan ridge lam, or p = (lam, sigma) as in the reference's
//   KRR system (systems.py:423-463)
//
// This is what the reference computes per p with the dense detour
//   online._sampled_rows -> rows_dense -> row_fn -> @ basis.basis
// (online.py:57-65, systems.py:151-162, _kernels.py:38-50 for the 1-D rbf_rows;
// the ridge is added to the kernel entry before the product, as `out[k, i] += lam`
// in _kernels.py:49).  D = squared distances of the s selected points to all n
// points (p-independent, built once per plan by k_gauss_dist), so only the exp
// and the contraction are per p.
//
// GEMM view per CTA: rows (p, i) for PW parameter values x all s rows, columns
// = basis columns (8*NT >= r), K = n.  One warp owns an 8-row group i0..i0+7
// for PW parameters; per k-step of 4 each lane evaluates PW exps (A-fragment
// element of mma.m8n8k4: row lane/4, col lane%4) and issues PW*NT DMMA
// (mma.sync.m8n8k4.f64, SASS DMMA.8x8x4 — the only FP64 tensor shape on sm_100a;
// FP64 has no tcgen05 kind).  D and X fragments stream through a 3-stage
// shared-memory ring filled by bulk async copies (below) and are reused by all
// PW parameters of the CTA.  The exp is sas_exp64_t2k_fast (5 FP64-pipe ops and
// ~10 integer/FP32 instructions; CTAs whose arguments could underflow use the
// masked sas_exp64_t2k_fr); DMMA and DFMA share one FP64 pipe on B200
// (profiles/r01_fp64_peaks.jsonl).  Split-K over n (grid.z) removes the
// partial last wave (1024 CTAs on 296 slots -> 2048 on 296).
#pragma once
#include "sas_common.cuh"

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// D[i][l] = sum_k (x_{S_i,k} - x_{l,k})^2, sequential over k, no FMA
// (the harness row oracle's order, oracle/online_ref.py gauss_rows).
__global__ void k_gauss_dist(const double* __restrict__ pts, const int64_t* __restrict__ S,
                             int64_t n, int d, int s, int64_t ld, double* __restrict__ D) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)s * n) return;
  int i = (int)(idx / n);
  int64_t l = idx - (int64_t)i * n;
  const double* xi = pts + S[i] * d;
  const double* xl = pts + l * d;
  double acc = 0.0;
  for (int k = 0; k < d; ++k) {
    double df = __dsub_rn(xi[k], xl[k]);
    acc = __dadd_rn(acc, __dmul_rn(df, df));
  }
  D[(int64_t)i * ld + l] = acc;
}

#ifndef K3_KC
#define K3_KC 32
#endif
#ifndef K3_STAGES
#define K3_STAGES 3
#endif
constexpr int kGaussKC = K3_KC;         // K chunk (columns l) per pipeline stage
constexpr int kGaussMaxWarps = 10;      // row groups (8 rows each) per CTA -> 320 threads
constexpr int kGaussMaxSplit = 2;       // split-K partial products (M scratch is sized for this many)
// parameter values per CTA: keep PW*NT*2 accumulator doubles <= 24 (2 CTAs/SM)
template <int NT>
__host__ __device__ constexpr int gauss_pw() { return NT <= 3 ? 4 : (NT == 4 ? 3 : (NT <= 6 ? 2 : 1)); }

// Row blocking of the s selected rows: gy CTAs along grid.y with rows_cta rows
// each, at most maxw 8-row groups (warps) per CTA (a plan property: the
// fragment-ordered D is packed per row block).
__host__ __device__ inline void gauss_row_blocks(int s, int maxw, int* gy, int* rows_cta) {
  const int s_pad = ((s + 7) / 8) * 8;
  *gy = (s_pad + 8 * maxw - 1) / (8 * maxw);
  *rows_cta = 8 * ((s_pad / 8 + *gy - 1) / *gy);
}

// ===========================================================================
// Fragment-ordered operands streamed with bulk async copies.
//
// Plan-time layouts put every DMMA fragment a warp needs for one k-step in 32
// consecutive doubles (lane order), so a pipeline stage is two contiguous
// blocks (the CTA's D fragments and the X^T fragments of one K chunk):
//   Dfrag[rb][ch][g][ks][lane] = D[rb*rows_cta + 8g + lane/4][ch*KC + 4ks + lane%4] * 2048/ln2
//   Xfrag[ch][t][ks][lane]     = X[ch*KC + 4ks + lane%4][8t + lane/4]
// One thread issues cp.async.bulk (SASS UBLKCP) per stage with an mbarrier
// transaction count; warps wait on the stage's full barrier and release it
// through an empty barrier, so there is no CTA-wide __syncthreads in the loop
// and fragment reads are conflict-free (lane-contiguous 8-byte loads).
// ===========================================================================
#ifndef K3_UNROLL
#define K3_UNROLL 4
#endif
constexpr int kK3Unroll = K3_UNROLL;  // k-steps unrolled per loop iteration
constexpr int kG3Stages = K3_STAGES;
constexpr int kG3KS = kGaussKC / 4;  // k-steps per chunk

// max of non-negative doubles (their bit patterns order like the values)
__global__ void k_max_nonneg(const double* __restrict__ v, int64_t n, unsigned long long* __restrict__ out) {
  unsigned long long m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, (unsigned long long)__double_as_longlong(v[i]));
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

__global__ void k_gauss_pack_dfrag(const double* __restrict__ D, int64_t ldd, int s, int64_t n, int gy,
                                   int rows_cta, int64_t nchunks, double* __restrict__ Df) {
  const int nrg = rows_cta / 8;
  const int64_t tot = (int64_t)gy * nchunks * nrg * kG3KS * 32;
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= tot) return;
  int lane = (int)(idx & 31);
  int64_t rest = idx >> 5;
  int ks = (int)(rest % kG3KS); rest /= kG3KS;
  int g = (int)(rest % nrg); rest /= nrg;
  int64_t ch = rest % nchunks;
  int rb = (int)(rest / nchunks);
  int row = rb * rows_cta + 8 * g + (lane >> 2);
  int64_t l = ch * kGaussKC + 4 * ks + (lane & 3);
  // pre-scaled by 2048/ln2: the exponential takes its argument in table units
  Df[idx] = (row < s && l < n) ? D[(int64_t)row * ldd + l] * SAS_INVLN2X2K : 0.0;
}

__global__ void k_gauss_pack_xfrag(const double* __restrict__ X, int64_t n, int r, int nt, int64_t nchunks,
                                   double* __restrict__ Xf) {
  const int64_t tot = nchunks * nt * kG3KS * 32;
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= tot) return;
  int lane = (int)(idx & 31);
  int64_t rest = idx >> 5;
  int ks = (int)(rest % kG3KS); rest /= kG3KS;
  int t = (int)(rest % nt);
  int64_t ch = rest / nt;
  int64_t l = ch * kGaussKC + 4 * ks + (lane & 3);
  int c = 8 * t + (lane >> 2);
  Xf[idx] = (c < r && l < n) ? X[l * r + c] : 0.0;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Shared memory: the stage ring, the negated exp table (2048) and the negated
// diagonal entries -(1 + lam_u), then the mbarriers.
constexpr int kGaussTabDoubles = 2048 + 16;
template <int NT>
__host__ __device__ constexpr size_t gauss3_smem_bytes(int rows_cta) {
  return (size_t)kG3Stages * (rows_cta / 8 + NT) * kG3KS * 32 * sizeof(double) + kGaussTabDoubles * sizeof(double) +
         2 * kG3Stages * sizeof(uint64_t);
}

// Exponentials: CTAs whose largest argument stays above -677 (dmax = max D in
// table units, times the CTA's largest 1/(2 sigma^2)) use sas_exp64_t2k_fast
// and add the kernel ridge after the contraction (M += lam X[S_i]); the others
// use the masked sas_exp64_t2k_fr with the ridge folded into the diagonal
// entry (the reference's exp(-0) + lam, _kernels.py:49).
// Split-K: grid.z splits the n chunks into gridDim.z contiguous ranges whose
// partial products go to Mout + z * msplit; K4 sums them in z order.
template <int NT, int PW, int MINB, int MAXW, int MODE = 0>
__global__ void __launch_bounds__(32 * MAXW, MINB)
k_gauss_rows(const double* __restrict__ Df, const double* __restrict__ Xf, const int64_t* __restrict__ S,
             const double* __restrict__ params, int dp, int64_t P, int s, int64_t nchunks, int r, double ridge,
             double* __restrict__ Mout, int64_t msplit, double dmax, const double* __restrict__ X) {
  // parameter value = bandwidth sigma (dp == 1, plan ridge) or (lambda, sigma)
  // (dp == 2, the reference's KRR system, systems.py:423-463)
  const int64_t pbase = (int64_t)blockIdx.x * PW;
  double ninv[PW];
  float ninvf[PW];
  double bmax = 0.0;
#pragma unroll
  for (int u = 0; u < PW; ++u) {
    const int64_t p = pbase + u;
    const double sg = (p < P) ? params[p * dp + dp - 1] : 1.0;
    ninv[u] = -(1.0 / (2.0 * sg * sg));  // reference: inv = 1.0 / (2.0 * sigma * sigma)
    ninvf[u] = (float)ninv[u];
    bmax = fmax(bmax, -ninv[u]);
  }
  // MODE 0: both paths; 1: fast CTAs only (others return); 2: masked CTAs only.
  // Decided before any bulk copy is issued.
  const bool fast = dmax * bmax < SAS_EXP2K_FAST_MAX;
  if ((MODE == 1 && !fast) || (MODE == 2 && fast)) return;
  extern __shared__ __align__(128) double gsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nrg = blockDim.x >> 5;            // row groups = warps
  const int rows_cta = nrg * 8;
  const int row0 = blockIdx.y * rows_cta;
  const int stage_d = (nrg + NT) * kG3KS * 32;  // doubles per stage
  double* ring = gsm;
  double* tabn = gsm + (size_t)kG3Stages * stage_d;  // -2^(j/2048), then -(1 + lam_u)
  uint64_t* full = reinterpret_cast<uint64_t*>(tabn + kGaussTabDoubles);
  uint64_t* empty = full + kG3Stages;
  const unsigned dbytes = (unsigned)(nrg * kG3KS * 32 * sizeof(double));
  const unsigned xbytes = (unsigned)(NT * kG3KS * 32 * sizeof(double));
  const double* dsrc = Df + (int64_t)blockIdx.y * nchunks * nrg * kG3KS * 32;

  if (threadIdx.x == 0) {
    for (int b = 0; b < kG3Stages; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], nrg);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int j = threadIdx.x; j < 2048; j += blockDim.x) tabn[j] = -g_exp2_tab2048[j];
  __syncthreads();

  const int64_t c0 = nchunks * blockIdx.z / gridDim.z, nloc = nchunks * (blockIdx.z + 1) / gridDim.z - c0;
  Mout += blockIdx.z * msplit;
  auto issue = [&](int64_t j) {  // local chunk j = chunk c0 + j into slot j mod stages
    const int b = (int)(j % kG3Stages);
    if (j >= kG3Stages) mbar_wait(&empty[b], (unsigned)(((j / kG3Stages) - 1) & 1));
    double* dst = ring + (size_t)b * stage_d;
    const int64_t ch = c0 + j;
    mbar_expect_tx(&full[b], dbytes + xbytes);
    bulk_g2s(dst, dsrc + ch * (int64_t)nrg * kG3KS * 32, dbytes, &full[b]);
    bulk_g2s(dst + nrg * kG3KS * 32, Xf + ch * (int64_t)NT * kG3KS * 32, xbytes, &full[b]);
  };
  if (threadIdx.x == 0)
    for (int64_t j = 0; j < kG3Stages - 1 && j < nloc; ++j) issue(j);

  auto lam_of = [&](int u) {
    const int64_t p = pbase + u;
    return (dp == 2) ? ((p < P) ? params[p * 2] : 0.0) : ridge;
  };
  if (threadIdx.x < PW) tabn[2048 + threadIdx.x] = -(1.0 + lam_of(threadIdx.x));
  __syncthreads();
  const int grow = row0 + warp * 8 + (lane >> 2);
  const int64_t srow = (grow < s) ? S[grow] : -1;

  double acc[PW][NT][2];
#pragma unroll
  for (int u = 0; u < PW; ++u)
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[u][t][0] = acc[u][t][1] = 0.0;

  if (MODE == 1 || (MODE == 0 && fast)) {
    for (int64_t j = 0; j < nloc; ++j) {
      if (threadIdx.x == 0 && j + kG3Stages - 1 < nloc) issue(j + kG3Stages - 1);
      const int b = (int)(j % kG3Stages);
      mbar_wait(&full[b], (unsigned)((j / kG3Stages) & 1));
      const double* dsb = ring + (size_t)b * stage_d + warp * kG3KS * 32 + lane;
      const double* xsb = ring + (size_t)b * stage_d + nrg * kG3KS * 32 + lane;
#pragma unroll kK3Unroll
      for (int ks = 0; ks < kG3KS; ++ks) {
        const double dv = dsb[ks * 32];
        double bf[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) bf[t] = xsb[(t * kG3KS + ks) * 32];
#pragma unroll
        for (int u = 0; u < PW; ++u) {
          const double e = sas_exp64_t2k_fast(dv, ninv[u], ninvf[u], tabn);
#pragma unroll
          for (int t = 0; t < NT; ++t) dmma884(acc[u][t][0], acc[u][t][1], e, bf[t]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[b]);
    }
    // the kernel-row ridge: M_p += lam_p X[S_i, :] (split 0 only)
    if (blockIdx.z == 0 && grow < s) {
      const double* xrow = X + srow * (int64_t)r;
#pragma unroll
      for (int u = 0; u < PW; ++u) {
        const double lam = lam_of(u);
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int c0c = t * 8 + 2 * (lane & 3);
          if (c0c < r) acc[u][t][0] = fma(lam, xrow[c0c], acc[u][t][0]);
          if (c0c + 1 < r) acc[u][t][1] = fma(lam, xrow[c0c + 1], acc[u][t][1]);
        }
      }
    }
  } else {
    for (int64_t j = 0; j < nloc; ++j) {
      if (threadIdx.x == 0 && j + kG3Stages - 1 < nloc) issue(j + kG3Stages - 1);
      const int b = (int)(j % kG3Stages);
      mbar_wait(&full[b], (unsigned)((j / kG3Stages) & 1));
      const int64_t ch = c0 + j;
      const double* dsb = ring + (size_t)b * stage_d + warp * kG3KS * 32 + lane;
      const double* xsb = ring + (size_t)b * stage_d + nrg * kG3KS * 32 + lane;
      const int64_t l0 = ch * kGaussKC;
      const int dcol = (srow >= l0 && srow < l0 + kGaussKC) ? (int)(srow - l0) : -1;
#pragma unroll kK3Unroll
      for (int ks = 0; ks < kG3KS; ++ks) {
        const double dv = dsb[ks * 32];
        double bf[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) bf[t] = xsb[(t * kG3KS + ks) * 32];
        const bool diag = (4 * ks + (lane & 3)) == dcol;
#pragma unroll
        for (int u = 0; u < PW; ++u) {
          const double e = sas_exp64_t2k_fr(dv, ninv[u], ninvf[u], tabn, diag ? 2048 + u : -1);
#pragma unroll
          for (int t = 0; t < NT; ++t) dmma884(acc[u][t][0], acc[u][t][1], e, bf[t]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[b]);
    }
  }
  if (grow < s) {
#pragma unroll
    for (int u = 0; u < PW; ++u) {
      const int64_t p = pbase + u;
      if (p >= P) continue;
      double* out = Mout + (p * s + grow) * (int64_t)r;
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const int c0c = t * 8 + 2 * (lane & 3);
        if (c0c < r) out[c0c] = acc[u][t][0];
        if (c0c + 1 < r) out[c0c + 1] = acc[u][t][1];
      }
    }
  }
}
