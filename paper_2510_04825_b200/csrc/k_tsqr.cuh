// TSQR: R factor of a tall m x w matrix (w <= 64), real or complex, by a tree
// of block Householder QRs -- the full least squares of solve_apsnap
// (reference online.py:156-165: linalg.solve_ls on B = A(p) Q_X, n x r') and
// the range basis of the leverage selector (subsample.py:144-159: thin SVD of
// the n x (r'+1) anchor matrix, whose R the host then decomposes).
//
// Level 0 splits the rows into blocks of MB = 32 RA rows; one CTA factors a
// block in shared memory with the Householder steps of k_lsq_sm (column-major,
// zero-padded rows, warp 0 forms reflector k+1 while the other warps update the
// trailing columns) and writes its w x w upper-triangular R (zero rows where
// the block has fewer than w rows).  Level L+1 runs the same kernel on the
// stacked R blocks of level L until one block remains.  Householder QR of
// the blocks is backward stable, so R matches the reference's np.linalg.qr R
// up to the signs of its rows and rounding.
#pragma once
#include "k_lsq_sm.cuh"

__host__ __device__ inline size_t tsqr_smem_bytes(int RA, int w, size_t esz) {
  const size_t n = (size_t)lsq_sm_lda(RA) * w + (size_t)w + 2;  // A, R_kk, v heads
  return (n * esz + 15) / 16 * 16 + (2 + 64) * sizeof(double);
}

// in: m x w row-major (ld = w); out: nblocks x w x w row-major.
template <typename T, int RA, int W>
__global__ void __launch_bounds__(32 * W) k_tsqr_block(const T* __restrict__ in, int64_t m, int w,
                                                       T* __restrict__ out) {
  using S = Sc<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int MB = 32 * RA;
  const int lda = lsq_sm_lda(RA);
  T* A = reinterpret_cast<T*>(smem_raw);
  T* rdiag = A + (size_t)lda * w;
  T* vk_s = rdiag + w;
  const size_t tb = (((size_t)lda * w + (size_t)w + 2) * sizeof(T) + 15) / 16 * 16;
  double* tau_s = reinterpret_cast<double*>(smem_raw + tb);
  double* nrm_s = tau_s + 2;
  SmShared sh{vk_s, tau_s, rdiag, nrm_s};

  const int64_t row0 = (int64_t)blockIdx.x * MB;
  const int mb = (int)((m - row0) < MB ? (m - row0) : MB);
  for (int idx = threadIdx.x; idx < lda * w; idx += blockDim.x) A[idx] = S::zero();
  __syncthreads();
  const T* src = in + row0 * w;
  for (int idx = threadIdx.x; idx < mb * w; idx += blockDim.x) {
    const int i = idx / w, j = idx - i * w;
    A[(size_t)j * lda + i] = src[idx];
  }
  __syncthreads();
  const int kmax = mb < w ? mb : w;
  if (warp == 0 && kmax > 0) {
    T y[RA];
    sm_load_col<T, RA>(y, A, lane);
    sm_reflector<T, RA>(y, 0, mb, lane, sh);
  }
  __syncthreads();
  for (int k = 0; k < kmax; ++k) {
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
      if (k + 1 < w) {
        T y[1][RA];
        T* col = A + (size_t)(k + 1) * lda;
        sm_load_col<T, RA>(y[0], col, lane);
        sm_apply<T, RA, 1>(y, v, tau);
        sm_store_col<T, RA>(y[0], col, lane);
        if (k + 1 < kmax) sm_reflector<T, RA>(y[0], k + 1, mb, lane, sh);
      }
    } else {
      int j = k + 1 + warp;
      for (; j + (W - 1) < w; j += 2 * (W - 1)) {
        T y[2][RA];
        T* c0 = A + (size_t)j * lda;
        T* c1 = A + (size_t)(j + W - 1) * lda;
        sm_load_col<T, RA>(y[0], c0, lane);
        sm_load_col<T, RA>(y[1], c1, lane);
        sm_apply<T, RA, 2>(y, v, tau);
        sm_store_col<T, RA>(y[0], c0, lane);
        sm_store_col<T, RA>(y[1], c1, lane);
      }
      if (j < w) {
        T y[1][RA];
        T* c0 = A + (size_t)j * lda;
        sm_load_col<T, RA>(y[0], c0, lane);
        sm_apply<T, RA, 1>(y, v, tau);
        sm_store_col<T, RA>(y[0], c0, lane);
      }
    }
    __syncthreads();
  }
  T* dst = out + (int64_t)blockIdx.x * w * w;
  for (int idx = threadIdx.x; idx < w * w; idx += blockDim.x) {
    const int i = idx / w, j = idx - i * w;
    T val = S::zero();
    if (i < kmax) val = (j > i) ? A[(size_t)j * lda + i] : (j == i ? rdiag[i] : S::zero());
    dst[idx] = val;
  }
}
