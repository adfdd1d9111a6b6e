// Leverage-score row selection on the GPU (replaces the dense
// part of subsample.select_rows' leverage branch, subsample.py:84-94, 124-134,
// 144-159): Q = A C for a tall A (m x w, row-major) and a small C (w x k), with
//   scores_i = || Q_i ||^2   (the leverage score of row i when Q is orthonormal)
// and, optionally, Q itself (m x k row-major) for the next TSQR pass.  The host
// side (offline.py) builds C from the TSQR R factor: R = U S V^H, C = V_k S_k^-1,
// then C <- C R2^-1 from the R factor of Q until Q is orthonormal to rounding.
//
// One CTA = 64 rows: the A tile and C sit in shared memory, a thread owns one
// row and every fourth group of four columns; the Q tile is staged through
// shared memory so that both global streams are contiguous.  Fixed summation
// order (the scores do not depend on the grid).
#pragma once
#include "sas_common.cuh"

constexpr int kSelRows = 64;

template <typename T>
__host__ __device__ inline size_t range_rows_smem_bytes(int w, int k) {
  return ((size_t)w * k + (size_t)kSelRows * (w + 1)) * sizeof(T) + 4 * kSelRows * sizeof(double);
}

template <typename T>
__global__ void __launch_bounds__(256) k_range_rows(const T* __restrict__ A, int64_t m, int w,
                                                    const T* __restrict__ C, int k, T* __restrict__ Q,
                                                    double* __restrict__ scores) {
  using S = Sc<T>;
  extern __shared__ __align__(16) unsigned char sel_smem[];
  T* Cs = reinterpret_cast<T*>(sel_smem);                  // w x k
  T* As = Cs + (size_t)w * k;                              // 64 x (w + 1); reused for the Q tile (64 x k)
  double* part = reinterpret_cast<double*>(As + (size_t)kSelRows * (w + 1));   // [4][64]
  const int tid = threadIdx.x;
  const int lda = w + 1;
  for (int e = tid; e < w * k; e += 256) Cs[e] = C[e];
  const int row = tid & (kSelRows - 1), cg = tid >> 6;
  for (int64_t r0 = (int64_t)blockIdx.x * kSelRows; r0 < m; r0 += (int64_t)gridDim.x * kSelRows) {
    const int nr = (int)((m - r0 < kSelRows) ? (m - r0) : kSelRows);
    __syncthreads();   // the previous tile's Q is out; Cs is in
    const T* src = A + r0 * w;
    for (int e = tid; e < nr * w; e += 256) {
      const int i = e / w, j = e - i * w;
      As[i * lda + j] = src[e];
    }
    __syncthreads();
    T acc[4][4];   // column groups cg, cg + 4, cg + 8, cg + 12 (k <= 64), four columns each
    double sc = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[q][c] = S::zero();
    if (row < nr) {
      const T* ar = As + row * lda;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c0 = 4 * (cg + 4 * q);
        if (c0 >= k) break;
        for (int j = 0; j < w; ++j) {
          const T a = ar[j];
          const T* cr = Cs + j * k + c0;
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (c0 + c < k) acc[q][c] = S::add(acc[q][c], S::mul(a, cr[c]));
        }
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (c0 + c < k) sc += S::abs2(acc[q][c]);
      }
    }
    part[cg * kSelRows + row] = sc;
    __syncthreads();   // every thread is done with the A tile
    if (Q && row < nr) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c0 = 4 * (cg + 4 * q);
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (c0 + c < k) As[row * k + c0 + c] = acc[q][c];
      }
    }
    if (scores && cg == 0 && row < nr)
      scores[r0 + row] = ((part[row] + part[kSelRows + row]) + part[2 * kSelRows + row]) + part[3 * kSelRows + row];
    if (Q) {
      __syncthreads();
      T* dst = Q + r0 * k;
      for (int e = tid; e < nr * k; e += 256) dst[e] = As[e];
    }
  }
}
