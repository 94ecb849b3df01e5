// One-time operators on the GPU, batched over every subsystem
// of any number of models (a scenario batch is one launch per stage):
//
//  k_row_reduce -- reference decompose.cpp:48-98, one warp per subsystem.
//     [A | b] in shared memory. Pivot = the first strict maximum |entry| of
//     the remaining rows in row-major scan order (> tol): every lane keeps
//     the first strict maximum of its own strided subsequence, then a warp
//     argmax prefers the larger magnitude and, on equal magnitudes, the
//     smaller scan index -- the same entry the sequential scan picks. Row
//     swap, division of the pivot row by the pivot (exact 1.0 written),
//     elimination below with the factors read before any row changes (exact
//     0.0 written), the zeroed rank-deficient tail, the rhs consistency check
//     and the |v| <= tol clean-up: every element sees the host restatement's
//     (csrc/host/decompose.cpp row_reduce) operations in the same order.
//
//  k_project -- reference admm.cpp:31-88, one CTA per subsystem, work in
//     shared memory: Gram entries (one thread per entry, sequential k),
//     left-looking Cholesky (the pivot on one thread, the column below it
//     one thread per row, sequential p), the reference's singularity guard,
//     forward / back substitution one thread per right-hand side ([A | b]
//     columns), P and v one thread per entry (sequential k). Each value is
//     the host restatement's (csrc/host/admm_host.cpp project_one) sequence
//     of IEEE operations -- --fmad=false, IEEE division and square root --
//     so P and v are bitwise the host's, hence bitwise the operators the
//     CPU oracle iterates with.
//
// Subsystems larger than shared memory run the same code on a slice of
// global scratch.
#include <cuda_runtime.h>

#include <cstdint>

#include "precompute_kernels.cuh"

namespace dopf::cuda {

namespace {

constexpr int kProjectThreads = 128;

__global__ void __launch_bounds__(32) k_row_reduce(PrepParams p) {
  extern __shared__ __align__(16) double smem[];
  const int64_t s = blockIdx.x;
  if (s >= p.count) return;
  const PrepSub d = p.subs[s];
  const int m = d.m, n = d.n, w = n + 1;
  const int lane = threadIdx.x;
  double* A = p.A + d.a_off;
  double* b = p.b + d.b_off;
  if (m == 0) {
    if (lane == 0) {
      p.rank[s] = 0;
      p.status[s] = kPrepOk;
    }
    return;
  }
  double* work = p.scratch_off ? p.scratch + p.scratch_off[s] : smem;  // m x (n+1)
  double* fac = work + static_cast<int64_t>(m) * w;                   // m
  for (int k = lane; k < m * w; k += 32) {
    const int i = k / w, j = k - i * w;
    work[k] = j < n ? A[static_cast<int64_t>(i) * n + j] : b[i];
  }
  __syncwarp();
  const double tol = p.tol;
  int rank = 0;
  while (rank < m) {
    // first strict maximum of |work| over rows [rank, m) x columns [0, n)
    double best = tol;
    int bidx = -1;
    const int cnt = (m - rank) * n;
    for (int q = lane; q < cnt; q += 32) {
      const int i = rank + q / n, j = q % n;
      const double mag = fabs(work[i * w + j]);
      if (mag > best) {
        best = mag;
        bidx = q;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bidx, off);
      // larger magnitude wins; equal magnitudes: the earlier scan position
      // (-1 = no candidate, only ever paired with best == tol)
      const unsigned mine = static_cast<unsigned>(bidx), theirs = static_cast<unsigned>(oi);
      if (ob > best || (ob == best && theirs < mine)) {
        best = ob;
        bidx = oi;
      }
    }
    if (bidx < 0) break;  // every remaining row is zero within tol
    const int prow = rank + bidx / n, pcol = bidx % n;
    if (prow != rank)
      for (int j = lane; j < w; j += 32) {
        const double t = work[rank * w + j];
        work[rank * w + j] = work[prow * w + j];
        work[prow * w + j] = t;
      }
    __syncwarp();
    const double pivot = work[rank * w + pcol];
    __syncwarp();
    for (int j = lane; j < w; j += 32) work[rank * w + j] = work[rank * w + j] / pivot;
    __syncwarp();
    if (lane == 0) work[rank * w + pcol] = 1.0;
    for (int i = rank + 1 + lane; i < m; i += 32) fac[i] = work[i * w + pcol];
    __syncwarp();
    const int below = (m - rank - 1) * w;
    for (int q = lane; q < below; q += 32) {
      const int i = rank + 1 + q / w, j = q % w;
      const double f = fac[i];
      if (f != 0.0) work[i * w + j] = work[i * w + j] - f * work[rank * w + j];
    }
    __syncwarp();
    for (int i = rank + 1 + lane; i < m; i += 32)
      if (fac[i] != 0.0) work[i * w + pcol] = 0.0;
    __syncwarp();
    ++rank;
  }
  bool bad = false;
  for (int i = rank + lane; i < m; i += 32)
    if (fabs(work[i * w + n]) > tol) bad = true;
  bad = __any_sync(0xffffffffu, bad);
  for (int q = lane; q < rank * n; q += 32) {
    const int i = q / n, j = q - i * n;
    const double v = work[i * w + j];
    A[q] = fabs(v) <= tol ? 0.0 : v;
  }
  for (int i = lane; i < rank; i += 32) b[i] = work[i * w + n];
  if (lane == 0) {
    p.rank[s] = rank;
    p.status[s] = bad ? kPrepInfeasible : kPrepOk;
  }
}

__global__ void __launch_bounds__(kProjectThreads) k_project(PrepParams p) {
  extern __shared__ __align__(16) double smem[];
  __shared__ int fail;
  const int64_t s = blockIdx.x;
  if (s >= p.count) return;
  const PrepSub d = p.subs[s];
  const int m = p.rank[s], n = d.n, tid = threadIdx.x;
  double* P = p.P + d.p_off;
  double* v = p.v + d.v_off;
  if (m == 0) {  // no equality rows: the kernel is everything
    for (int k = tid; k < n * n; k += kProjectThreads) P[k] = (k / n == k % n) ? 1.0 : 0.0;
    for (int i = tid; i < n; i += kProjectThreads) v[i] = 0.0;
    if (tid == 0) p.status[s] = kPrepOk;
    return;
  }
  double* A = p.scratch_off ? p.scratch + p.scratch_off[s] : smem;  // m x n
  double* G = A + m * n;                                             // m x m
  double* L = G + m * m;                                             // m x m
  double* X = L + m * m;                                             // m x (n+1): G^{-1} [A | b]
  const int w = n + 1;
  const double* gA = p.A + d.a_off;
  const double* gb = p.b + d.b_off;
  for (int k = tid; k < m * n; k += kProjectThreads) A[k] = gA[k];
  for (int k = tid; k < m * w; k += kProjectThreads) {
    const int i = k / w, j = k - i * w;
    X[k] = j < n ? gA[i * n + j] : gb[i];
  }
  if (tid == 0) fail = 0;
  __syncthreads();
  // G = A A' (lower triangle, mirrored)
  const int pairs = m * (m + 1) / 2;
  for (int q = tid; q < pairs; q += kProjectThreads) {
    int i = static_cast<int>((sqrt(8.0 * q + 1.0) - 1.0) * 0.5);
    while (i * (i + 1) / 2 > q) --i;
    while ((i + 1) * (i + 2) / 2 <= q) ++i;
    const int j = q - i * (i + 1) / 2;
    double acc = 0.0;
    for (int k = 0; k < n; ++k) acc = acc + A[i * n + k] * A[j * n + k];
    G[i * m + j] = acc;
    G[j * m + i] = acc;
  }
  __syncthreads();
  // left-looking Cholesky
  for (int k = 0; k < m; ++k) {
    if (tid == 0) {
      double dk = G[k * m + k];
      for (int q = 0; q < k; ++q) dk = dk - L[k * m + q] * L[k * m + q];
      if (!(dk > 0.0)) fail = 1;
      else L[k * m + k] = sqrt(dk);
    }
    __syncthreads();
    if (fail) break;
    const double lkk = L[k * m + k];
    for (int i = k + 1 + tid; i < m; i += kProjectThreads) {
      double acc = G[i * m + k];
      for (int q = 0; q < k; ++q) acc = acc - L[i * m + q] * L[k * m + q];
      L[i * m + k] = acc / lkk;
    }
    __syncthreads();
  }
  if (!fail && tid == 0) {
    double dmin = L[0], dmax = L[0];
    for (int k = 1; k < m; ++k) {
      const double dk = L[k * m + k];
      dmin = (dk < dmin) ? dk : dmin;  // std::min
      dmax = (dmax < dk) ? dk : dmax;  // std::max
    }
    if (!(dmin > 0.0) || (dmin / dmax) * (dmin / dmax) < 1e-14) fail = 1;
  }
  __syncthreads();
  if (fail) {
    if (tid == 0) p.status[s] = kPrepSingular;
    return;
  }
  // G^{-1} [A | b]: one right-hand side per thread, L y = rhs then L' x = y
  for (int j = tid; j < w; j += kProjectThreads) {
    for (int i = 0; i < m; ++i) {
      double acc = X[i * w + j];
      for (int q = 0; q < i; ++q) acc = acc - L[i * m + q] * X[q * w + j];
      X[i * w + j] = acc / L[i * m + i];
    }
    for (int i = m - 1; i >= 0; --i) {
      double acc = X[i * w + j];
      for (int q = i + 1; q < m; ++q) acc = acc - L[q * m + i] * X[q * w + j];
      X[i * w + j] = acc / L[i * m + i];
    }
  }
  __syncthreads();
  // P = I - A' G^{-1} A, v = A' G^{-1} b
  for (int q = tid; q < n * n; q += kProjectThreads) {
    const int i = q / n, j = q - i * n;
    double acc = 0.0;
    for (int k = 0; k < m; ++k) acc = acc + A[k * n + i] * X[k * w + j];
    P[q] = (i == j ? 1.0 : 0.0) - acc;
  }
  for (int i = tid; i < n; i += kProjectThreads) {
    double acc = 0.0;
    for (int k = 0; k < m; ++k) acc = acc + A[k * n + i] * X[k * w + n];
    v[i] = acc;
  }
  if (tid == 0) p.status[s] = kPrepOk;
}

cudaError_t launch_grid(const void* fn, int threads, const PrepParams& p, int64_t smem_words,
                        cudaStream_t stream) {
  const std::size_t smem = static_cast<std::size_t>(smem_words) * sizeof(double);
  cudaError_t err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
  if (err != cudaSuccess) return err;
  PrepParams local = p;
  void* args[] = {&local};
  // one CTA per subsystem; grids beyond 2^31 - 1 do not occur (int32 S per model)
  return cudaLaunchKernel(fn, dim3(static_cast<unsigned>(p.count)), dim3(threads), args, smem, stream);
}

}  // namespace

cudaError_t launch_row_reduce(const PrepParams& p, int64_t smem_words, cudaStream_t stream) {
  if (p.count == 0) return cudaSuccess;
  return launch_grid(reinterpret_cast<const void*>(&k_row_reduce), 32, p, smem_words, stream);
}

cudaError_t launch_project(const PrepParams& p, int64_t smem_words, cudaStream_t stream) {
  if (p.count == 0) return cudaSuccess;
  return launch_grid(reinterpret_cast<const void*>(&k_project), kProjectThreads, p, smem_words, stream);
}

}  // namespace dopf::cuda
