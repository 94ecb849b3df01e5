// Batched one-time operators on the GPU: for every subsystem
// the projector P_s = I - A'(AA')^{-1}A and the shift v_s = A'(AA')^{-1}b,
// with the reference's singularity guard (proj/src/admm.cpp:31-88).
//
// One thread per subsystem runs exactly the host restatement's sequence
// (csrc/host/admm_host.cpp project_one): Gram by sequential-k dot products,
// left-looking Cholesky, forward/back substitution per column of [A | b],
// P and v by sequential-k sums -- compiled with --fmad=false, IEEE division
// and sqrt, so P and v are bitwise identical to the host's (and therefore to
// the operators the CPU oracle iterates with). Scratch (G, L, X, y) lives in
// a per-subsystem slice of global memory.
#include <cuda_runtime.h>

#include <cstdint>

#include "precompute_kernels.cuh"

namespace dopf::cuda {

namespace {

__global__ void k_precompute(PrecomputeParams p) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= p.S) return;
  const int off = p.z_offsets[s];
  const int n = p.z_offsets[s + 1] - off;
  const int m = p.m_s[s];
  double* P = p.P + p.p_offsets[s];
  double* v = p.v + off;
  p.singular[s] = 0;
  if (m == 0) {
    for (int i = 0; i < n; ++i) {
      for (int j = 0; j < n; ++j) P[i * n + j] = i == j ? 1.0 : 0.0;
      v[i] = 0.0;
    }
    return;
  }
  const double* A = p.A + p.a_offsets[s];  // row-major m x n
  const double* b = p.b + p.b_offsets[s];
  double* G = p.scratch + p.scratch_offsets[s];  // m x m
  double* L = G + m * m;                          // m x m
  double* X = L + m * m;                          // m x n
  double* y = X + m * n;                          // m
  for (int i = 0; i < m; ++i)
    for (int j = 0; j <= i; ++j) {
      double acc = 0.0;
      for (int k = 0; k < n; ++k) acc += A[i * n + k] * A[j * n + k];
      G[i * m + j] = acc;
      G[j * m + i] = acc;
    }
  for (int i = 0; i < m * m; ++i) L[i] = 0.0;
  for (int k = 0; k < m; ++k) {
    double d = G[k * m + k];
    for (int q = 0; q < k; ++q) d -= L[k * m + q] * L[k * m + q];
    if (!(d > 0.0)) {
      p.singular[s] = 1;
      return;
    }
    const double lkk = sqrt(d);
    L[k * m + k] = lkk;
    for (int i = k + 1; i < m; ++i) {
      double acc = G[i * m + k];
      for (int q = 0; q < k; ++q) acc -= L[i * m + q] * L[k * m + q];
      L[i * m + k] = acc / lkk;
    }
  }
  double dmin = L[0], dmax = L[0];
  for (int k = 1; k < m; ++k) {
    const double d = L[k * m + k];
    dmin = (d < dmin) ? d : dmin;  // std::min
    dmax = (dmax < d) ? d : dmax;  // std::max
  }
  if (!(dmin > 0.0) || (dmin / dmax) * (dmin / dmax) < 1e-14) {
    p.singular[s] = 1;
    return;
  }
  auto solve_in_place = [&](double* col) {
    for (int i = 0; i < m; ++i) {
      double acc = col[i];
      for (int q = 0; q < i; ++q) acc -= L[i * m + q] * col[q];
      col[i] = acc / L[i * m + i];
    }
    for (int i = m - 1; i >= 0; --i) {
      double acc = col[i];
      for (int q = i + 1; q < m; ++q) acc -= L[q * m + i] * col[q];
      col[i] = acc / L[i * m + i];
    }
  };
  for (int j = 0; j < n; ++j) {
    for (int i = 0; i < m; ++i) y[i] = A[i * n + j];
    solve_in_place(y);
    for (int i = 0; i < m; ++i) X[i * n + j] = y[i];
  }
  for (int i = 0; i < m; ++i) y[i] = b[i];
  solve_in_place(y);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int k = 0; k < m; ++k) acc += A[k * n + i] * X[k * n + j];
      P[i * n + j] = (i == j ? 1.0 : 0.0) - acc;
    }
  for (int i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int k = 0; k < m; ++k) acc += A[k * n + i] * y[k];
    v[i] = acc;
  }
}

}  // namespace

cudaError_t launch_precompute(const PrecomputeParams& p, cudaStream_t stream) {
  const int threads = 128;
  k_precompute<<<(p.S + threads - 1) / threads, threads, 0, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace dopf::cuda
