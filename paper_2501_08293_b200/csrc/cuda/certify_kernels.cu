// Post-solve certification on the GPU (reference
// proj/src/oracle.cpp:10-43 check_feasibility, :275-292
// reconstruct_centralized), for models too large to check comfortably on the
// host (the tiled feeder):
//  * ||A x - b||_inf over the centralized LP (row-per-thread sequential sums,
//    the same order as the host check), worst row = first maximum;
//  * bound violation max(lo - x, x - hi, 0), worst column = first maximum;
//  * copy-average reconstruction: per column the sum of its copies in
//    ascending s, divided by the copy count, clamped to the bounds.
#include <cuda_runtime.h>

#include <cstdint>

#include "certify_kernels.cuh"

namespace dopf::cuda {

namespace {

constexpr int kT = 256;

struct MaxIdx {
  double v;
  int32_t i;
};

__device__ __forceinline__ MaxIdx better(MaxIdx a, MaxIdx b) {
  // larger value wins; ties go to the lower index (the host's strict '>' scan)
  if (b.v > a.v || (b.v == a.v && b.i >= 0 && (a.i < 0 || b.i < a.i))) return b;
  return a;
}

__device__ MaxIdx block_best(MaxIdx m) {
  __shared__ double sv[kT / 32];
  __shared__ int32_t si[kT / 32];
  for (int off = 16; off > 0; off >>= 1) {
    MaxIdx o{__shfl_xor_sync(0xffffffffu, m.v, off), __shfl_xor_sync(0xffffffffu, m.i, off)};
    m = better(m, o);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    sv[warp] = m.v;
    si[warp] = m.i;
  }
  __syncthreads();
  if (warp == 0) {
    m = lane < kT / 32 ? MaxIdx{sv[lane], si[lane]} : MaxIdx{0.0, -1};
    for (int off = 16; off > 0; off >>= 1) {
      MaxIdx o{__shfl_xor_sync(0xffffffffu, m.v, off), __shfl_xor_sync(0xffffffffu, m.i, off)};
      m = better(m, o);
    }
  }
  return m;
}

__global__ void k_rows(CertifyParams p) {
  const int i = blockIdx.x * kT + threadIdx.x;
  MaxIdx m{0.0, -1};
  if (i < p.rows) {
    double s = 0.0;
    for (int k = p.row_ptr[i]; k < p.row_ptr[i + 1]; ++k) s += p.values[k] * p.x[p.col_idx[k]];
    const double v = fabs(s - p.b[i]);
    if (v > 0.0) m = MaxIdx{v, i};
  }
  m = block_best(m);
  if (threadIdx.x == 0) {
    p.blk_v[blockIdx.x] = m.v;
    p.blk_i[blockIdx.x] = m.i;
  }
}

__global__ void k_cols(CertifyParams p) {
  const int j = blockIdx.x * kT + threadIdx.x;
  MaxIdx m{0.0, -1};
  if (j < p.cols) {
    const double a = p.lo[j] - p.x[j], b = p.x[j] - p.hi[j];
    const double v = (a < b ? b : a) < 0.0 ? 0.0 : (a < b ? b : a);  // std::max(std::max(a, b), 0.0)
    if (v > 0.0) m = MaxIdx{v, j};
  }
  m = block_best(m);
  if (threadIdx.x == 0) {
    p.blk_v[p.row_blocks + blockIdx.x] = m.v;
    p.blk_i[p.row_blocks + blockIdx.x] = m.i;
  }
}

__global__ void k_fold(CertifyParams p) {
  // blocks [0, row_blocks) -> equality, [row_blocks, +col_blocks) -> bounds
  for (int part = 0; part < 2; ++part) {
    const int b0 = part == 0 ? 0 : p.row_blocks;
    const int b1 = part == 0 ? p.row_blocks : p.row_blocks + p.col_blocks;
    MaxIdx m{0.0, -1};
    for (int b = b0 + threadIdx.x; b < b1; b += kT) m = better(m, MaxIdx{p.blk_v[b], p.blk_i[b]});
    m = block_best(m);
    if (threadIdx.x == 0) {
      p.out[part] = m.v;
      p.out_idx[part] = m.i;
    }
    __syncthreads();
  }
}

__global__ void k_reconstruct(ReconstructParams p) {
  const int i = blockIdx.x * kT + threadIdx.x;
  if (i >= p.n) return;
  const int c0 = p.csr_ptr[i], c1 = p.csr_ptr[i + 1];
  double value = p.x[i];
  if (c1 > c0) {
    double sum = 0.0;
    for (int q = c0; q < c1; ++q) sum += p.z[p.csr_copy[q]];
    value = sum / static_cast<double>(c1 - c0);
  }
  const double lo = p.lo[i], hi = p.hi[i];
  const double t = value < lo ? lo : value;  // std::max(value, lo)
  p.out[i] = hi < t ? hi : t;                // std::min(., hi)
}

}  // namespace

cudaError_t launch_certify(const CertifyParams& p, cudaStream_t s) {
  k_rows<<<p.row_blocks, kT, 0, s>>>(p);
  k_cols<<<p.col_blocks, kT, 0, s>>>(p);
  k_fold<<<1, kT, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_reconstruct(const ReconstructParams& p, cudaStream_t s) {
  k_reconstruct<<<(p.n + kT - 1) / kT, kT, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace dopf::cuda
