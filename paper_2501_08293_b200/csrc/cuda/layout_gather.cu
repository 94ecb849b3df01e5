// Re-upload fast path: when a model's sparsity structure matches the plan
// already on the device, only its raw value arrays are copied (contiguous
// H2D, no host-side repacking) and this kernel scatters them into the
// resident kernel's layout through the plan's index maps (layout_builder.hpp
// InstancePlan: p_src / a_src / ref_of_dev / gcol / ab_src).
#include <cuda_runtime.h>

#include <cstdint>

#include "layout_gather.cuh"

namespace dopf::cuda {

namespace {

__global__ void k_gather(const GatherParams g) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t k = i; k < g.np; k += stride) g.P[k] = g.p_src[k] >= 0 ? g.rawP[g.p_src[k]] : 0.0;
  for (int64_t k = i; k < g.na; k += stride) g.A[k] = g.a_src[k] >= 0 ? g.rawA[g.a_src[k]] : 0.0;
  for (int64_t k = i; k < g.rows; k += stride) {
    g.v[k] = g.rawv[g.ref_of_dev[k]];
    g.z0[k] = g.rawz0[g.ref_of_dev[k]];
  }
  for (int64_t k = i; k < g.cols; k += stride) {
    const int32_t c = g.gcol[k];
    g.cc[k] = g.rawc[c];
    g.cinv[k] = g.rawinv[c];
    g.clo[k] = g.rawlo[c];
    g.chi[k] = g.rawhi[c];
  }
  for (int64_t k = i; k < g.nab; k += stride) g.ab[k] = g.rawb[g.ab_src[k]];
}

// final iterate of every instance out of the z / lambda rings (one CTA per
// instance): instance i stopped at iters[i], its (z, lambda) in ring slot
// iters[i] % ring
__global__ void k_final_iterates(const double* zring, const double* lring, int64_t rows_total,
                                 const int32_t* row0, const int32_t* rows, const int32_t* iters,
                                 int ring, double* zout, double* lout) {
  const int i = blockIdx.x;
  const int64_t base = static_cast<int64_t>(iters[i] % ring) * rows_total;
  for (int d = row0[i] + threadIdx.x; d < row0[i] + rows[i]; d += blockDim.x) {
    zout[d] = zring[base + d];
    lout[d] = lring[base + d];
  }
}

// single instance: the stopping iterate's ring slot, permuted to reference
// order, plus the scalar results packed for one copy
__global__ void k_final_single(const double* zring, const double* lring, int64_t rows, const int32_t* ref_of_dev,
                               const int32_t* iters, int ring, const int32_t* status, const double* maxinf,
                               const double* obj, const int32_t* ties, double* zout, double* lout,
                               double* scalars) {
  const int64_t base = static_cast<int64_t>(iters[0] % ring) * rows;
  for (int64_t d = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; d < rows;
       d += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t ref = ref_of_dev[d];
    zout[ref] = zring[base + d];
    lout[ref] = lring[base + d];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    scalars[0] = iters[0];
    scalars[1] = status[0];
    scalars[2] = maxinf[0];
    scalars[3] = obj[0];
    scalars[4] = ties[0];
    scalars[5] = ties[1];
  }
}

}  // namespace

cudaError_t launch_final_single(const double* zring, const double* lring, int64_t rows, const int32_t* ref_of_dev,
                                const int32_t* iters, int ring, const int32_t* status, const double* maxinf,
                                const double* obj, const int32_t* ties, double* zout, double* lout,
                                double* scalars, int sm_count, cudaStream_t s) {
  k_final_single<<<sm_count, 256, 0, s>>>(zring, lring, rows, ref_of_dev, iters, ring, status, maxinf, obj, ties,
                                          zout, lout, scalars);
  return cudaGetLastError();
}

cudaError_t launch_final_iterates(const double* zring, const double* lring, int64_t rows_total,
                                  const int32_t* row0, const int32_t* rows, const int32_t* iters,
                                  int instances, int ring, double* zout, double* lout, cudaStream_t s) {
  k_final_iterates<<<instances, 256, 0, s>>>(zring, lring, rows_total, row0, rows, iters, ring, zout, lout);
  return cudaGetLastError();
}

cudaError_t launch_gather(const GatherParams& g, int sm_count, cudaStream_t s) {
  k_gather<<<sm_count * 4, 512, 0, s>>>(g);
  return cudaGetLastError();
}

}  // namespace dopf::cuda
