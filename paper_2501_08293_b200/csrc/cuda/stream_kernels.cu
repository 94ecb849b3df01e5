// HBM-streaming fp64 ADMM iteration for instances whose operators do not fit
// shared memory (the tiled 0.5M-bus feeder). Three kernels per iteration,
// replayed by ONE CUDA-graph launch with a conditional while-node whose
// condition the finalize kernel clears at the stop test -- no host round trip
// per iteration:
//
//  k_global   (thread per boundary column)  admm.cpp:118-129: acc = sum over
//             the column's copies (CSR, ascending s) of u = z - lambda/rho;
//             x = clamp((acc - c/rho) * inv_count, lo, hi); c'x partials.
//  k_local    (CTA per chunk of whole subsystems, thread per row)
//             the same global update for the chunk's interior columns (all
//             copies in the chunk) from the z, lambda it loads anyway, then
//             admm.cpp:131-143, 203-205, 150-163: target in shared memory,
//             z = P target + v with P streamed from HBM (sliced ELL: 256
//             contiguous bytes per warp load), dual update, u, ||A z - b||_inf,
//             residual partials.
//  k_final    (one CTA) admm.cpp:164-169, 223-234: fixed-order combine of the
//             partials, trace row, running max, stop test.
//
// Bitwise parity with the oracle: --fmad=false and the reference's operation
// forms and summation orders for every iterate; only the residual/objective
// reductions are trees (stop test and trace only).
#include "stream_kernels.cuh"

#include <cstdlib>

namespace dopf::cuda {

namespace {

__device__ __forceinline__ double sel_max(double a, double b) { return (a < b) ? b : a; }

// one bulk (TMA-engine) prefetch of [ptr, ptr + bytes) into L2; bytes % 16 == 0
__device__ __forceinline__ void bulk_prefetch_l2(const void* ptr, uint32_t bytes) {
  if (bytes) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ptr), "r"(bytes) : "memory");
}
__device__ __forceinline__ void prefetch_l1(const void* ptr) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(ptr));
}
__device__ __forceinline__ double sel_min(double a, double b) { return (b < a) ? b : a; }

// fixed-shape block reduction of `V` values (sum; index `imax` uses max)
template <int V, int T>
__device__ __forceinline__ void block_reduce(double (&v)[V], double* sh, int imax) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int q = 0; q < V; ++q)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double o = __shfl_xor_sync(0xffffffffu, v[q], off);
      v[q] = q == imax ? sel_max(v[q], o) : v[q] + o;
    }
  constexpr int W = T / 32;
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < V; ++q) sh[q * W + warp] = v[q];
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int q = 0; q < V; ++q) {
      double x = lane < W ? sh[q * W + lane] : (q == imax ? 0.0 : 0.0);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, x, off);
        x = q == imax ? sel_max(x, o) : x + o;
      }
      v[q] = x;
    }
  }
}

__device__ __forceinline__ void finalize_iteration(const StreamParams& p, const double (&v)[7]) {
  StreamCtl* ctl = p.ctl;
  const int t = ctl->t + 1;
  const double pres = sqrt(v[0]);
  const double dres = p.rho * sqrt(v[1]);
  const double eps_prim = p.eps * sel_max(sqrt(v[2]), sqrt(v[3]));
  const double eps_dual = p.eps * sqrt(v[4]);
  const bool stop = pres <= eps_prim && dres <= eps_dual;
  ctl->t = t;
  ctl->maxinf = sel_max(ctl->maxinf, v[5]);
  ctl->objective = v[6];
  if (p.trace) {
    double* row = p.trace + static_cast<int64_t>(t - 1) * 6;
    row[0] = t;
    row[1] = pres;
    row[2] = dres;
    row[3] = eps_prim;
    row[4] = eps_dual;
    row[5] = v[6];
  }
  if (stop || t >= p.max_iter) {
    ctl->status = stop ? 0 : 1;
    ctl->done = 1;
    if (p.use_cond) cudaGraphSetConditional(p.cond, 0);
  }
}

__global__ void __launch_bounds__(kStreamRows, 4) k_global(const StreamParams p) {
  __shared__ double sh[8];
  if (p.ctl->done) return;  // partitioned loops may run past the stop (lazy host check)
  const int c = blockIdx.x * kStreamRows + threadIdx.x;
  double o[1] = {0.0};
  if (c < p.bcols) {
    // the column's first four copies: index loads, then value loads, all in
    // flight before the ascending-s sum
    const int q0 = p.col_ptr[c], q1 = p.col_ptr[c + 1];
    int32_t ref[4];
    double uv[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) ref[e] = q0 + e < q1 ? p.copies[q0 + e] : 0;
#pragma unroll
    for (int e = 0; e < 4; ++e)
      uv[e] = q0 + e < q1 ? (ref[e] >= 0 ? p.u[ref[e]] : p.u_remote[-ref[e] - 1]) : 0.0;
    double acc = 0.0;
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (q0 + e < q1) acc = acc + uv[e];
    for (int q = q0 + 4; q < q1; ++q) {
      const int32_t rq = p.copies[q];
      acc = acc + (rq >= 0 ? p.u[rq] : p.u_remote[-rq - 1]);
    }
    const double unclamped = (acc - p.cost[c] / p.rho) * p.inv[c];
    const double xv = sel_min(sel_max(unclamped, p.lo[c]), p.hi[c]);
    p.x[c] = xv;
    if (p.owner[c]) o[0] = p.cost[c] * xv;
  }
  block_reduce<1, kStreamRows>(o, sh, -1);
  if (threadIdx.x == 0) p.objp[blockIdx.x] = o[0];
}

template <int kMinBlocks>
__global__ void __launch_bounds__(kStreamRows, kMinBlocks) k_local(const StreamParams p) {
  __shared__ double tgt[kStreamRows];
  __shared__ double ush[kStreamRows];  // u = z - lambda/rho of the chunk's rows, then z
  __shared__ double xsh[kStreamRows];  // x of the chunk's interior columns
  __shared__ double zsh[kStreamRows];  // z^{t-1} (kept out of registers across the GEMV)
  __shared__ int32_t csh[kStreamRows + 1];  // interior CSR: chunk-local copy rows, column offsets
  __shared__ int32_t psh[kStreamRows + 1];
  __shared__ double osh[kStreamRows / 32];  // per-warp c'x of the interior columns
  __shared__ double sh[6 * (kStreamRows / 32)];
  if (p.ctl->done) return;
  // chunk fields are re-read where used (uniform, L1-resident) rather than
  // held in registers across the whole kernel
  const StreamChunk* ch = p.chunks + blockIdx.x;
  const int r = threadIdx.x, lane = r & 31, warp = r >> 5;
  const double rho = p.rho;
  const bool on = r < ch->rows;
  const int d = ch->row0 + r;
  // the chunk's operator slabs start moving HBM -> L2 now, overlapping the
  // dependent row loads and the interior-column update below
  if (r == 0) {
    bulk_prefetch_l2(p.P + ch->p0, static_cast<uint32_t>(8 * (ch->p1 - ch->p0)));
    bulk_prefetch_l2(p.A + ch->a0, static_cast<uint32_t>(8 * (ch->a1 - ch->a0)));
  }
  if (r < ch->icols) {
    const int c = ch->icol0 + r;
    prefetch_l1(p.cost + c);
    prefetch_l1(p.inv + c);
    prefetch_l1(p.lo + c);
    prefetch_l1(p.hi + c);
    prefetch_l1(p.owner + c);
  }
  // interior columns (admm.cpp:118-129): their CSR slice is staged in shared
  // memory by the same load round as the rows (copies <= rows)
  if (r < ch->icopies) csh[r] = p.copies[ch->icopy0 + r] - ch->row0;
  if (r <= ch->icols) psh[r] = p.col_ptr[ch->icol0 + r] - ch->icopy0;
  StreamRow rm{0, 0, 0, 0};
  double bx = 0.0, lamv = 0.0;
  if (on) {
    rm = p.rmeta[d];
    lamv = p.lam[d];
    const double zprev = p.z[d];
    if (rm.xcol < p.bcols) bx = p.x[rm.xcol];  // boundary column: k_global wrote x^t
    ush[r] = zprev - lamv / rho;               // the u the previous iteration stored
    zsh[r] = zprev;
  }
  __syncthreads();
  double o = 0.0;
  if (r < ch->icols) {
    const int c = ch->icol0 + r;
    const int q1 = psh[r + 1];
    double acc = 0.0;
    for (int q = psh[r]; q < q1; ++q) acc = acc + ush[csh[q]];  // ascending s
    const double unclamped = (acc - p.cost[c] / rho) * p.inv[c];
    const double xv = sel_min(sel_max(unclamped, p.lo[c]), p.hi[c]);
    xsh[r] = xv;
    p.x[c] = xv;
    if (p.owner[c]) o = p.cost[c] * xv;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) o = o + __shfl_xor_sync(0xffffffffu, o, off);
  if (lane == 0) osh[warp] = o;
  __syncthreads();
  if (on) {
    if (rm.xcol >= p.bcols) bx = xsh[rm.xcol - ch->icol0];
    tgt[r] = bx + lamv / rho;  // admm.cpp:136
  }
  __syncthreads();
  double v[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  if (on) {
    const double* pr = p.P + p.pslice[blockIdx.x * (kStreamRows / 32) + warp] + lane;
    const double* tb = tgt + rm.base;
    double acc = 0.0;
    for (int j0 = 0; j0 < rm.n; j0 += 8) {
      double pv[8], tv[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        pv[e] = 0.0;
        tv[e] = 0.0;
        if (j0 + e < rm.n) {
          pv[e] = __ldcs(pr + 32 * (j0 + e));  // streamed once per iteration
          tv[e] = tb[j0 + e];
        }
      }
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (j0 + e < rm.n) acc = acc + pv[e] * tv[e];
    }
    const double z = acc + p.v[d];
    const double dd = bx - z;
    const double ln = lamv + rho * dd;  // admm.cpp:142
    p.z[d] = z;
    p.lam[d] = ln;
    if (rm.xcol < p.bcols) p.u[d] = z - ln / rho;  // read by the next boundary update / exports
    v[0] = dd * dd;
    const double dz = z - zsh[r];
    v[1] = dz * dz;
    v[2] = bx * bx;
    v[3] = z * z;
    v[4] = ln * ln;
    ush[r] = z;  // every read of u happened before the previous barrier
  }
  __syncthreads();
  if (r < ch->arows) {
    const StreamARow am = p.ameta[blockIdx.x * kStreamRows + r];
    const double* ar = p.A + p.aslice[blockIdx.x * (kStreamRows / 32) + warp] + lane;
    const double* zb = ush + am.base;
    double acc = 0.0;
    for (int j0 = 0; j0 < am.n; j0 += 8) {
      double av[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) av[e] = j0 + e < am.n ? __ldcs(ar + 32 * (j0 + e)) : 0.0;
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (j0 + e < am.n) acc = acc + av[e] * zb[j0 + e];
    }
    v[5] = fabs(acc - p.ab[ch->arow0 + r]);
  }
  block_reduce<6, kStreamRows>(v, sh, 5);
  if (threadIdx.x == 0) {
    double* out = p.part + static_cast<int64_t>(blockIdx.x) * 8;
#pragma unroll
    for (int q = 0; q < 6; ++q) out[q] = v[q];
    double obj = 0.0;
#pragma unroll
    for (int w = 0; w < kStreamRows / 32; ++w) obj = obj + osh[w];
    out[6] = obj;
  }
}

constexpr int kFinalThreads = 256;
constexpr int kFinalBlocks = 128;

// Two-level fixed-order reduction of the chunk partials and objective
// partials: CTA g folds a contiguous range into level-2 slot g; the last CTA
// to finish (device-scope counter) folds the 128 slots in order and decides.
__global__ void __launch_bounds__(kFinalThreads) k_final(const StreamParams p) {
  __shared__ double sh[7 * (kFinalThreads / 32)];
  __shared__ bool last;
  if (p.ctl->done) return;
  double v[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};  // gap, step, bx2, z2, lam2, maxinf, objective
  const int g = blockIdx.x;
  const int c0 = static_cast<int>(static_cast<int64_t>(p.nchunks) * g / kFinalBlocks);
  const int c1 = static_cast<int>(static_cast<int64_t>(p.nchunks) * (g + 1) / kFinalBlocks);
  for (int k = c0 + threadIdx.x; k < c1; k += kFinalThreads) {
    const double* q = p.part + static_cast<int64_t>(k) * 8;
#pragma unroll
    for (int i = 0; i < 5; ++i) v[i] = v[i] + __ldcg(q + i);
    v[5] = sel_max(v[5], __ldcg(q + 5));
    v[6] = v[6] + __ldcg(q + 6);  // interior columns' c'x
  }
  const int o0 = static_cast<int>(static_cast<int64_t>(p.col_blocks) * g / kFinalBlocks);
  const int o1 = static_cast<int>(static_cast<int64_t>(p.col_blocks) * (g + 1) / kFinalBlocks);
  for (int k = o0 + threadIdx.x; k < o1; k += kFinalThreads) v[6] = v[6] + __ldcg(p.objp + k);
  block_reduce<7, kFinalThreads>(v, sh, 5);
  if (threadIdx.x == 0) {
    double* slot = p.part2 + g * 8;
#pragma unroll
    for (int q = 0; q < 7; ++q) slot[q] = v[q];
    __threadfence();
    const unsigned done_blocks = atomicAdd(p.final_count, 1u);
    last = done_blocks == kFinalBlocks - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double w[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  if (threadIdx.x < kFinalBlocks) {
    const double* q = p.part2 + threadIdx.x * 8;
#pragma unroll
    for (int i = 0; i < 7; ++i) w[i] = __ldcg(q + i);
  }
  block_reduce<7, kFinalThreads>(w, sh, 5);
  if (threadIdx.x == 0) {
    *p.final_count = 0;  // ready for the next iteration (kernel boundary orders it)
    if (p.partials_out) {  // partitioned: the host combines ranks, then calls k_decide
#pragma unroll
      for (int q = 0; q < 7; ++q) p.partials_out[q] = w[q];
      return;
    }
    finalize_iteration(p, w);
  }
}

__global__ void k_pack(const StreamParams p) {
  // this rank's exported u values -> its send slots (zero padded)
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < p.max_export) p.send[e] = e < p.n_export ? p.u[p.export_rows[e]] : 0.0;
}

__global__ void k_decide(const StreamParams p, const double* ranks, int nranks) {
  if (p.ctl->done) return;
  // rank partials combined in rank order: identical decision on every rank
  double v[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  for (int r = 0; r < nranks; ++r) {
#pragma unroll
    for (int q = 0; q < 5; ++q) v[q] = v[q] + ranks[r * 8 + q];
    v[5] = sel_max(v[5], ranks[r * 8 + 5]);
    v[6] = v[6] + ranks[r * 8 + 6];
  }
  finalize_iteration(p, v);
}

}  // namespace

using LocalKernel = void (*)(const StreamParams);

LocalKernel local_kernel() {
  // CTAs per SM for k_local: 4 (32 registers) measured fastest; DOPF_KLOCAL=3 for experiments
  static const LocalKernel k = [] {
    const char* e = std::getenv("DOPF_KLOCAL");
    return (e && e[0] == '3') ? &k_local<3> : &k_local<4>;
  }();
  return k;
}

void stream_launch_iteration(const StreamParams& p, cudaStream_t s) {
  k_global<<<p.col_blocks, kStreamRows, 0, s>>>(p);
  local_kernel()<<<p.nchunks, kStreamRows, 0, s>>>(p);
  k_final<<<kFinalBlocks, kFinalThreads, 0, s>>>(p);
}

void stream_launch_global(const StreamParams& p, cudaStream_t s) {
  k_global<<<p.col_blocks, kStreamRows, 0, s>>>(p);
}
void stream_launch_local(const StreamParams& p, cudaStream_t s) {
  local_kernel()<<<p.nchunks, kStreamRows, 0, s>>>(p);
  if (p.max_export > 0) k_pack<<<(p.max_export + 255) / 256, 256, 0, s>>>(p);
  k_final<<<kFinalBlocks, kFinalThreads, 0, s>>>(p);
}
void stream_launch_pack(const StreamParams& p, cudaStream_t s) {
  if (p.max_export > 0) k_pack<<<(p.max_export + 255) / 256, 256, 0, s>>>(p);
}
void stream_launch_decide(const StreamParams& p, const double* ranks, int nranks, cudaStream_t s) {
  k_decide<<<1, 1, 0, s>>>(p, ranks, nranks);
}

cudaError_t stream_build_graph(StreamParams p, cudaGraphExec_t* exec) {
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaGraphCreate(&g, 0);
  if (e != cudaSuccess) return e;
  cudaGraphConditionalHandle h;
  e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  if (e != cudaSuccess) return e;
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  e = cudaGraphAddNode(&node, g, nullptr, 0, &cp);
  if (e != cudaSuccess) return e;
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  p.cond = h;
  p.use_cond = 1;
  p.partials_out = nullptr;
  void* args[] = {&p};
  cudaKernelNodeParams kg = {}, kl = {}, kf = {};
  kg.func = reinterpret_cast<void*>(k_global);
  kg.gridDim = dim3(p.col_blocks);
  kg.blockDim = dim3(kStreamRows);
  kg.kernelParams = args;
  kl = kg;
  kl.func = reinterpret_cast<void*>(local_kernel());
  kl.gridDim = dim3(p.nchunks);
  kf = kg;
  kf.func = reinterpret_cast<void*>(k_final);
  kf.gridDim = dim3(kFinalBlocks);
  kf.blockDim = dim3(kFinalThreads);
  cudaGraphNode_t ng, nl, nf;
  if ((e = cudaGraphAddKernelNode(&ng, body, nullptr, 0, &kg)) != cudaSuccess) return e;
  if ((e = cudaGraphAddKernelNode(&nl, body, &ng, 1, &kl)) != cudaSuccess) return e;
  if ((e = cudaGraphAddKernelNode(&nf, body, &nl, 1, &kf)) != cudaSuccess) return e;
  e = cudaGraphInstantiate(exec, g, 0);
  cudaGraphDestroy(g);
  return e;
}

}  // namespace dopf::cuda
