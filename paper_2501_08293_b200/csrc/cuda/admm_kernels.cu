// Persistent fp64 ADMM iteration kernel for sm_100a.
//
// One launch runs the whole loop of reference proj/src/admm.cpp:190-235 on
// the device. Per iteration and per CTA ("block", a contiguous range of
// subsystems, layout.hpp):
//
//   (1) global update, admm.cpp:118-129 (K2): for every column the block's
//       rows reference, acc = sum of u = z - lambda/rho over its copies in
//       ascending s (read from L2), x = clamp((acc - c/rho) * inv, lo, hi).
//       Blocks compute shared columns redundantly (bitwise identical), so no
//       second barrier is needed to broadcast x.
//   (2) local update, admm.cpp:131-138 (K1): t = x[l2g] + lambda/rho,
//       z = P t + v as a sequential-j dot product per row; P comes from
//       shared memory (staged once per launch) or, when it does not fit, HBM.
//   (3) ||A z - b||_inf, admm.cpp:203-205.
//   (4) dual update, admm.cpp:140-143, and u = z - lambda/rho for the next
//       global step; residual partial sums, admm.cpp:150-163.
//   (5) warp-shuffle + block reduction of the partials (fixed order), one
//       grid / cluster barrier, every block combines all partials in the same
//       fixed order and takes the same stop decision (admm.hpp:63) -- the
//       on-device convergence check. Block 0 writes the trace row.
//
// Bitwise parity with the CPU oracle: compiled with --fmad=false; every
// iterate operation keeps the reference's form (division by rho, multiply by
// the inverse copy count, std::min/std::max select semantics, sequential sums
// in the reference order). Only the residual/objective reductions use a
// different (tree) order; they feed the stop test and the trace only.
#include <cooperative_groups.h>

#include "admm_kernels.cuh"

namespace dopf::cuda {

namespace {

__device__ __forceinline__ double ld_l2(const double* p) { return __ldcg(p); }

__device__ __forceinline__ double sel_max(double a, double b) { return (a < b) ? b : a; }  // std::max
__device__ __forceinline__ double sel_min(double a, double b) { return (b < a) ? b : a; }  // std::min

__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    unsigned int seen;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(bar) : "memory");
    } while (seen < target);
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ void cluster_barrier() {
  asm volatile(
      "barrier.cluster.arrive.release.aligned;\n\t"
      "barrier.cluster.wait.acquire.aligned;\n" ::
          : "memory");
}

constexpr int kWarps = kThreads / 32;

template <int K>
__global__ void __launch_bounds__(kThreads, 1) admm_persistent(const KernelParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const BlockDesc bd = p.blocks[blockIdx.x];
  const InstDesc id = p.inst[bd.instance];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;

  // ---- shared-memory carve-up (must match block_smem_bytes) ----
  unsigned char* cur = smem;
  const double* sP;
  const double* sA;
  if (bd.ops_in_smem) {
    double* dP = reinterpret_cast<double*>(cur);
    cur += sizeof(double) * bd.p_len;
    double* dA = reinterpret_cast<double*>(cur);
    cur += sizeof(double) * bd.a_len;
    for (int i = tid; i < bd.p_len; i += kThreads) dP[i] = p.P[bd.p_off + i];
    for (int i = tid; i < bd.a_len; i += kThreads) dA[i] = p.A[bd.a_off + i];
    sP = dP;
    sA = dA;
  } else {
    sP = p.P + bd.p_off;
    sA = p.A + bd.a_off;
  }
  double* tgt = reinterpret_cast<double*>(cur);
  cur += sizeof(double) * bd.rows;
  double* zs = reinterpret_cast<double*>(cur);
  cur += sizeof(double) * bd.rows;
  double* xs = reinterpret_cast<double*>(cur);
  cur += sizeof(double) * bd.cols;
  double* c_rho = reinterpret_cast<double*>(cur);
  cur += sizeof(double) * bd.cols;
  double* c_inv = reinterpret_cast<double*>(cur);
  cur += sizeof(double) * bd.cols;
  double* c_lo = reinterpret_cast<double*>(cur);
  cur += sizeof(double) * bd.cols;
  double* c_hi = reinterpret_cast<double*>(cur);
  cur += sizeof(double) * bd.cols;
  double* c_cost = reinterpret_cast<double*>(cur);
  cur += sizeof(double) * bd.cols;
  int32_t* cps = reinterpret_cast<int32_t*>(cur);
  cur += sizeof(int32_t) * bd.copy_len;
  cur = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(cur) + 15) & ~uintptr_t(15));
  double* red = reinterpret_cast<double*>(cur);  // [kWarps + 2][kPartials]

  const double rho = p.rho;
  for (int i = tid; i < bd.copy_len; i += kThreads) cps[i] = p.copies[bd.copy_off + i];
  for (int c = tid; c < bd.cols; c += kThreads) {
    const double cost = p.cc[bd.col_off + c];
    c_rho[c] = cost / rho;  // admm.cpp:126 evaluates c_i / rho; same value every iteration
    c_cost[c] = cost;
    c_inv[c] = p.cinv[bd.col_off + c];
    c_lo[c] = p.clo[bd.col_off + c];
    c_hi[c] = p.chi[bd.col_off + c];
  }

  // ---- per-thread state (rows, columns, equality rows) in registers ----
  RowMeta rm[K];
  ColMeta cm[K];
  AMeta am[K];
  double lam[K], zp[K], vv[K], bb[K], zn[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int r = tid + k * kThreads;
    if (r < bd.rows) {
      rm[k] = p.rmeta[bd.row0 + r];
      vv[k] = p.v[bd.row0 + r];
      zp[k] = p.z0[bd.row0 + r];
    } else {
      rm[k] = RowMeta{0, 0, 0, 0};
      vv[k] = 0.0;
      zp[k] = 0.0;
    }
    lam[k] = 0.0;
    zn[k] = 0.0;
    const int c = tid + k * kThreads;
    cm[k] = c < bd.cols ? p.cmeta[bd.col_off + c] : ColMeta{0, 0, 0, 0};
    const int a = tid + k * kThreads;
    if (a < bd.arows) {
      am[k] = p.ameta[bd.amet_off + a];
      bb[k] = p.ab[bd.amet_off + a];
    } else {
      am[k] = AMeta{0, 0, 0, 0};
      bb[k] = 0.0;
    }
  }
  __syncthreads();

  const double eps = p.eps_rel;
  const int G = id.blocks;
  double* part = p.part + static_cast<int64_t>(bd.instance) * 2 * p.blocks_per_instance * kPartials;
  double* u_even = p.u;
  double* u_odd = p.u + p.rows_total;
  double* trace = p.trace ? p.trace + static_cast<int64_t>(bd.instance) * p.trace_stride * 6 : nullptr;
  const bool leader = bd.inst_block == 0 && tid == 0;

  double run_max = 0.0, last_obj = 0.0;
  int status = 1;
  int it = 1;
  for (; it <= p.max_iter; ++it) {
    const int parity = (it - 1) & 1;
    const double* u_in = parity ? u_odd : u_even;
    double* u_out = parity ? u_even : u_odd;

    // (1) global update of the block's columns
    double obj = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int c = tid + k * kThreads;
      if (c < bd.cols) {
        const int32_t* q = cps + cm[k].copy_start;
        const int cnt = cm[k].copy_count;
        double acc = 0.0;
        int e = 0;
        for (; e + 4 <= cnt; e += 4) {
          const double a0 = ld_l2(u_in + q[e]), a1 = ld_l2(u_in + q[e + 1]);
          const double a2 = ld_l2(u_in + q[e + 2]), a3 = ld_l2(u_in + q[e + 3]);
          acc = acc + a0;
          acc = acc + a1;
          acc = acc + a2;
          acc = acc + a3;
        }
        for (; e < cnt; ++e) acc = acc + ld_l2(u_in + q[e]);
        const double unclamped = (acc - c_rho[c]) * c_inv[c];
        const double xv = sel_min(sel_max(unclamped, c_lo[c]), c_hi[c]);
        xs[c] = xv;
        if (cm[k].owner) {
          p.x_out[id.x_off + cm[k].gcol] = xv;
          obj = obj + c_cost[c] * xv;
        }
      }
    }
    __syncthreads();

    // (2a) consensus target t = x[l2g] + lambda / rho
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int r = tid + k * kThreads;
      if (r < bd.rows) tgt[r] = xs[rm[k].xloc] + lam[k] / rho;
    }
    __syncthreads();

    // (2b) z = P t + v, one row per thread, P column-major per subsystem
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int r = tid + k * kThreads;
      if (r < bd.rows) {
        const int n = rm[k].n;
        const double* pr = sP + rm[k].pofs;
        const double* tb = tgt + rm[k].base;
        double acc = 0.0;
        int j = 0;
        for (; j + 4 <= n; j += 4) {
          const double p0 = pr[(j + 0) * n], p1 = pr[(j + 1) * n];
          const double p2 = pr[(j + 2) * n], p3 = pr[(j + 3) * n];
          acc = acc + p0 * tb[j];
          acc = acc + p1 * tb[j + 1];
          acc = acc + p2 * tb[j + 2];
          acc = acc + p3 * tb[j + 3];
        }
        for (; j < n; ++j) acc = acc + pr[j * n] * tb[j];
        zn[k] = acc + vv[k];
        zs[r] = zn[k];
      }
    }
    __syncthreads();

    // (3) local equality residual ||A_s z_s - b_s||_inf
    double mx = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int a = tid + k * kThreads;
      if (a < bd.arows) {
        const int m = am[k].m, n = am[k].n;
        const double* ar = sA + am[k].aofs;
        const double* zb = zs + am[k].base;
        double acc = 0.0;
        for (int j = 0; j < n; ++j) acc = acc + ar[j * m] * zb[j];
        mx = sel_max(mx, fabs(acc - bb[k]));
      }
    }

    // (4) dual update, exchange value, residual partials
    double gap = 0.0, step = 0.0, bx2 = 0.0, z2 = 0.0, l2 = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int r = tid + k * kThreads;
      if (r < bd.rows) {
        const double z = zn[k];
        const double bx = xs[rm[k].xloc];
        const double d = bx - z;
        const double ln = lam[k] + rho * d;
        gap = gap + d * d;
        const double dz = z - zp[k];
        step = step + dz * dz;
        bx2 = bx2 + bx * bx;
        z2 = z2 + z * z;
        l2 = l2 + ln * ln;
        u_out[bd.row0 + r] = z - ln / rho;
        lam[k] = ln;
        zp[k] = z;
      }
    }

    // (5) block reduction (fixed butterfly + fixed warp order)
    double vals[7] = {gap, step, bx2, z2, l2, obj, mx};
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
      for (int q = 0; q < 6; ++q) vals[q] = vals[q] + __shfl_xor_sync(0xffffffffu, vals[q], off);
      vals[6] = sel_max(vals[6], __shfl_xor_sync(0xffffffffu, vals[6], off));
    }
    if (lane == 0) {
#pragma unroll
      for (int q = 0; q < 7; ++q) red[warp * kPartials + q] = vals[q];
    }
    __syncthreads();
    if (tid == 0) {
      double s[7];
#pragma unroll
      for (int q = 0; q < 7; ++q) s[q] = red[q];
      for (int w = 1; w < kWarps; ++w) {
#pragma unroll
        for (int q = 0; q < 6; ++q) s[q] = s[q] + red[w * kPartials + q];
        s[6] = sel_max(s[6], red[w * kPartials + 6]);
      }
      double* dst = part + (static_cast<int64_t>(parity) * p.blocks_per_instance + bd.inst_block) * kPartials;
#pragma unroll
      for (int q = 0; q < 7; ++q) dst[q] = s[q];
    }

    // (6) one barrier per iteration
    if (p.sync_mode == static_cast<int32_t>(SyncMode::grid))
      grid_barrier(p.bar + bd.instance, static_cast<unsigned int>(G) * static_cast<unsigned int>(it));
    else if (p.sync_mode == static_cast<int32_t>(SyncMode::cluster))
      cluster_barrier();
    else
      __syncthreads();

    // (7) combine the instance's partials (same order in every block)
    if (warp == 0) {
      const double* src = part + static_cast<int64_t>(parity) * p.blocks_per_instance * kPartials;
      double t[7] = {0, 0, 0, 0, 0, 0, 0};
      for (int g = lane; g < G; g += 32) {
        const double* row = src + g * kPartials;
#pragma unroll
        for (int q = 0; q < 6; ++q) t[q] = t[q] + ld_l2(row + q);
        t[6] = sel_max(t[6], ld_l2(row + 6));
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
        for (int q = 0; q < 6; ++q) t[q] = t[q] + __shfl_xor_sync(0xffffffffu, t[q], off);
        t[6] = sel_max(t[6], __shfl_xor_sync(0xffffffffu, t[6], off));
      }
      if (lane == 0) {
#pragma unroll
        for (int q = 0; q < 7; ++q) red[kWarps * kPartials + q] = t[q];
      }
    }
    __syncthreads();
    const double* tot = red + kWarps * kPartials;
    const double pres = sqrt(tot[0]);
    const double dres = rho * sqrt(tot[1]);
    const double eps_prim = eps * sel_max(sqrt(tot[2]), sqrt(tot[3]));
    const double eps_dual = eps * sqrt(tot[4]);
    last_obj = tot[5];
    run_max = sel_max(run_max, tot[6]);
    if (leader && trace) {
      double* row = trace + static_cast<int64_t>(it - 1) * 6;
      row[0] = it;
      row[1] = pres;
      row[2] = dres;
      row[3] = eps_prim;
      row[4] = eps_dual;
      row[5] = last_obj;
    }
    const bool done = pres <= eps_prim && dres <= eps_dual;
    __syncthreads();  // everyone has read `tot` before the next iteration overwrites red[]
    if (done) {
      status = 0;
      break;
    }
  }
  const int iterations = it > p.max_iter ? p.max_iter : it;

#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int r = tid + k * kThreads;
    if (r < bd.rows) {
      p.z_out[bd.row0 + r] = zp[k];
      p.lam_out[bd.row0 + r] = lam[k];
    }
  }
  if (leader) {
    p.iters[bd.instance] = iterations;
    p.status[bd.instance] = status;
    p.maxinf[bd.instance] = run_max;
    p.objective[bd.instance] = last_obj;
  }
}

template <int K>
cudaError_t launch_k(const KernelParams& p, int num_blocks, std::size_t smem, SyncMode mode,
                     int cluster_size, cudaStream_t stream) {
  auto kern = admm_persistent<K>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
  if (err != cudaSuccess) return err;
  if (mode == SyncMode::grid) {
    KernelParams local = p;
    void* args[] = {&local};
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(num_blocks),
                                       dim3(kThreads), args, smem, stream);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(num_blocks);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  int nattr = 0;
  if (mode == SyncMode::cluster && cluster_size > 1) {
    if (cluster_size > 8) {
      err = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (err != cudaSuccess) return err;
    }
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cluster_size;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    nattr = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = nattr;
  return cudaLaunchKernelEx(&cfg, kern, p);
}

}  // namespace

cudaError_t launch_admm(const KernelParams& p, int num_blocks, int K, std::size_t smem,
                        SyncMode mode, int cluster_size, cudaStream_t stream) {
  switch (K) {
    case 1: return launch_k<1>(p, num_blocks, smem, mode, cluster_size, stream);
    case 2: return launch_k<2>(p, num_blocks, smem, mode, cluster_size, stream);
    case 3: return launch_k<3>(p, num_blocks, smem, mode, cluster_size, stream);
    case 4: return launch_k<4>(p, num_blocks, smem, mode, cluster_size, stream);
    default: return cudaErrorInvalidValue;
  }
}

int max_dynamic_smem(int device) {
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  return v;
}

}  // namespace dopf::cuda
