// Persistent fp64 ADMM iteration kernel for sm_100a.
//
// One launch runs the whole loop of reference proj/src/admm.cpp:190-235 on
// the device. Each CTA ("block", a contiguous range of subsystems,
// layout.hpp) is warp-specialised:
//
//  compute warps 1..15, per iteration t
//   (L) local update, admm.cpp:131-138 (K1): target = x[l2g] + lambda/rho,
//       z = P target + v, a sequential-j dot product per row; P staged in
//       shared memory once per launch (or read from HBM when it does not fit).
//   (A) ||A_s z_s - b_s||_inf, admm.cpp:203-205.
//   (D) dual update, admm.cpp:140-143; exchange value u = z - lambda/rho;
//       per-warp residual partials, admm.cpp:150-163.
//   --- arrive(publish) / sync(exchanged) with the service warp ---
//   (G) global update for t+1, admm.cpp:118-129 (K2): for every column the
//       block's rows reference, acc = sum of u over the column's copies in
//       ascending s (L2 reads), x = clamp((acc - c/rho) * inv, lo, hi). Shared
//       columns are computed redundantly (bitwise identical) by every block
//       that needs them, so x is never broadcast.
//
//  service warp 0, per iteration t
//   (F) after the compute warps' u(t) stores: release the block's flag(t) --
//       the only inter-CTA synchronisation of the iteration;
//   (R) reduce the 15 warp partials in a fixed order into the block's slot(t);
//   (W) poll every block's flag(t) (relaxed loads + one acquire fence), then
//       let the compute warps start (G);
//   (S) combine all blocks' slots of t-1 (published before their flag(t)) in a
//       fixed order: residuals, trace row, stop test (admm.hpp:63). The compute
//       warps read the decision for t-2 after the exchange of t, so residual
//       work never sits on the critical path. State of the last two
//       iterations is kept (x in a 3-deep ring, z/lambda in 3 result buffers),
//       so the output is exactly the iterate of the stopping iteration.
//
// Bitwise parity with the CPU oracle: compiled with --fmad=false; every
// iterate operation keeps the reference's form (division by rho, multiply by
// the inverse copy count, std::min/std::max select semantics, sequential sums
// in the reference order). Only the residual/objective reductions use a
// different (tree) order; they feed the stop test and the trace only.
#include "admm_kernels.cuh"

namespace dopf::cuda {

namespace {

constexpr int kWarps = kThreads / 32;
constexpr int kCW = kThreads - 32;  // compute threads (warps 1..)
constexpr int kSlots = 3;           // partial-slot ring (see header)
constexpr int kDec = 4;             // decision ring
enum : int { kBarCompute = 1, kBarPublish = 2, kBarExchanged = 3 };

__device__ __forceinline__ double ld_l2(const double* p) { return __ldcg(p); }
__device__ __forceinline__ double sel_max(double a, double b) { return (a < b) ? b : a; }  // std::max
__device__ __forceinline__ double sel_min(double a, double b) { return (b < a) ? b : a; }  // std::min

__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// Warp 0: wait until every block of the instance published flag >= value
// (relaxed polls, then one acquire fence for the whole warp).
__device__ __forceinline__ void wait_flags(const unsigned long long* flags, int G, int lane,
                                           unsigned long long value) {
  for (int g = lane; g < G; g += 32)
    while (ld_relaxed_u64(flags + g) < value) {
    }
  fence_acq_rel();
  __syncwarp();
}

// 7 reduction lanes: 0..5 sums (gap, step, bx2, z2, lam2, objective), 6 max.
__device__ __forceinline__ void warp_reduce7(double (&v)[7], int width) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    if (off >= width) continue;
#pragma unroll
    for (int q = 0; q < 6; ++q) v[q] = v[q] + __shfl_xor_sync(0xffffffffu, v[q], off);
    v[6] = sel_max(v[6], __shfl_xor_sync(0xffffffffu, v[6], off));
  }
}

template <int K, bool kSmemOps>
__global__ void __launch_bounds__(kThreads, 1) admm_persistent(const KernelParams p) {
  extern __shared__ __align__(16) double smem[];
  const BlockDesc bd = p.blocks[blockIdx.x];
  const InstDesc id = p.inst[bd.instance];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;

  // ---- shared-memory carve-up, in doubles (must match block_smem_bytes) ----
  std::size_t off = 0;
  const double* gP = p.P + bd.p_off;
  const double* gA = p.A + bd.a_off;
  double* sP = smem;
  double* sA = smem;
  if (kSmemOps) {
    sP = smem + off;
    off += bd.p_len;
    sA = smem + off;
    off += bd.a_len;
    for (int i = tid; i < bd.p_len; i += kThreads) sP[i] = gP[i];
    for (int i = tid; i < bd.a_len; i += kThreads) sA[i] = gA[i];
  }
  const double* Pop = kSmemOps ? sP : gP;
  const double* Aop = kSmemOps ? sA : gA;
  double* tgt = smem + off;
  off += bd.rows;
  double* zs = smem + off;
  off += bd.rows;
  double* vs = smem + off;
  off += bd.rows;
  double* xring = smem + off;  // [3][cols]
  off += 3 * static_cast<std::size_t>(bd.cols);
  double* c_rho = smem + off;
  off += bd.cols;
  double* c_inv = smem + off;
  off += bd.cols;
  double* c_lo = smem + off;
  off += bd.cols;
  double* c_hi = smem + off;
  off += bd.cols;
  double* c_cost = smem + off;
  off += bd.cols;
  double* red = smem + off;  // [kWarps][kPartials] warp partials
  off += kWarps * kPartials;
  double* dec = smem + off;  // [kDec][4]: done, objective, running max, spare
  off += kDec * 4;
  double* a_rhs = smem + off;  // equality-row rhs b_r
  off += bd.arows;
  AMeta* a_meta = reinterpret_cast<AMeta*>(smem + off);  // 16 B each
  off += 2 * static_cast<std::size_t>(bd.arows);
  int32_t* cps = reinterpret_cast<int32_t*>(smem + off);

  const double rho = p.rho;
  const double eps = p.eps_rel;
  for (int i = tid; i < bd.copy_len; i += kThreads) cps[i] = p.copies[bd.copy_off + i];
  for (int r = tid; r < bd.rows; r += kThreads) vs[r] = p.v[bd.row0 + r];
  for (int a = tid; a < bd.arows; a += kThreads) {
    a_meta[a] = p.ameta[bd.amet_off + a];
    a_rhs[a] = p.ab[bd.amet_off + a];
  }
  for (int c = tid; c < bd.cols; c += kThreads) {
    const double cost = p.cc[bd.col_off + c];
    c_rho[c] = cost / rho;  // admm.cpp:126 evaluates c_i / rho; same value every iteration
    c_cost[c] = cost;
    c_inv[c] = p.cinv[bd.col_off + c];
    c_lo[c] = p.clo[bd.col_off + c];
    c_hi[c] = p.chi[bd.col_off + c];
  }
  if (tid < kDec * 4) dec[tid] = 0.0;

  const int G = id.blocks;
  const int64_t slot_stride = static_cast<int64_t>(p.blocks_per_instance) * kPartials;
  double* slots = p.part + static_cast<int64_t>(bd.instance) * kSlots * slot_stride;
  unsigned long long* flags = p.flags + static_cast<int64_t>(bd.instance) * p.blocks_per_instance;
  double* u_buf[2] = {p.u, p.u + p.rows_total};
  double* trace = p.trace ? p.trace + static_cast<int64_t>(bd.instance) * p.trace_stride * 6 : nullptr;
  const SyncMode mode = static_cast<SyncMode>(p.sync_mode);
  const bool exchange = mode != SyncMode::block;  // flags needed across CTAs
  __syncthreads();

  int stop_at = 0;  // set by the branch that detects the stop; broadcast below
  if (warp == 0) {
    // ======================= service warp =======================
    const bool leader = bd.inst_block == 0 && lane == 0;
    double run_max = 0.0;
    // combine every block's slot of iteration s in a fixed order
    auto combine = [&](int s) {
      const double* base = slots + static_cast<int64_t>(s % kSlots) * slot_stride;
      double t7[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      for (int g0 = lane; g0 < G; g0 += 64) {  // two slots per lane in flight
        const int g1 = g0 + 32;
        const double* r0 = base + g0 * kPartials;
        const double* r1 = base + g1 * kPartials;
        double a0[7], a1[7];
#pragma unroll
        for (int q = 0; q < 7; ++q) {
          a0[q] = ld_l2(r0 + q);
          a1[q] = g1 < G ? ld_l2(r1 + q) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 6; ++q) t7[q] = t7[q] + a0[q];
        t7[6] = sel_max(t7[6], a0[6]);
        if (g1 < G) {
#pragma unroll
          for (int q = 0; q < 6; ++q) t7[q] = t7[q] + a1[q];
          t7[6] = sel_max(t7[6], a1[6]);
        }
      }
      warp_reduce7(t7, 32);
      const double pres = sqrt(t7[0]);
      const double dres = rho * sqrt(t7[1]);
      const double eps_prim = eps * sel_max(sqrt(t7[2]), sqrt(t7[3]));
      const double eps_dual = eps * sqrt(t7[4]);
      run_max = sel_max(run_max, t7[6]);
      if (lane == 0) {
        double* rec = dec + (s % kDec) * 4;
        rec[0] = (pres <= eps_prim && dres <= eps_dual) ? 1.0 : 0.0;
        rec[1] = t7[5];
        rec[2] = run_max;
        if (leader && trace) {
          double* row = trace + static_cast<int64_t>(s - 1) * 6;
          row[0] = s;
          row[1] = pres;
          row[2] = dres;
          row[3] = eps_prim;
          row[4] = eps_dual;
          row[5] = t7[5];
        }
      }
      __syncwarp();
    };
    auto publish_and_wait = [&](int value) {
      if (!exchange) return;
      if (lane == 0) st_release_u64(flags + bd.inst_block, static_cast<unsigned long long>(value));
      wait_flags(flags, G, lane, static_cast<unsigned long long>(value));
    };

    int t = 1;
    for (;; ++t) {
      named_sync(kBarPublish, kThreads);  // compute warps: u(t) stored, warp partials in red[]
      if (exchange && lane == 0)
        st_release_u64(flags + bd.inst_block, static_cast<unsigned long long>(t));
      // (R) fixed-order reduction of the 15 warp partials -> slot(t)
      double w7[7];
#pragma unroll
      for (int q = 0; q < 7; ++q) w7[q] = (lane >= 1 && lane < kWarps) ? red[lane * kPartials + q] : 0.0;
      warp_reduce7(w7, kWarps);
      if (lane == 0) {
        double* my_slot = slots + static_cast<int64_t>(t % kSlots) * slot_stride +
                          static_cast<int64_t>(bd.inst_block) * kPartials;
#pragma unroll
        for (int q = 0; q < 7; ++q) my_slot[q] = w7[q];
      }
      // (W) every block's u(t) is visible
      if (exchange) wait_flags(flags, G, lane, static_cast<unsigned long long>(t));
      const bool cw_stop = (t >= 3 && dec[((t - 2) % kDec) * 4] != 0.0) || t == p.max_iter;
      named_arrive(kBarExchanged, kThreads);
      // (S) residuals / stop test of t-1 (slots published before flag(t))
      if (t >= 2) combine(t - 1);
      if (cw_stop) break;
    }
    if (t >= 3 && dec[((t - 2) % kDec) * 4] != 0.0) {
      stop_at = t - 2;
    } else {
      // reached max_iter: the slots of max_iter become visible with one more flag
      publish_and_wait(t + 1);
      combine(t);
      stop_at = (t >= 2 && dec[((t - 1) % kDec) * 4] != 0.0) ? t - 1 : t;
    }
    if (lane == 0) {
      const double* rec = dec + (stop_at % kDec) * 4;
      red[0] = stop_at;
      if (bd.inst_block == 0) {
        p.iters[bd.instance] = stop_at;
        p.status[bd.instance] = rec[0] != 0.0 ? 0 : 1;
        p.maxinf[bd.instance] = rec[2];
        p.objective[bd.instance] = rec[1];
      }
    }
  } else {
    // ======================= compute warps =======================
    const int ctid = tid - 32;
    RowMeta rm[K];
    ColMeta cm[K];
    double lam[K], lr[K], zp[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int r = ctid + k * kCW;
      if (r < bd.rows) {
        rm[k] = p.rmeta[bd.row0 + r];
        zp[k] = p.z0[bd.row0 + r];
      } else {
        rm[k] = RowMeta{0, 0, 0, 0};
        zp[k] = 0.0;
      }
      lam[k] = 0.0;
      lr[k] = 0.0 / rho;  // lambda^0 / rho
      cm[k] = r < bd.cols ? p.cmeta[bd.col_off + r] : ColMeta{0, 0, 0, 0};
    }

    // (G) global update from u_in into xdst; returns the c'x share of owned columns
    auto global_update = [&](const double* u_in, double* xdst) -> double {
      double obj = 0.0;
      double a[K][4];
#pragma unroll
      for (int k = 0; k < K; ++k) {  // issue the first (up to) 4 copy loads of every column
        const int c = ctid + k * kCW;
        const int cnt = c < bd.cols ? cm[k].copy_count : 0;
        const int32_t* q = cps + cm[k].copy_start;
#pragma unroll
        for (int e = 0; e < 4; ++e) a[k][e] = e < cnt ? ld_l2(u_in + q[e]) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int c = ctid + k * kCW;
        if (c < bd.cols) {
          const int cnt = cm[k].copy_count;
          const int32_t* q = cps + cm[k].copy_start;
          double acc = 0.0;
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (e < cnt) acc = acc + a[k][e];
          for (int e = 4; e < cnt; ++e) acc = acc + ld_l2(u_in + q[e]);
          const double unclamped = (acc - c_rho[c]) * c_inv[c];
          const double xv = sel_min(sel_max(unclamped, c_lo[c]), c_hi[c]);
          xdst[c] = xv;
          if (cm[k].owner) obj = obj + c_cost[c] * xv;
        }
      }
      return obj;
    };

    double obj = global_update(u_buf[0], xring);  // x^1 from u^0 = z^0
    named_sync(kBarCompute, kCW);
    for (int t = 1;; ++t) {
      const double* xt = xring + static_cast<std::size_t>((t - 1) % 3) * bd.cols;  // x^t
      double* u_out = u_buf[t & 1];
      double* z_res = p.z_out + static_cast<int64_t>(t % 3) * p.rows_total;
      double* l_res = p.lam_out + static_cast<int64_t>(t % 3) * p.rows_total;

      // (L1) consensus target
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int r = ctid + k * kCW;
        if (r < bd.rows) tgt[r] = xt[rm[k].xloc] + lr[k];  // lr = lambda / rho, same rounding
      }
      named_sync(kBarCompute, kCW);

      // (L2) z = P t + v, one row per thread, P column-major per subsystem
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int r = ctid + k * kCW;
        if (r < bd.rows) {
          const int n = rm[k].n;
          const double* pr = Pop + rm[k].pofs;
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
          zs[r] = acc + vs[r];
        }
      }
      named_sync(kBarCompute, kCW);

      // (A) local equality residual ||A_s z_s - b_s||_inf
      double v7[7] = {0.0, 0.0, 0.0, 0.0, 0.0, obj, 0.0};
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int a = ctid + k * kCW;
        if (a < bd.arows) {
          const AMeta am = a_meta[a];
          const double* ar = Aop + am.aofs;
          const double* zb = zs + am.base;
          double acc = 0.0;
          for (int j = 0; j < am.n; ++j) acc = acc + ar[j * am.m] * zb[j];
          v7[6] = sel_max(v7[6], fabs(acc - a_rhs[a]));
        }
      }
      // (D) dual update, exchange value, residual partials
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int r = ctid + k * kCW;
        if (r < bd.rows) {
          const double z = zs[r];
          const double bx = xt[rm[k].xloc];
          const double d = bx - z;
          const double ln = lam[k] + rho * d;
          v7[0] = v7[0] + d * d;
          const double dz = z - zp[k];
          v7[1] = v7[1] + dz * dz;
          v7[2] = v7[2] + bx * bx;
          v7[3] = v7[3] + z * z;
          v7[4] = v7[4] + ln * ln;
          lr[k] = ln / rho;  // reused as lambda/rho by the next target (admm.cpp:136)
          u_out[bd.row0 + r] = z - lr[k];
          z_res[bd.row0 + r] = z;   // (z, lambda)^t kept until the stop test of t is known
          l_res[bd.row0 + r] = ln;
          lam[k] = ln;
          zp[k] = z;
        }
      }
      warp_reduce7(v7, 32);
      if (lane == 0) {
#pragma unroll
        for (int q = 0; q < 7; ++q) red[warp * kPartials + q] = v7[q];
      }
      named_arrive(kBarPublish, kThreads);
      named_sync(kBarExchanged, kThreads);
      if ((t >= 3 && dec[((t - 2) % kDec) * 4] != 0.0) || t == p.max_iter) break;
      obj = global_update(u_out, xring + static_cast<std::size_t>(t % 3) * bd.cols);  // x^{t+1}
      named_sync(kBarCompute, kCW);
    }
  }
  __syncthreads();
  stop_at = static_cast<int>(red[0]);
  if (warp != 0) {
    // owners write x^stop_at (still in the ring); (z, lambda)^stop_at are in
    // result buffer stop_at % 3, which the host reads
    const int ctid = tid - 32;
    const double* xfinal = xring + static_cast<std::size_t>((stop_at - 1) % 3) * bd.cols;
    for (int c = ctid; c < bd.cols; c += kCW) {
      const ColMeta cmc = p.cmeta[bd.col_off + c];
      if (cmc.owner) p.x_out[id.x_off + cmc.gcol] = xfinal[c];
    }
  }
}

template <int K, bool kSmemOps>
cudaError_t launch_k(const KernelParams& p, int num_blocks, std::size_t smem, SyncMode mode,
                     int cluster_size, cudaStream_t stream) {
  auto kern = admm_persistent<K, kSmemOps>;
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

template <int K>
cudaError_t launch_ops(const KernelParams& p, int num_blocks, std::size_t smem, SyncMode mode,
                       int cluster_size, bool smem_ops, cudaStream_t stream) {
  return smem_ops ? launch_k<K, true>(p, num_blocks, smem, mode, cluster_size, stream)
                  : launch_k<K, false>(p, num_blocks, smem, mode, cluster_size, stream);
}

}  // namespace

cudaError_t launch_admm(const KernelParams& p, int num_blocks, int K, std::size_t smem,
                        SyncMode mode, int cluster_size, bool smem_ops, cudaStream_t stream) {
  switch (K) {
    case 1: return launch_ops<1>(p, num_blocks, smem, mode, cluster_size, smem_ops, stream);
    case 2: return launch_ops<2>(p, num_blocks, smem, mode, cluster_size, smem_ops, stream);
    case 3: return launch_ops<3>(p, num_blocks, smem, mode, cluster_size, smem_ops, stream);
    case 4: return launch_ops<4>(p, num_blocks, smem, mode, cluster_size, smem_ops, stream);
    default: return cudaErrorInvalidValue;
  }
}

int max_dynamic_smem(int device) {
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  return v;
}

}  // namespace dopf::cuda
