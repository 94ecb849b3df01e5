// HBM-streaming fp64 ADMM iteration for instances whose operators do not fit
// shared memory (the tiled 0.5M-bus feeder). Per iteration, replayed by ONE
// CUDA-graph launch with a conditional while-node whose condition the final
// kernel clears at the stop test (no host round trip per iteration):
//
//  k_global   (thread per boundary column)  admm.cpp:118-129: acc = sum over
//             the column's copies (CSR, ascending s) of u = z - lambda/rho;
//             x = clamp((acc - c/rho) * inv_count, lo, hi); c'x partials; x is
//             also written to the import slots of the chunks that read it.
//  k_staged   (persistent, 2 CTAs/SM: 8 compute warps + 1 producer warp)
//             the producer moves each chunk (image, z, lambda, imports) into
//             a shared-memory stage with four bulk copies (TMA engine,
//             mbarrier completion, two stages in flight); the compute warps
//             run the chunk's iteration out of shared memory: interior
//             columns' global update (all copies in the chunk), target, GEMV
//             z = P target + v (admm.cpp:131-138), dual update (:140-143),
//             ||A z - b||_inf (:203-205), residual partials (:150-163).
//  k_local    the same chunk iteration for the few chunks whose stage would
//             not fit shared memory (image read straight from HBM), on SMs
//             the staged kernel leaves free (parallel graph branch).
//  (final)    the last chunk CTA of the iteration (k_staged or k_local)
//             folds the partials in a fixed order and takes the stop test
//             (admm.cpp:164-169, 223-234): trace row, running max, graph
//             condition -- no separate kernel.
//
// Bitwise parity with the oracle: --fmad=false, the reference's operation
// forms and summation orders for every iterate, and divisions by rho that are
// exactly the IEEE quotient (div_rho.cuh); only the residual/objective
// reductions are trees (stop test and trace only).
#include "stream_kernels.cuh"
#include "stop_test.cuh"

#include "div_rho.cuh"

#include <algorithm>
#include <cstdlib>

namespace dopf::cuda {

namespace {

__device__ __forceinline__ double sel_max(double a, double b) { return (a < b) ? b : a; }


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
  if (stop_near_tie(pres, eps_prim, dres, eps_dual)) {
    ++ctl->ties;
    if (ctl->first_tie == 0) ctl->first_tie = t;
  }
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

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// PhaseTimings stamps: one thread of the first CTA of each kernel
__device__ __forceinline__ void stamp_chunks_start(StreamCtl* ctl) {
  const unsigned long long now = gtimer();
  ctl->t_global += static_cast<long long>(now - ctl->g0);
  ctl->c0 = now;
}

__global__ void __launch_bounds__(kStreamRows, 4) k_global(const StreamParams p) {
  __shared__ double sh[8];
  if (p.ctl->done) return;  // partitioned loops may run past the stop (lazy host check)
  if (blockIdx.x == 0 && threadIdx.x == 0) p.ctl->g0 = gtimer();
  const int c = blockIdx.x * kStreamRows + threadIdx.x;
  double o[1] = {0.0};
  if (c < p.bcols) {
    // every load that does not depend on another goes out first (column data,
    // import range, copy range), then the copies' indices, then their u
    const int q0 = __ldg(p.col_ptr + c), q1 = __ldg(p.col_ptr + c + 1);
    const double cost = __ldg(p.cost + c), inv = __ldg(p.inv + c), lo = __ldg(p.lo + c), hi = __ldg(p.hi + c);
    const int i0 = __ldg(p.imp_ptr + c), i1 = __ldg(p.imp_ptr + c + 1);
    const bool own = __ldg(p.owner + c) != 0;
    int32_t ref[4];
    double uv[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) ref[e] = q0 + e < q1 ? __ldg(p.copies + q0 + e) : 0;
    const double cr = div_rho(cost, p.rho, p.rho_inv);
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
    const double unclamped = (acc - cr) * inv;
    const double xv = sel_min(sel_max(unclamped, lo), hi);
    p.x[c] = xv;
    for (int e = i0; e < i1; ++e) p.ximp[__ldg(p.imp_slot + e)] = xv;  // chunk imports
    if (own) o[0] = cost * xv;
  }
  block_reduce<1, kStreamRows>(o, sh, -1);
  if (threadIdx.x == 0) p.objp[blockIdx.x] = o[0];
}

template <typename T>
__device__ __forceinline__ const T* sec(const unsigned char* img, const ChunkHead& h, int id) {
  return reinterpret_cast<const T*>(img + h.off[id]);
}

// Sliced-ELL row dot product in the reference's sequential-j order
// (admm.cpp:137): batches of 8 operator loads in flight, then the sum.
template <typename Ld>
__device__ __forceinline__ double row_dot(const double* pr, const double* tb, int n, Ld ld) {
  double acc = 0.0;
  for (int j0 = 0; j0 < n; j0 += 8) {
    double pv[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) pv[e] = j0 + e < n ? ld(pr + 32 * (j0 + e)) : 0.0;
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (j0 + e < n) acc = acc + pv[e] * tb[j0 + e];
  }
  return acc;
}

// One chunk's iteration, shared by the direct-load kernel (image in HBM) and
// the staged kernel (image in shared memory): thread r = row r, interior
// column r, equality row r. `img` is the chunk image, zin / lin / xin the
// chunk's z^{t-1}, lambda^{t-1} and imported boundary x. Four barriers
// (`sync`) separate: u -> interior x -> target -> GEMV/dual -> A z - b.
// Accumulates the residual partials into v (gap, step, bx2, z2, lam2, maxinf, c'x).
template <int kRows, typename Sync, typename Ld>
__device__ __forceinline__ void chunk_iteration(const StreamParams& p, const unsigned char* img,
                                                const ChunkHead& h, const double* zin, const double* lin,
                                                const double* xin, double* tgt, double* ush, double* xsh,
                                                double* zsh, double (&v)[7], Sync sync, Ld ld) {
  const int r = threadIdx.x, lane = r & 31, warp = r >> 5;
  const double rho = p.rho;
  // the chunk's sections, read once (later smem stores could alias them for the compiler)
  const int rows = h.rows, arows = h.arows, icols = h.icols, row0 = h.row0, icol0 = h.icol0;
  const StreamRow* s_rows = reinterpret_cast<const StreamRow*>(img + h.off[kImgRows]);
  const int2* s_sl = reinterpret_cast<const int2*>(img + h.off[kImgSlices]);
  const double* s_P = reinterpret_cast<const double*>(img + h.off[kImgP]);
  const double* s_A = reinterpret_cast<const double*>(img + h.off[kImgA]);
  const StreamARow* s_ar = reinterpret_cast<const StreamARow*>(img + h.off[kImgArows]);
  const StreamCol* s_cols = reinterpret_cast<const StreamCol*>(img + h.off[kImgCols]);
  const uint32_t* s_cm = reinterpret_cast<const uint32_t*>(img + h.off[kImgCmeta]);
  const int16_t* s_cc = reinterpret_cast<const int16_t*>(img + h.off[kImgCopies]);
  const bool on = r < rows;
  StreamRow rm{0, 0, -1, -1, 0.0};
  double lamv = 0.0, q = 0.0;
  if (on) {
    rm = s_rows[r];
    lamv = lin[r];
    const double zprev = zin[r];
    q = div_rho(lamv, rho, p.rho_inv);
    ush[r] = zprev - q;  // the u = z - lambda/rho the previous iteration produced
    zsh[r] = zprev;
  }
  sync();
  if (r < icols) {  // interior column: admm.cpp:118-129 over the chunk's own copies
    const uint32_t cm = s_cm[r];
    const int16_t* cc = s_cc + cmeta_start(cm);
    const int cnt = cmeta_count(cm);
    double acc = 0.0;
#pragma unroll 1
    for (int e = 0; e < cnt; ++e) acc = acc + ush[cc[e]];  // ascending s
    const StreamCol col = s_cols[r];
    const double unclamped = (acc - div_rho(col.cost, rho, p.rho_inv)) * col.inv;
    const double xv = sel_min(sel_max(unclamped, col.lo), col.hi);
    xsh[r] = xv;
    p.x[icol0 + r] = xv;
    if (cmeta_owner(cm)) v[6] = v[6] + col.cost * xv;
  }
  sync();
  double bx = 0.0;
  if (on) {
    bx = rm.xin >= 0 ? xin[rm.xin] : xsh[rm.xloc];
    tgt[r] = bx + q;  // admm.cpp:136
  }
  sync();
  if (on) {
    const double acc = row_dot(s_P + s_sl[warp].x + lane, tgt + rm.base, rm.n, ld);
    const double z = acc + rm.v;
    const double dd = bx - z;
    const double ln = lamv + rho * dd;  // admm.cpp:142
    const int d = row0 + r;
    p.z[d] = z;
    p.lam[d] = ln;
    if (rm.xin >= 0) p.u[d] = z - div_rho(ln, rho, p.rho_inv);  // read by the next boundary update / exports
    v[0] = v[0] + dd * dd;
    const double dz = z - zsh[r];
    v[1] = v[1] + dz * dz;
    v[2] = v[2] + bx * bx;
    v[3] = v[3] + z * z;
    v[4] = v[4] + ln * ln;
    ush[r] = z;  // every read of u happened before the previous barrier
  }
  sync();
  if (r < arows) {  // ||A_s z_s - b_s||_inf (admm.cpp:203-205)
    const StreamARow ar = s_ar[r];
    const double acc = row_dot(s_A + s_sl[warp].y + lane, ush + ar.base, ar.n, ld);
    v[5] = sel_max(v[5], fabs(acc - ar.b));
  }
}

// CTA reduction of the 7 partials (fixed shape), written to part[slot]
template <int kRows, typename Sync>
__device__ __forceinline__ void write_partials(const StreamParams& p, double (&v)[7], double* red, int slot,
                                               Sync sync) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int qv = 0; qv < 7; ++qv)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double o = __shfl_xor_sync(0xffffffffu, v[qv], off);
      v[qv] = qv == 5 ? sel_max(v[qv], o) : v[qv] + o;
    }
  constexpr int W = kRows / 32;
  if (lane == 0)
#pragma unroll
    for (int qv = 0; qv < 7; ++qv) red[qv * W + warp] = v[qv];
  sync();
  if (warp == 0) {
#pragma unroll
    for (int qv = 0; qv < 7; ++qv) {
      double x = lane < W ? red[qv * W + lane] : 0.0;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, x, off);
        x = qv == 5 ? sel_max(x, o) : x + o;
      }
      if (lane == 0) p.part[static_cast<int64_t>(slot) * 8 + qv] = x;
    }
  }
}

// The CTA that writes the last partial of the iteration folds all of them
// (fixed order, fixed 256-thread shape whichever kernel it belongs to) and
// takes the stop decision (admm.cpp:164-169, 223-234) -- no separate kernel.
constexpr int kFoldThreads = 256;
__device__ __forceinline__ void fold_barrier() { asm volatile("bar.sync 2, %0;" ::"n"(kFoldThreads) : "memory"); }

__device__ void arrive_and_finish(const StreamParams& p, double* red, bool* last) {
  const int tid = threadIdx.x;
  if (tid >= kFoldThreads) return;
  if (tid == 0) {
    __threadfence();  // this CTA's partial (written by thread 0) before the count
    *last = atomicAdd(p.final_count, 1u) == static_cast<unsigned>(p.npart - 1);
  }
  fold_barrier();
  if (!*last) return;
  __threadfence();
  double v[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};  // gap, step, bx2, z2, lam2, maxinf, objective
  for (int k = tid; k < p.npart; k += kFoldThreads) {
    const double* q = p.part + static_cast<int64_t>(k) * 8;
#pragma unroll
    for (int i = 0; i < 5; ++i) v[i] = v[i] + __ldcg(q + i);
    v[5] = sel_max(v[5], __ldcg(q + 5));
    v[6] = v[6] + __ldcg(q + 6);  // interior columns' c'x
  }
  for (int k = tid; k < p.col_blocks; k += kFoldThreads) v[6] = v[6] + __ldcg(p.objp + k);  // boundary c'x
  const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int q = 0; q < 7; ++q)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double o = __shfl_xor_sync(0xffffffffu, v[q], off);
      v[q] = q == 5 ? sel_max(v[q], o) : v[q] + o;
    }
  constexpr int W = kFoldThreads / 32;
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < 7; ++q) red[q * W + warp] = v[q];
  fold_barrier();
  if (tid == 0) {
    double w[7];
#pragma unroll
    for (int q = 0; q < 7; ++q) {
      w[q] = red[q * W];
      for (int k = 1; k < W; ++k) w[q] = q == 5 ? sel_max(w[q], red[q * W + k]) : w[q] + red[q * W + k];
    }
    *p.final_count = 0;  // ready for the next iteration (kernel boundary orders it)
    p.ctl->t_local += static_cast<long long>(gtimer() - p.ctl->c0);
    if (p.partials_out) {  // partitioned: the host combines ranks, then calls k_decide
#pragma unroll
      for (int q = 0; q < 7; ++q) p.partials_out[q] = w[q];
      return;
    }
    finalize_iteration(p, w);
  }
}

// Direct-load kernel for chunks whose stage would not fit shared memory:
// one CTA per chunk, image read straight from HBM; kRows = kWideRows when a
// chunk holds a subsystem wider than kStreamRows (a hub bus).
template <int kRows>
__global__ void __launch_bounds__(kRows, 1024 / kRows) k_local(const StreamParams p) {
  __shared__ double tgt[kRows], ush[kRows], xsh[kRows], zsh[kRows];
  __shared__ double red[7 * (kRows / 32)];
  __shared__ ChunkHead hsh;
  __shared__ bool lastflag;
  if (p.ctl->done) return;
  if (p.n_staged == 0 && blockIdx.x == 0 && threadIdx.x == 0) stamp_chunks_start(p.ctl);
  const StreamChunk ch = p.chunks[p.big_ids[blockIdx.x]];
  const unsigned char* img = p.blob + ch.image_off;
  if (threadIdx.x < sizeof(ChunkHead) / 4)
    reinterpret_cast<int32_t*>(&hsh)[threadIdx.x] = reinterpret_cast<const int32_t*>(img)[threadIdx.x];
  __syncthreads();
  double v[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  auto sync = [] { __syncthreads(); };
  auto ld = [](const double* a) { return __ldcs(a); };
  chunk_iteration<kRows>(p, img, hsh, p.z + ch.row0, p.lam + ch.row0, p.ximp + ch.bimp0, tgt, ush, xsh,
                               zsh, v, sync, ld);
  __syncthreads();
  write_partials<kRows>(p, v, red, p.staged_grid + blockIdx.x, sync);
  __syncthreads();  // red is reused by the fold
  arrive_and_finish(p, red, &lastflag);
}

// ---------------------------------------------------------------- staged kernel
//
// Persistent, two CTAs per SM, each 8 compute warps + 1 producer warp. Every
// chunk the CTA owns (static round robin over staged_ids) is brought into one
// of the CTA's pipeline stages in shared memory by four bulk copies
// (cp.async.bulk, TMA engine): the chunk image, its z and lambda slices and
// its imported boundary x, completing on the stage's "full" mbarrier (armed
// with the byte count). While the compute warps work on chunk i entirely out
// of shared memory, the next chunk is in flight; the compute warps release a
// stage through its "empty" mbarrier.

__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(ptr));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* b, unsigned parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  unsigned long long spins = 0;
  while (!mbar_try(b, parity))
    if (++spins > (1ull << 28)) __trap();  // watchdog: never hang the device
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// clock read ordered after the preceding barrier (a dependent shared load)
__device__ __forceinline__ long long clock_after(const void* smem_word) {
  long long c;
  asm volatile("{ .reg .u32 t; ld.volatile.shared.u32 t, [%1]; mov.u64 %0, %%clock64; }"
               : "=l"(c)
               : "r"(smem_u32(smem_word))
               : "memory");
  return c;
}

// barrier of the compute warps only (the producer warp never joins)
__device__ __forceinline__ void compute_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kStagedRows) : "memory");
}

template <int kCtasPerSm, bool kProf>
__global__ void __launch_bounds__(kStagedThreads, kCtasPerSm) k_staged(const StreamParams p) {
  extern __shared__ __align__(128) unsigned char stages[];  // [p.stages][p.stage_bytes]
  __shared__ double tgt[kStagedRows], ush[kStagedRows], xsh[kStagedRows], zsh[kStagedRows];
  __shared__ double red[7 * (kStagedRows / 32)];
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages];
  __shared__ bool lastflag;
  if (p.ctl->done) return;
  const int tid = threadIdx.x;
  if (tid == 0 && blockIdx.x == 0) stamp_chunks_start(p.ctl);
  if (tid == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int G = gridDim.x;

  if (tid >= kStagedRows) {  // ---------------- producer warp (one elected lane)
    if ((tid & 31) != 0) return;
    int k = blockIdx.x;
    StreamChunk ch{};
    if (k < p.n_staged) ch = p.chunks[p.staged_ids[k]];
    for (int i = 0; k < p.n_staged; k += G, ++i) {
      const int s = i % p.stages;
      const unsigned use = static_cast<unsigned>(i / p.stages);
      // next chunk's descriptor: its load overlaps the wait and the issue below
      StreamChunk next{};
      if (k + G < p.n_staged) next = p.chunks[p.staged_ids[k + G]];
      if (use > 0) mbar_wait(&empty[s], (use - 1) & 1u);
      StagePlan sp;
      stage_plan(ch, sp);
      unsigned char* st = stages + s * p.stage_bytes;
      mbar_expect_tx(&full[s], sp.total);
      // four bulk copies: image, z slice, lambda slice, imported boundary x
      bulk_g2s(st, p.blob + ch.image_off, static_cast<unsigned>(ch.image_bytes), &full[s]);
      auto slice = [&](const StageSeg& g, const double* base, int64_t first) {
        if (g.bytes)
          bulk_g2s(st + g.dst, reinterpret_cast<const unsigned char*>(base + first) - g.shift, g.bytes, &full[s]);
      };
      slice(sp.z, p.z, ch.row0);
      slice(sp.lam, p.lam, ch.row0);
      slice(sp.ximp, p.ximp, ch.bimp0);
      mbar_arrive(&full[s]);
      ch = next;
    }
    return;
  }

  // ---------------- compute warps
  double v[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  // optional phase clock (thread 0): [0] data wait, [1] rows/u, [2] interior x,
  // [3] target, [4] GEMV/dual, [5] A z - b + release
  const bool prof = kProf && tid == 0;  // compiled out unless profiling
  long long ph[6] = {0, 0, 0, 0, 0, 0}, last = 0;
  int phase = 0;
  auto sync = [&] {
    compute_sync();
    if (prof) {
      const long long c = clock_after(ush);
      ph[phase < 5 ? phase : 5] += c - last;
      last = c;
      ++phase;
    }
  };
  auto ld = [](const double* a) { return *a; };
  int i = 0;
  for (int k = blockIdx.x; k < p.n_staged; k += G, ++i) {
    const int s = i % p.stages;
    if (prof) last = clock64();
    mbar_wait(&full[s], static_cast<unsigned>(i / p.stages) & 1u);  // every compute thread acquires the stage
    if (prof) {
      const long long c = clock64();
      ph[0] += c - last;
      last = c;
      phase = 1;
    }
    const unsigned char* st = stages + s * p.stage_bytes;
    const ChunkHead& h = *reinterpret_cast<const ChunkHead*>(st);
    StreamChunk ch{};  // the fields the stage plan and the iteration use, from the image head
    ch.row0 = h.row0;
    ch.rows = h.rows;
    ch.icol0 = h.icol0;
    ch.bimp0 = h.bimp0;
    ch.nbimp = h.nbimp;
    ch.image_bytes = h.image_bytes;
    StagePlan sp;
    stage_plan(ch, sp);
    chunk_iteration<kStagedRows>(p, st, h, reinterpret_cast<const double*>(st + sp.z.dst + sp.z.shift),
                                 reinterpret_cast<const double*>(st + sp.lam.dst + sp.lam.shift),
                                 reinterpret_cast<const double*>(st + sp.ximp.dst + sp.ximp.shift), tgt, ush,
                                 xsh, zsh, v, sync, ld);
    sync();  // the stage and the scratch arrays are free again
    if (tid == 0) mbar_arrive(&empty[s]);
  }
  if (prof)
    for (int q = 0; q < 6; ++q) p.prof[static_cast<int64_t>(blockIdx.x) * 8 + q] = ph[q];
  write_partials<kStagedRows>(p, v, red, blockIdx.x, sync);
  compute_sync();  // red is reused by the fold
  arrive_and_finish(p, red, &lastflag);
}

__global__ void k_pack(const StreamParams p) {
  // this rank's exported u values -> the head of its send record (zero
  // padded); the chunk kernels' last CTA already wrote the partials behind them
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < p.max_export) p.send[e] = e < p.n_export ? p.u[p.export_rows[e]] : 0.0;
}

__global__ void k_decide(const StreamParams p, const double* recv, int nranks, int stride) {
  if (p.ctl->done) return;
  // every rank's partials (at r * stride + max_export of the gathered
  // records) combined in rank order: identical decision on every rank
  const double* ranks = recv + p.max_export;
  double v[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  for (int r = 0; r < nranks; ++r) {
    const double* rp = ranks + static_cast<int64_t>(r) * stride;
#pragma unroll
    for (int q = 0; q < 5; ++q) v[q] = v[q] + rp[q];
    v[5] = sel_max(v[5], rp[5]);
    v[6] = v[6] + rp[6];
  }
  finalize_iteration(p, v);
}

__global__ void k_regather(const StreamRegather g) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < g.nblob; i += stride) {
    const int32_t src = g.blob_src[i];
    if (src >= 0) g.blob[i] = g.raw[src];
    else if (src == -1) g.blob[i] = 0.0;  // -2: metadata, kept
  }
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < g.rows; i += stride)
    g.z0[i] = g.raw[g.off_z0 + g.ref_of_dev[i]];
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < g.bcols; i += stride) {
    const int32_t c = g.gcol[i];
    g.cost[i] = g.raw[g.off_c + c];
    g.inv[i] = g.raw[g.off_inv + c];
    g.lo[i] = g.raw[g.off_lo + c];
    g.hi[i] = g.raw[g.off_hi + c];
  }
}

// results to reference order on the device: z, lambda by device row -> reference
// copy index, x by column -> global column
__global__ void k_stream_results(const double* z, const double* lam, const double* x, const int32_t* ref_of_dev,
                                 const int32_t* gcol, int64_t rows, int64_t cols, double* zout, double* lout,
                                 double* xout) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t d = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; d < rows; d += stride) {
    const int32_t ref = ref_of_dev[d];
    zout[ref] = z[d];
    lout[ref] = lam[d];
  }
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < cols; q += stride)
    xout[gcol[q]] = x[q];
}

__global__ void k_div_rho_check(const double* a, int64_t n, double rho, double rinv, double* out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = div_rho(a[i], rho, rinv);
}

}  // namespace

cudaError_t stream_launch_results(const double* z, const double* lam, const double* x, const int32_t* ref_of_dev,
                                  const int32_t* gcol, int64_t rows, int64_t cols, double* zout, double* lout,
                                  double* xout, int sm_count, cudaStream_t s) {
  k_stream_results<<<4 * sm_count, 256, 0, s>>>(z, lam, x, ref_of_dev, gcol, rows, cols, zout, lout, xout);
  return cudaGetLastError();
}

cudaError_t launch_div_rho_check(const double* a, int64_t n, double rho, double rinv, double* out, cudaStream_t s) {
  k_div_rho_check<<<1024, 256, 0, s>>>(a, n, rho, rinv, out);
  return cudaGetLastError();
}

cudaError_t stream_launch_regather(const StreamRegather& g, int sm_count, cudaStream_t s) {
  k_regather<<<8 * sm_count, 256, 0, s>>>(g);
  return cudaGetLastError();
}

using LocalKernel = void (*)(const StreamParams);

LocalKernel local_kernel(int threads) { return threads > kStreamRows ? &k_local<kWideRows> : &k_local<kStreamRows>; }

// kernel attributes are per device: set on every upload (the caller has made
// the context's device current)
cudaError_t stream_prepare() {
  cudaError_t e2 = cudaSuccess;
  for (auto k : {&k_staged<2, false>, &k_staged<2, true>})
    if (e2 == cudaSuccess) e2 = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (auto k : {&k_staged<3, false>, &k_staged<3, true>})
    if (e2 == cudaSuccess) e2 = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  return e2;
}

using StagedKernel = void (*)(const StreamParams);
StagedKernel staged_kernel(int ctas_per_sm, bool prof) {
  if (ctas_per_sm >= 3) return prof ? &k_staged<3, true> : &k_staged<3, false>;
  return prof ? &k_staged<2, true> : &k_staged<2, false>;
}

void launch_local_all(const StreamParams& p, cudaStream_t s) {
  if (p.n_big > 0) local_kernel(p.local_threads)<<<p.n_big, p.local_threads, 0, s>>>(p);
  if (p.n_staged > 0)
    staged_kernel(p.staged_ctas, p.prof != nullptr)<<<p.staged_grid, kStagedThreads, p.stages * p.stage_bytes, s>>>(p);
}

void stream_launch_iteration(const StreamParams& p, cudaStream_t s) {
  k_global<<<p.col_blocks, kStreamRows, 0, s>>>(p);
  launch_local_all(p, s);  // the last chunk CTA folds the partials and decides
}

void stream_launch_global(const StreamParams& p, cudaStream_t s) {
  k_global<<<p.col_blocks, kStreamRows, 0, s>>>(p);
}
void stream_launch_local(const StreamParams& p, cudaStream_t s) {
  launch_local_all(p, s);  // the last chunk CTA writes this rank's partials
  if (p.max_export > 0) k_pack<<<(p.max_export + 255) / 256, 256, 0, s>>>(p);
}
void stream_launch_direct(const StreamParams& p, cudaStream_t s) {
  if (p.n_big > 0) local_kernel(p.local_threads)<<<p.n_big, p.local_threads, 0, s>>>(p);
}
void stream_launch_staged(const StreamParams& p, cudaStream_t s) {
  if (p.n_staged > 0)
    staged_kernel(p.staged_ctas, p.prof != nullptr)<<<p.staged_grid, kStagedThreads, p.stages * p.stage_bytes, s>>>(p);
}
void stream_launch_pack(const StreamParams& p, cudaStream_t s) {
  if (p.max_export > 0) k_pack<<<(p.max_export + 255) / 256, 256, 0, s>>>(p);
}
void stream_launch_decide(const StreamParams& p, const double* recv, int nranks, int stride, cudaStream_t s) {
  k_decide<<<1, 1, 0, s>>>(p, recv, nranks, stride);
}

int stream_graph_unroll() {
  static const int u = [] {
    const char* env = std::getenv("DOPF_GRAPH_UNROLL");
    return env ? std::max(1, std::min(16, std::atoi(env))) : 4;
  }();
  return u;
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
  cudaKernelNodeParams kg = {}, kb = {}, ks = {};
  kg.func = reinterpret_cast<void*>(k_global);
  kg.gridDim = dim3(p.col_blocks);
  kg.blockDim = dim3(kStreamRows);
  kg.kernelParams = args;
  kb = kg;
  kb.func = reinterpret_cast<void*>(local_kernel(p.local_threads));
  kb.gridDim = dim3(p.n_big);
  kb.blockDim = dim3(p.local_threads);
  ks = kg;
  ks.func = reinterpret_cast<void*>(staged_kernel(p.staged_ctas, p.prof != nullptr));
  ks.gridDim = dim3(p.staged_grid);
  ks.blockDim = dim3(kStagedThreads);
  ks.sharedMemBytes = p.stages * p.stage_bytes;
  // the direct-load chunks run beside the staged kernel (which leaves one SM
  // for them), not after it
  // the body holds `unroll` iterations (the condition is evaluated once per
  // body; kernels after the stop return at once, so the result is the same)
  const int unroll = stream_graph_unroll();
  cudaGraphNode_t prev[2];
  int nprev = 0;
  for (int it = 0; it < unroll; ++it) {
    // k_global, then the chunk kernels side by side; the last chunk CTA to
    // finish folds the partials and decides (no final kernel)
    cudaGraphNode_t ng, dep[2];
    int ndep = 0;
    if ((e = cudaGraphAddKernelNode(&ng, body, prev, nprev, &kg)) != cudaSuccess) return e;
    if (p.n_big > 0 && (e = cudaGraphAddKernelNode(&dep[ndep++], body, &ng, 1, &kb)) != cudaSuccess) return e;
    if (p.n_staged > 0 && (e = cudaGraphAddKernelNode(&dep[ndep++], body, &ng, 1, &ks)) != cudaSuccess) return e;
    for (int q = 0; q < ndep; ++q) prev[q] = dep[q];
    nprev = ndep;
  }
  e = cudaGraphInstantiate(exec, g, 0);
  cudaGraphDestroy(g);
  return e;
}

}  // namespace dopf::cuda
