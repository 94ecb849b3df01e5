// Persistent fp64 ADMM iteration kernel for sm_100a.
//
// One launch runs the whole loop of reference proj/src/admm.cpp:190-235 on
// the device. Each CTA ("block": a piece of the depth-first walk of the
// component graph, layout.hpp) is warp-specialised:
//
//  compute warps 1..15, per iteration t
//   (L) local update, admm.cpp:131-138 (K1): target = x[l2g] + lambda/rho,
//       z = P target + v, a sequential-j dot product per row (the K rows of a
//       thread are interleaved for ILP); P staged in shared memory once per
//       launch (or read from HBM/L2 when it does not fit).
//   (D) dual update, admm.cpp:140-143, and the exchange value
//       u = z - lambda/rho, kept in shared memory; rows another block reads
//       ("exported") are also stored to global memory.
//   --- arrive(publish): the service warp releases this block's flag(t) ---
//   (A) ||A_s z_s - b_s||_inf (admm.cpp:203-205) and the residual partial
//       sums (admm.cpp:150-163) -- off the critical path, overlapping the
//       exchange.
//   --- sync(exchanged): every neighbour block published u(t) ---
//   (G) global update for t+1, admm.cpp:118-129 (K2): for every column the
//       block's rows reference, acc = sum of u over the column's copies in
//       ascending s (own copies from shared memory, a neighbour's from L2),
//       x = clamp((acc - c/rho) * inv, lo, hi). Shared columns are computed
//       redundantly (bitwise identical) by every block that needs them, so x
//       is never broadcast.
//
//  service warp 0, per iteration t
//   (F) after the compute warps' u(t) stores: release the block's flag(t);
//   (R) reduce the 15 warp partials in a fixed order into the block's slot(t)
//       and count it in the instance's slot counter (red.release.gpu.add);
//   (W) poll the NEIGHBOURS' flag(t) (one relaxed load per lane, then one
//       acquire fence) and fetch the decision record of t-2, then let the
//       compute warps start (G);
//   (S) once the counter shows every block's slot of t-1, combine them in a
//       fixed order (residuals, stop test admm.hpp:63, objective; the leader
//       CTA writes the trace row). Every CTA combines for itself -- bitwise
//       identical decisions, no second hop -- and polls ONE counter word
//       instead of scanning all blocks' flags. The compute warps act on the
//       decision for t-2 after the exchange of t, so the residual reduction
//       never sits on the critical path. State of the
//       last iterations is kept (x in a 3-deep ring, z/lambda in 3 result
//       buffers), so the output is exactly the iterate of the stopping
//       iteration.
//
// Memory ordering of the exchange: compute warps store u(t) (plain st.global),
// bar.arrive(publish) synchronises with the service warp's bar.sync, whose
// lane 0 then does st.release.gpu of flag(t) (cumulative release). A reader
// observes flag >= t with relaxed loads, executes fence.acq_rel.gpu, then
// bar.arrive(exchanged) -> the compute warps' bar.sync; their ld.global.cg of
// u(t) follow. Remote u is double-buffered by iteration parity: a block
// overwrites u(t) (at t+2) only after seeing every neighbour's flag(t+1),
// i.e. after each neighbour finished reading u(t).
//
// Bitwise parity with the CPU oracle: compiled with --fmad=false; every
// iterate operation keeps the reference's form (division by rho, multiply by
// the inverse copy count, std::min/std::max select semantics, sequential sums
// in the reference order). Only the residual/objective reductions use a
// different (tree) order; they feed the stop test and the trace only.
#include "admm_kernels.cuh"
#include "stop_test.cuh"

#include "div_rho.cuh"

namespace dopf::cuda {

namespace {

constexpr int kWarps = kThreads / 32;
constexpr int kHoist = kThreads > 512 ? 4 : 8;  // operator loads in flight per row (register budget)
constexpr int kCW = kComputeThreads;  // compute threads (warps 2..)
constexpr int kSyncThreads = kCW + 32;  // service + compute warps (the check warp runs decoupled)
constexpr int kSlots = kSlotRing;  // partial-slot ring (see header)
constexpr int kDec = 8;             // decision ring (shared memory), > kLag
static_assert(kDec > kLag, "decision ring too small");
constexpr int kDecG = 8;            // decision ring (global, written by the leader CTA)
constexpr int kLine = 16;           // u64 words per 128-byte line: flags are one per line
enum : int { kBarCompute = 1, kBarExchanged = 3, kBarPartials = 4,
             kBarZReady = 5,   // 5, 6 by iteration parity: z^t written (compute arrive, check warp syncs)
             kBarZFree = 7 };  // 7, 8 by iteration parity: z^t checked (check warp arrives, compute syncs)
// phase clock slots (per CTA): compute warp 1 lane 0, service lane 0
enum : int { kPhTarget = 0, kPhGemv, kPhDual, kPhEqRed, kPhWait, kPhGlobal, kPhSvcNbr, kPhSvcAll };

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
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Phase clock read that cannot run ahead of a deferred-blocking bar.sync:
// the shared-memory load blocks until the barrier completes, and the clock is
// read in the same asm block after it.
__device__ __forceinline__ long long clock_after_barrier(const void* smem_word) {
  long long c;
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(smem_word));
  asm volatile("{ .reg .u32 t; ld.volatile.shared.u32 t, [%1]; mov.u64 %0, %%clock64; }"
               : "=l"(c) : "r"(a) : "memory");
  return c;
}

// Spin-wait watchdog: a protocol bug must fail the launch loudly
// (cudaErrorLaunchFailure) instead of hanging the device.
constexpr unsigned kSpinLimit = 1u << 28;
__device__ __forceinline__ void spin_check(unsigned& spins) {
  if (++spins > kSpinLimit) __trap();
}

// Tagged exchange record {iteration, value}: one single-copy-atomic 128-bit
// access, so a reader that sees the expected tag also sees the value -- no
// separate flag round trip.
__device__ __forceinline__ void st_tagged(unsigned long long* rec, unsigned long long tag, double v) {
  asm volatile("{ .reg .b128 d; mov.b128 d, {%1, %2}; st.relaxed.gpu.global.b128 [%0], d; }"
               ::"l"(rec), "l"(tag), "l"(__double_as_longlong(v)) : "memory");
}
__device__ __forceinline__ unsigned long long ld_tagged(const unsigned long long* rec, double& v) {
  unsigned long long tag, bits;
  asm volatile("{ .reg .b128 d; ld.relaxed.gpu.global.b128 d, [%2]; mov.b128 {%0, %1}, d; }"
               : "=l"(tag), "=l"(bits) : "l"(rec) : "memory");
  v = __longlong_as_double(static_cast<long long>(bits));
  return tag;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// Sums of 8 values over the 32 lanes of a warp by recursive halving (9
// double shuffles instead of 40). On return lane L holds the total of value
// index sum8_index(L); the four lanes sharing an index hold identical bits
// (every step is a commutative a + b). Fixed pattern => deterministic.
__device__ __forceinline__ int sum8_index(int lane) {
  return ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
}
__device__ __forceinline__ int sum8_lane(int index) {
  return ((index >> 2) & 1) * 16 + ((index >> 1) & 1) * 8 + (index & 1) * 4;
}
__device__ __forceinline__ double sum8(const double (&v)[8], int lane) {
  double w[4];
  const bool h1 = (lane >> 4) & 1;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double keep = h1 ? v[q + 4] : v[q];
    const double send = h1 ? v[q] : v[q + 4];
    w[q] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
  const bool h2 = (lane >> 3) & 1;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const double keep = h2 ? w[q + 2] : w[q];
    const double send = h2 ? w[q] : w[q + 2];
    w[q] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  const bool h3 = (lane >> 2) & 1;
  double x = (h3 ? w[1] : w[0]) + __shfl_xor_sync(0xffffffffu, h3 ? w[0] : w[1], 4);
  x = x + __shfl_xor_sync(0xffffffffu, x, 2);
  x = x + __shfl_xor_sync(0xffffffffu, x, 1);
  return x;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = sel_max(v, __shfl_xor_sync(0xffffffffu, v, off));
  return v;
}

// The whole solve of one block descriptor `blk` (one CTA's share of one
// instance) -- the body of the persistent kernel below.
template <int K, bool kSmemOps>
__device__ __forceinline__ void solve_block(const KernelParams& p, const int blk) {
  extern __shared__ __align__(16) double smem[];
  const BlockDesc bd = p.blocks[blk];
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
  // tu: GEMV target during (L), then the exchange value u from (D) to (G)
  double* tu = smem + off;
  off += bd.rows;
  double* zbuf = smem + off;  // [2][rows]: z^t in buffer t & 1 (the service warp checks A z^t
  off += 2 * static_cast<std::size_t>(bd.rows);  // while the compute warps write z^{t+1})
  double* vs = smem + off;
  off += bd.rows;
  double* xring = smem + off;  // [kXRing][cols]: x^s in slot s % kXRing
  off += kXRing * static_cast<std::size_t>(bd.cols);
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
  double* red = smem + off;  // [2][kWarps][kPartials] warp partials, by iteration parity
  off += 2 * kWarps * kPartials;
  double* dec = smem + off;  // [kDec][4]: done, objective, running max, spare
  off += kDec * 4;
  long long* ph = reinterpret_cast<long long*>(smem + off);  // [8] phase clock
  off += 8;
  double* emax = smem + off;  // [kLag + 1] block infeasibility of the last iterations (check warp)
  off += kLag + 1;
  double* adone = smem + off;  // t_last + 1 once the compute warps left their loop (ends the check warp)
  off += 1;
  double* a_rhs = smem + off;  // equality-row rhs b_r
  off += bd.arows;
  AMeta* a_meta = reinterpret_cast<AMeta*>(smem + off);  // 16 B each
  off += 2 * static_cast<std::size_t>(bd.arows);
  int32_t* cps = reinterpret_cast<int32_t*>(smem + off);

  const double rho = p.rho;
  const double eps = p.eps_rel;
  for (int i = tid; i < bd.copy_len; i += kThreads) cps[i] = p.copies[bd.copy_off + i];
  for (int r = tid; r < bd.rows; r += kThreads) {
    vs[r] = p.v[bd.row0 + r];
    tu[r] = p.z0[bd.row0 + r];  // u^0 = z^0 - 0/rho
  }
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
  if (tid < kLag + 1) emax[tid] = 0.0;
  if (tid == 0) adone[0] = 0.0;
  for (int i = tid; i < 2 * kWarps * kPartials; i += kThreads) red[i] = 0.0;  // the check warp adds zeros
  if (tid < 8) ph[tid] = 0;

  const int G = id.blocks;
  const int64_t slot_stride = static_cast<int64_t>(p.blocks_per_instance) * kPartials;
  double* slots = p.part + static_cast<int64_t>(bd.instance) * kSlots * slot_stride;
  unsigned long long* flags =
      p.flags + static_cast<int64_t>(bd.instance) * p.blocks_per_instance * kLine;
  unsigned long long* ctl = p.ctl + static_cast<int64_t>(bd.instance) * kCtlWords;
  double* trace = p.trace ? p.trace + static_cast<int64_t>(bd.instance) * p.trace_stride * 6 : nullptr;
  const SyncMode mode = static_cast<SyncMode>(p.sync_mode);
  const bool exchange = mode != SyncMode::block;  // flags needed across CTAs
  const bool clock_on = p.prof != nullptr;
  __syncthreads();

  int stop_at = 0;  // set by the branch that detects the stop; broadcast below
  double m_old = 0.0;  // check warp (lane 0): infeasibility max over iterations <= s - kLag - 1
  if (warp == 0) {
    // ======================= service warp =======================
    const bool leader_cta = bd.inst_block == 0;  // writes the trace and the scalar results
    const bool tick = clock_on && lane == 0;
    unsigned long long* counter = ctl;            // slots published, G per iteration
    int ties = 0, first_tie = 0;                  // lane 0: near-tie stop tests (stop_test.cuh)
    bool stop_seen = false;
    // (S) combine every block's slot of iteration s in a fixed order (every
    // CTA does this itself, bitwise identically): residuals, stop test,
    // objective -> the block's decision ring; the leader writes the trace row
    auto combine = [&](int s) {
      if (exchange) {
        if (lane == 0) {
          unsigned spins = 0;
          while (ld_acquire_u64(counter) < static_cast<unsigned long long>(G) * s) spin_check(spins);
        }
        __syncwarp();
      }
      const double* base = slots + static_cast<int64_t>(s % kSlots) * slot_stride;
      double t8[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      for (int g0 = lane; g0 < G; g0 += 64) {  // two slots per lane in flight
        const int g1 = g0 + 32;
        const double* r0 = base + g0 * kPartials;
        const double* r1 = base + g1 * kPartials;
        double a0[6], a1[6];
#pragma unroll
        for (int q = 0; q < 6; ++q) {
          a0[q] = ld_l2(r0 + q);
          a1[q] = g1 < G ? ld_l2(r1 + q) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 6; ++q) t8[q] = t8[q] + a0[q];
        if (g1 < G) {
#pragma unroll
          for (int q = 0; q < 6; ++q) t8[q] = t8[q] + a1[q];
        }
      }
      const double mine = sum8(t8, lane);
      double tot[6];
#pragma unroll
      for (int q = 0; q < 6; ++q) tot[q] = __shfl_sync(0xffffffffu, mine, sum8_lane(q));
      if (lane == 0) {
        const double pres = sqrt(tot[0]);
        const double dres = rho * sqrt(tot[1]);
        const double eps_prim = eps * sel_max(sqrt(tot[2]), sqrt(tot[3]));
        const double eps_dual = eps * sqrt(tot[4]);
        double* rec = dec + (s % kDec) * 4;
        const bool stop = pres <= eps_prim && dres <= eps_dual;
        rec[0] = stop ? 1.0 : 0.0;
        rec[1] = tot[5];
        if (!stop_seen) {  // iterations 1..stop (combine runs in ascending s)
          if (stop_near_tie(pres, eps_prim, dres, eps_dual)) {
            ++ties;
            if (first_tie == 0) first_tie = s;
          }
          stop_seen = stop;
        }
        if (leader_cta && trace) {
          double* row = trace + static_cast<int64_t>(s - 1) * 6;
          row[0] = s;
          row[1] = pres;
          row[2] = dres;
          row[3] = eps_prim;
          row[4] = eps_dual;
          row[5] = tot[5];
        }
      }
      __syncwarp();
    };

    int t = 1;
    for (;; ++t) {
      const long long c0 = tick ? clock64() : 0;
      named_sync(kBarPartials, kSyncThreads);  // warp partials of t in red[t & 1]
      const long long c1 = tick ? clock_after_barrier(ph) : 0;
      const bool cw_stop = (t > kLag && dec[((t - kLag) % kDec) * 4] != 0.0) || t == p.max_iter;
      named_arrive(kBarExchanged, kSyncThreads);
      // residuals / stop test of t-1 (read by the compute warps at t+1) --
      // BEFORE counting slot(t): a block's count for t then also certifies it
      // finished reading every slot of t-1, so the slot ring cannot be
      // overwritten under a slower block's combine
      if (t >= 2) combine(t - 1);
      // (R) fixed-order reduction of the 15 warp partials -> slot(t), counted
      {
        const double* rb = red + (t & 1) * kWarps * kPartials;
        double w8[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) w8[q] = (lane >= 1 && lane < kWarps && q < 6) ? rb[lane * kPartials + q] : 0.0;
        const double mine = sum8(w8, lane);
        double* my_slot = slots + static_cast<int64_t>(t % kSlots) * slot_stride +
                          static_cast<int64_t>(bd.inst_block) * kPartials;
        if ((lane & 3) == 0 && sum8_index(lane) < 6) my_slot[sum8_index(lane)] = mine;
        __syncwarp();
        if (exchange && lane == 0) {
          __threadfence();  // the other lanes' slot stores, then the counted release
          red_release_add_u64(counter, 1ull);
        }
      }
      if (tick) {
        ph[kPhSvcNbr] += c1 - c0;
        ph[kPhSvcAll] += clock64() - c1;
      }
      if (cw_stop) break;
    }
    if (t > kLag && dec[((t - kLag) % kDec) * 4] != 0.0) {
      stop_at = t - kLag;
    } else {
      // reached max_iter: the first stop among the undecided iterations, else t
      combine(t);
      stop_at = t;
      for (int q = t; q > t - kLag && q >= 1; --q)
        if (dec[(q % kDec) * 4] != 0.0) stop_at = q;
    }
    if (lane == 0) {
      red[0] = stop_at;
      if (leader_cta) {
        p.iters[bd.instance] = stop_at;
        p.status[bd.instance] = dec[(stop_at % kDec) * 4] != 0.0 ? 0 : 1;
        p.objective[bd.instance] = dec[(stop_at % kDec) * 4 + 1];
        p.ties[2 * bd.instance] = ties;
        p.ties[2 * bd.instance + 1] = first_tie;
      }
    }
  } else if (warp == 1) {
    // ======================= equality-check warp =======================
    // Decoupled from the exchange: it waits only for z^t (barrier
    // kBarZReady + t % 2) and releases its buffer (kBarZFree + t % 2) for
    // the compute warps' GEMV of t + 2; barriers alternate by parity so no
    // side can arrive twice on one barrier before the other has passed it.
    // (A) local equality residual ||A_s z_s - b_s||_inf of iteration s
    // (admm.cpp:203-205) over the block's equality rows, from z^s in shared
    // memory -- off the compute warps' critical path. Lane l takes rows l,
    // l + 32, ... (the rows of one sliced-ELL lane: conflict-free); four rows
    // in flight per lane. The infeasibility is a max over iterations
    // (admm.cpp:219-220): m_old holds iterations <= s - kLag - 1, emax the last
    // kLag + 1, folded once the stopping iteration is known.
    auto acheck = [&](int s) {
      const double* zsrc = zbuf + static_cast<std::size_t>(s & 1) * bd.rows;
      double e = 0.0;
      for (int a0 = lane; a0 < bd.arows; a0 += 4 * 32) {
        double acc[4];
        AMeta am[4];
        int nmax = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          acc[i] = 0.0;
          const int a = a0 + 32 * i;
          am[i] = a < bd.arows ? a_meta[a] : AMeta{0, 0, 0, 0};
          nmax = am[i].n > nmax ? am[i].n : nmax;
        }
        for (int j = 0; j < nmax; ++j) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (j < am[i].n) acc[i] = acc[i] + Aop[am[i].aofs + 32 * j] * zsrc[am[i].base + j];
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (a0 + 32 * i < bd.arows) e = sel_max(e, fabs(acc[i] - a_rhs[a0 + 32 * i]));
      }
      e = warp_max(e);
      if (lane == 0) {
        double* slot = emax + s % (kLag + 1);
        m_old = sel_max(m_old, *slot);
        *slot = e;
      }
      __syncwarp();
    };

    for (int s = 1;; ++s) {
      named_sync(kBarZReady + (s & 1), kCW + 32);
      if (static_cast<int>(*reinterpret_cast<volatile double*>(adone)) == s) break;
      acheck(s);
      named_arrive(kBarZFree + (s & 1), kCW + 32);
    }
  } else {
    // ======================= compute warps =======================
    const int ctid = tid - 64;
    // phase clock: every iteration when profiling, else every kSampleEvery-th
    // iteration of block 0 of instance 0 (the solve's PhaseTimings split)
    const bool sampler = ctid == 0 && (clock_on || (bd.instance == 0 && bd.inst_block == 0));
    // per-thread metadata, packed to keep the K-way state in registers:
    //  row: pofs, and n (bits 0-6) | exported (7) | base (8-19) | xloc (20-31)
    //  col: copy_start (bits 0-22) | copy_count (23-30) | owner (31)
    // Interior columns (every copy in this block) are [0, cols_int), thread
    // slots c = ctid + k * kCW; boundary columns [cols_int, cols) get one slot
    // per thread, c = cols_int + ctid (the layout guarantees <= kCW of them).
    int32_t pofs[K];
    uint32_t rpk[K], cpk[K];
    double lam[K], lr[K], zp[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int r = ctid + k * kCW;
      pofs[k] = 0;
      rpk[k] = 0;
      zp[k] = 0.0;
      if (r < bd.rows) {
        const RowMeta rm = p.rmeta[bd.row0 + r];
        pofs[k] = rm.pofs;
        rpk[k] = static_cast<uint32_t>(rm.n) | (static_cast<uint32_t>(rm.exported) << 7) |
                 (static_cast<uint32_t>(rm.base) << 8) | (static_cast<uint32_t>(rm.xloc) << 20);
        zp[k] = p.z0[bd.row0 + r];
      }
      lam[k] = 0.0;
      lr[k] = 0.0 / rho;  // lambda^0 / rho
    }
    auto pack_col = [&](int c) -> uint32_t {
      const ColMeta cm = p.cmeta[bd.col_off + c];
      return static_cast<uint32_t>(cm.copy_start) | (static_cast<uint32_t>(cm.copy_count) << 23) |
             (static_cast<uint32_t>(cm.owner) << 31);
    };
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int c = ctid + k * kCW;
      cpk[k] = c < bd.cols_int ? pack_col(c) : 0u;
    }
    // boundary columns spread over the compute warps (lane-major): each warp
    // polls a few neighbours' records instead of three warps polling all
    const int cb = bd.cols_int + (ctid & 31) * (kCW / 32) + (ctid >> 5);
    const uint32_t cpkb = cb < bd.cols ? pack_col(cb) : 0u;

    auto row_n = [](uint32_t v) { return static_cast<int>(v & 0x7fu); };
    auto row_exported = [](uint32_t v) { return (v >> 7) & 1u; };
    auto row_base = [](uint32_t v) { return static_cast<int>((v >> 8) & 0xfffu); };
    auto row_xloc = [](uint32_t v) { return static_cast<int>(v >> 20); };
    auto col_start = [](uint32_t v) { return static_cast<int>(v & 0x7fffffu); };
    auto col_count = [](uint32_t v) { return static_cast<int>((v >> 23) & 0xffu); };

    // x_c = clamp((acc - c/rho) * inv, lo, hi) (admm.cpp:126-127); returns c_c x_c for owners
    auto finish_col = [&](int c, uint32_t pk, double acc, double* xdst) -> double {
      const double unclamped = (acc - c_rho[c]) * c_inv[c];
      const double xv = sel_min(sel_max(unclamped, c_lo[c]), c_hi[c]);
      xdst[c] = xv;
      return (pk >> 31) ? c_cost[c] * xv : 0.0;
    };
    // (G, interior) every copy in shared memory: acc = sum in ascending s
    auto global_interior = [&](double* xdst) -> double {
      double obj = 0.0;
      double a[K][4];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int c = ctid + k * kCW;
        const int cnt = c < bd.cols_int ? col_count(cpk[k]) : 0;
        const int32_t* q = cps + col_start(cpk[k]);
#pragma unroll
        for (int e = 0; e < 4; ++e) a[k][e] = e < cnt ? tu[q[e]] : 0.0;
      }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int c = ctid + k * kCW;
        if (c < bd.cols_int) {
          const int cnt = col_count(cpk[k]);
          const int32_t* q = cps + col_start(cpk[k]);
          double acc = 0.0;
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (e < cnt) acc = acc + a[k][e];
          for (int e = 4; e < cnt; ++e) acc = acc + tu[q[e]];
          obj = obj + finish_col(c, cpk[k], acc, xdst);
        }
      }
      return obj;
    };
    // (G, boundary) copies of other blocks are tagged records of iteration
    // `it` in L2 (polled until the tag matches), own copies from shared
    // memory; the first four loads of the column are issued before any wait
    auto global_boundary = [&](int it, double* xdst) -> double {
      if (cb >= bd.cols) return 0.0;
      const unsigned long long* ub = p.ux + static_cast<int64_t>(it & 1) * 2 * p.rows_total;
      const unsigned long long want = static_cast<unsigned long long>(it);
      const int cnt = col_count(cpkb);
      const int32_t* q = cps + col_start(cpkb);
      // every copy's load is in flight before the first wait (<= 8 copies per
      // column in the feeders here; more are read after the first eight)
      constexpr int H = kThreads > 512 ? 4 : 8;
      double a[H];
      unsigned long long tg[H];
#pragma unroll
      for (int e = 0; e < H; ++e) {
        a[e] = 0.0;
        tg[e] = want;
        if (e < cnt) {
          const int32_t ref = q[e];
          if (ref >= 0)
            a[e] = tu[ref];
          else
            tg[e] = ld_tagged(ub + 2 * static_cast<int64_t>(decode_remote(ref)), a[e]);
        }
      }
      double acc = 0.0;
#pragma unroll
      for (int e = 0; e < H; ++e) {
        if (e < cnt) {
          unsigned spins = 0;
          while (tg[e] != want) {
            spin_check(spins);
            tg[e] = ld_tagged(ub + 2 * static_cast<int64_t>(decode_remote(q[e])), a[e]);
          }
          acc = acc + a[e];
        }
      }
      for (int e = H; e < cnt; ++e) {
        const int32_t ref = q[e];
        double v;
        if (ref >= 0) {
          v = tu[ref];
        } else {
          unsigned spins = 0;
          while (ld_tagged(ub + 2 * static_cast<int64_t>(decode_remote(ref)), v) != want) spin_check(spins);
        }
        acc = acc + v;
      }
      return finish_col(cb, cpkb, acc, xdst);
    };

    // x^1 from u^0 = z^0 (tu holds z^0; remote copies: records {0, z^0} written by the host)
    double obj = global_interior(xring + bd.cols);
    obj = obj + global_boundary(0, xring + bd.cols);
    named_sync(kBarCompute, kCW);
    long long c0 = sampler ? clock64() : 0, c1 = 0;
    int t = 1;
    for (;; ++t) {
      const bool tick = sampler && (clock_on || t % kSampleEvery == 1);
      const double* xt = xring + static_cast<std::size_t>(t % kXRing) * bd.cols;  // x^t
      double* xnext = xring + static_cast<std::size_t>((t + 1) % kXRing) * bd.cols;
      unsigned long long* u_out = p.ux + static_cast<int64_t>(t & 1) * 2 * p.rows_total;
      double* z_res = p.z_out + static_cast<int64_t>(t % kZRing) * p.rows_total;
      double* l_res = p.lam_out + static_cast<int64_t>(t % kZRing) * p.rows_total;
      double* zs = zbuf + static_cast<std::size_t>(t & 1) * bd.rows;

      // (L1) consensus target
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int r = ctid + k * kCW;
        if (r < bd.rows) tu[r] = xt[row_xloc(rpk[k])] + lr[k];  // lr = lambda / rho, same rounding
      }
      named_sync(kBarCompute, kCW);
      if (tick) {
        c1 = clock_after_barrier(ph);
        ph[kPhTarget] += c1 - c0;
        c0 = c1;
      }

      // (L2) z = P t + v, one row per thread and slot k; P in sliced-ELL order
      // (entry j of a warp's 32 rows is 256 contiguous bytes). Each row's
      // loads are issued 8 at a time ahead of its sequential-j sum. z^t goes
      // to buffer t % 2, once the check warp is done with z^{t-2} there.
      if (t >= 3) named_sync(kBarZFree + (t & 1), kCW + 32);
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int r = ctid + k * kCW;
        if (r < bd.rows) {
          const int n = row_n(rpk[k]);
          const double* pr = Pop + pofs[k];
          const double* tb = tu + row_base(rpk[k]);
          double acc = 0.0;
          for (int j0 = 0; j0 < n; j0 += kHoist) {
            double pv[kHoist], tv[kHoist];
#pragma unroll
            for (int e = 0; e < kHoist; ++e) {
              pv[e] = 0.0;
              tv[e] = 0.0;
              if (j0 + e < n) {
                pv[e] = pr[(j0 + e) * 32];
                tv[e] = tb[j0 + e];
              }
            }
#pragma unroll
            for (int e = 0; e < kHoist; ++e)
              if (j0 + e < n) acc = acc + pv[e] * tv[e];
          }
          zs[r] = acc + vs[r];
        }
      }
      named_arrive(kBarZReady + (t & 1), kCW + 32);  // z^t for the check warp
      // every row's target read before (D) overwrites tu; z visible to (A)
      named_sync(kBarCompute, kCW);
      if (tick) {
        c1 = clock_after_barrier(ph);
        ph[kPhGemv] += c1 - c0;
        c0 = c1;
      }

      // (D) dual update, exchange value (critical path: only what others need)
      double v8[8] = {0.0, 0.0, 0.0, 0.0, 0.0, obj, 0.0, 0.0};
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int r = ctid + k * kCW;
        if (r < bd.rows) {
          const double z = zs[r];
          const double bx = xt[row_xloc(rpk[k])];
          const double d = bx - z;
          const double ln = lam[k] + rho * d;
          v8[0] = v8[0] + d * d;
          const double dz = z - zp[k];
          v8[1] = v8[1] + dz * dz;
          v8[2] = v8[2] + bx * bx;
          v8[3] = v8[3] + z * z;
          v8[4] = v8[4] + ln * ln;
          lr[k] = div_rho(ln, rho, p.rho_inv);  // = ln / rho; reused as lambda/rho by the next target (admm.cpp:136)
          const double u = z - lr[k];
          tu[r] = u;
          if (row_exported(rpk[k]))
            st_tagged(u_out + 2 * static_cast<int64_t>(bd.row0 + r), static_cast<unsigned long long>(t), u);
          lam[k] = ln;
          zp[k] = z;
        }
      }
      if (p.snap != nullptr && t <= p.snap_iters) {
        // parity mode (reference record_iterates, admm.cpp:228-229): the
        // state after iteration t -- z^t, lambda^t by device row, x^t by
        // column (owners)
        double* sn = p.snap + static_cast<int64_t>(t - 1) * p.snap_stride;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int r = ctid + k * kCW;
          if (r < bd.rows) {
            sn[bd.row0 + r] = zp[k];
            sn[p.rows_total + bd.row0 + r] = lam[k];
          }
        }
        for (int c = ctid; c < bd.cols; c += kCW) {
          const ColMeta cmc = p.cmeta[bd.col_off + c];
          if (cmc.owner) sn[2 * p.rows_total + id.x_off + cmc.gcol] = xt[c];
        }
      }
      named_sync(kBarCompute, kCW);  // every u(t) in shared memory
      unsigned long long* tl = nullptr;
      if (p.timeline && ctid == 0 && t >= kTimelineT0 && t < kTimelineT0 + kTimelineIters) {
        tl = p.timeline + (static_cast<int64_t>(blk) * kTimelineIters + (t - kTimelineT0)) * 3;
        tl[0] = globaltimer();  // u(t) published (every warp's stores issued)
      }
      if (tick) {
        c1 = clock_after_barrier(ph);
        ph[kPhDual] += c1 - c0;
        c0 = c1;
      }
      // (G, interior) x^{t+1} of the columns no other block holds -- overlaps
      // the exchange; x^{t+1} goes to slot (t+1) % 4, so x^{t-2} (a possible
      // stopping iterate) survives
      double obj_next = global_interior(xnext);
      // result copies and partial reductions -- overlapping the exchange
      // (the equality check of z^t runs on the service warp)
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int r = ctid + k * kCW;
        if (r < bd.rows) {
          z_res[bd.row0 + r] = zp[k];  // (z, lambda)^t kept until the stop test of t is known
          l_res[bd.row0 + r] = lam[k];
        }
      }
      {
        const double mine = sum8(v8, lane);
        if ((lane & 3) == 0) red[(t & 1) * kWarps * kPartials + warp * kPartials + sum8_index(lane)] = mine;
      }
      named_arrive(kBarPartials, kSyncThreads);
      if (tick) {
        c1 = clock_after_barrier(ph);
        ph[kPhEqRed] += c1 - c0;
        c0 = c1;
      }
      // (G, boundary) x^{t+1} of the columns shared with neighbours (waits for
      // their u(t) records); x^{t+1} is speculative until the stop test
      if (tl) tl[1] = globaltimer();  // boundary update starts
      obj = obj_next + global_boundary(t, xnext);
      if (tick) {
        c1 = clock_after_barrier(ph);
        ph[kPhGlobal] += c1 - c0;
        c0 = c1;
      }
      named_sync(kBarExchanged, kSyncThreads);  // decision of t-2 in dec[]; x^{t+1} complete
      if (tl) {
        (void)clock_after_barrier(ph);
        tl[2] = globaltimer();  // every boundary column of the block done
      }
      if (tick) {
        c1 = clock_after_barrier(ph);
        ph[kPhWait] += c1 - c0;
        c0 = c1;
      } else if (sampler && (t + 1) % kSampleEvery == 1) {
        c0 = clock_after_barrier(ph);  // start of the next sampled iteration
      }
      if ((t > kLag && dec[((t - kLag) % kDec) * 4] != 0.0) || t == p.max_iter) break;
    }
    // release the check warp from its wait for z^{t+1}
    if (ctid == 0) *reinterpret_cast<volatile double*>(adone) = t + 1;
    named_arrive(kBarZReady + ((t + 1) & 1), kCW + 32);
    // consume the check warp's last "z^s checked" arrivals (s = t - 1, t; the
    // loop consumed s <= t - 2): hardware barriers keep pending arrivals, and
    // a CTA of a persistent group solves its next instance with the same ones
    for (int s = t > 1 ? t - 1 : 1; s <= t; ++s) named_sync(kBarZFree + (s & 1), kCW + 32);
  }
  __syncthreads();
  stop_at = static_cast<int>(red[0]);
  if (clock_on && tid < 8) p.prof[blk * 8 + tid] += ph[tid];
  if (p.phase_sample && bd.instance == 0 && bd.inst_block == 0 && tid < 8) p.phase_sample[tid] = ph[tid];
  if (warp == 1 && lane == 0) {
    // max_local_infeasibility over iterations 1..stop_at: the check warp saw
    // iterations up to the compute warps' last one, last - kLag <= stop_at <= last
    const int last = static_cast<int>(adone[0]) - 1;
    double mx = m_old;
    for (int q = last - kLag; q <= stop_at; ++q)
      if (q >= 1) mx = sel_max(mx, emax[q % (kLag + 1)]);
    atomicMax(reinterpret_cast<unsigned long long*>(p.maxinf + bd.instance),
              static_cast<unsigned long long>(__double_as_longlong(mx)));  // mx >= 0: bit order = value order
  }
  if (warp >= 2) {
    // owners write x^stop_at (still in the ring); (z, lambda)^stop_at are in
    // result buffer stop_at % kZRing, which the host reads
    const int ctid = tid - 64;
    const double* xfinal = xring + static_cast<std::size_t>(stop_at % kXRing) * bd.cols;
    for (int c = ctid; c < bd.cols; c += kCW) {
      const ColMeta cmc = p.cmeta[bd.col_off + c];
      if (cmc.owner) p.x_out[id.x_off + cmc.gcol] = xfinal[c];
    }
  }
}

// One CTA per block descriptor (single instance, clusters: admm_persistent),
// or -- scenario batches, admm_groups -- a persistent grid of CTA groups: group g
// (CTAs gG .. gG+G-1, co-resident through the cooperative launch) solves
// instances g, g + groups, g + 2 groups, ... one after another, restaging
// each instance's operators. Unlike one thread-block cluster per instance,
// which must fit one GPC (33 clusters of 4 = 132 of 148 SMs on this B200,
// tools/micro/cluster_occupancy.cu), every SM holds a CTA. Instances share
// no state, so which group solves one does not change its results.
template <int K, bool kSmemOps>
__global__ void __launch_bounds__(kThreads, 512 / kThreads) admm_persistent(const KernelParams p) {
  solve_block<K, kSmemOps>(p, blockIdx.x);
}

template <int K, bool kSmemOps>
__global__ void __launch_bounds__(kThreads, 512 / kThreads) admm_groups(const KernelParams p) {
  const int G = p.group_size, groups = gridDim.x / G;
  const int g = blockIdx.x / G, b = blockIdx.x - g * G;
  for (int inst = g; inst < p.instances; inst += groups) {
    solve_block<K, kSmemOps>(p, inst * G + b);
    __syncthreads();  // shared memory is restaged for the next instance
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

namespace {
template <int K, bool kSmemOps>
cudaError_t launch_groups_k(const KernelParams& p, int groups, std::size_t smem, cudaStream_t stream) {
  auto kern = admm_groups<K, kSmemOps>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (err != cudaSuccess) return err;
  KernelParams local = p;
  void* args[] = {&local};
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(groups * p.group_size), dim3(kThreads),
                                     args, smem, stream);
}
template <int K>
cudaError_t launch_groups_ops(const KernelParams& p, int groups, std::size_t smem, bool smem_ops, cudaStream_t s) {
  return smem_ops ? launch_groups_k<K, true>(p, groups, smem, s) : launch_groups_k<K, false>(p, groups, smem, s);
}
}  // namespace

cudaError_t launch_admm_groups(const KernelParams& p, int groups, int K, std::size_t smem, bool smem_ops,
                               cudaStream_t stream) {
  switch (K) {
    case 1: return launch_groups_ops<1>(p, groups, smem, smem_ops, stream);
    case 2: return launch_groups_ops<2>(p, groups, smem, smem_ops, stream);
    case 3: return launch_groups_ops<3>(p, groups, smem, smem_ops, stream);
    case 4: return launch_groups_ops<4>(p, groups, smem, smem_ops, stream);
    default: return cudaErrorInvalidValue;
  }
}

int max_dynamic_smem(int device) {
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  return v;
}

}  // namespace dopf::cuda
