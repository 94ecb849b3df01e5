// Drop-in C ABI (include/dopf_cuda.h) over the persistent ADMM kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/dopf_cuda.h"
#include "admm_kernels.cuh"
#include "layout_builder.hpp"
#include "certify_kernels.cuh"
#include "layout_gather.cuh"
#include "precompute_kernels.cuh"
#include "stream_kernels.cuh"
#include "div_rho.cuh"
#include "nccl_dyn.hpp"

using namespace dopf::cuda;

namespace {

struct SingularFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct CudaFailure : std::runtime_error {
  cudaError_t code;
  CudaFailure(cudaError_t c, const std::string& what)
      : std::runtime_error(what + ": " + cudaGetErrorString(c)), code(c) {}
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaFailure(e, what);
}

}  // namespace

struct dopf_cuda_ctx {
  int device = 0;
  int sm_count = 0;
  int smem_optin = 0;
  int smem_per_sm = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::string err;

  HostLayout L;
  bool uploaded = false;
  SyncMode mode = SyncMode::block;
  int cluster = 1;
  int num_blocks = 0;
  std::vector<int32_t> inst_nz, inst_n;

  // Device buffers grow only: a re-upload of a model of the same (or
  // smaller) size reuses them -- no cudaFree/cudaMalloc on the e2e path.
  struct Buf {
    void* p = nullptr;
    std::size_t cap = 0;  // bytes
  };
  std::vector<Buf> bufs = std::vector<Buf>(128);
  BlockDesc* d_blocks = nullptr;
  InstDesc* d_inst = nullptr;
  double *d_P = nullptr, *d_A = nullptr, *d_v = nullptr, *d_z0 = nullptr;
  int32_t* d_copies = nullptr;
  RowMeta* d_rmeta = nullptr;
  ColMeta* d_cmeta = nullptr;
  double *d_cc = nullptr, *d_cinv = nullptr, *d_clo = nullptr, *d_chi = nullptr;
  AMeta* d_ameta = nullptr;
  double* d_ab = nullptr;
  int32_t* d_nbrs = nullptr;
  double *d_u = nullptr, *d_z = nullptr, *d_lam = nullptr, *d_x = nullptr, *d_part = nullptr;
  unsigned long long* d_flags = nullptr;
  unsigned long long* d_ctl = nullptr;
  int32_t *d_iters = nullptr, *d_status = nullptr;
  double *d_maxinf = nullptr, *d_obj = nullptr;
  int32_t* d_ties = nullptr;  // [instances][2] near-tie count, first near tie
  long long* d_phase = nullptr;  // [8] sampled phase cycles of block 0 (PhaseTimings)
  double* d_trace = nullptr;
  std::size_t trace_cap = 0;  // doubles
  // cached layout plans (structure only), reused while the structure repeats
  std::shared_ptr<InstancePlan> plan, batch_plan;
  // HBM-streaming path (instances too large for shared-memory residency)
  int path_request = 0;      // 0 auto, 1 resident persistent kernel, 2 streaming graph
  double* snap_dev = nullptr;  // parity mode: per-iteration snapshots of the next resident run (slot 118)
  std::vector<double> block_weights;  // tuned cost shares of the resident split (dopf_cuda_tune_partition)
  uint64_t weights_sig = 0;           // structure they were tuned for (0: any)
  int snap_iters = 0;
  bool streaming = false;    // path of the uploaded model
  StreamLayout SL;
  struct StreamDev {
    StreamChunk* chunks = nullptr;
    int32_t* staged_ids = nullptr;
    int32_t* big_ids = nullptr;
    int32_t *imp_ptr = nullptr, *imp_slot = nullptr;
    double* ximp = nullptr;
    unsigned char* blob = nullptr;  // chunk images
    double* z0 = nullptr;
    int32_t *col_ptr = nullptr, *copies = nullptr;
    double *cost = nullptr, *inv = nullptr, *lo = nullptr, *hi = nullptr;
    uint8_t* owner = nullptr;
    double *x = nullptr, *z = nullptr, *lam = nullptr, *u = nullptr, *u_remote = nullptr;
    double *part = nullptr, *objp = nullptr;
    unsigned* final_count = nullptr;
    StreamCtl* ctl = nullptr;
    int32_t* export_rows = nullptr;
    double* send = nullptr;
  } sd;
  bool partitioned = false;
  unsigned long long* d_timeline = nullptr;
  std::size_t timeline_len = 0;
  StreamParams part_params{};
  bool part_trace = false;
  cudaStream_t own_stream = nullptr;  // the context's stream (set_stream may point elsewhere)
  cudaGraphExec_t graph = nullptr;
  double graph_key[3] = {0, 0, 0};  // rho, eps, max_iter the graph was built for
  const double* graph_trace = nullptr;
  int64_t kernels = 0;       // kernels launched (graph iterations x 3 + persistent launches)
  // re-upload fast path: the plan whose index maps / structure sit on the device
  const InstancePlan* dev_plan = nullptr;
  int staged_grid = 1;       // persistent CTAs of the staged streaming kernel
  int staged_ctas = 2;       // of them per SM
  int local_threads = kStreamRows;  // direct-load CTA size (kWideRows for a hub subsystem wider than kStreamRows)
  bool stream_maps = false;  // the streaming layout's maps are on the device
  int64_t* d_psrc = nullptr;
  int64_t* d_asrc = nullptr;
  int64_t* d_absrc = nullptr;
  int32_t* d_refdev = nullptr;
  int32_t* d_gcol = nullptr;
  int32_t* d_blobsrc = nullptr;  // streaming re-upload: chunk-image value map
  double* d_raw = nullptr;       // streaming re-upload: raw value concatenation
  double *d_rawP = nullptr, *d_rawA = nullptr, *d_rawb = nullptr, *d_rawv = nullptr, *d_rawz0 = nullptr,
         *d_rawc = nullptr, *d_rawinv = nullptr, *d_rawlo = nullptr, *d_rawhi = nullptr;
  std::vector<const void*> pinned;  // host ranges registered by dopf_cuda_pin_model
  // pinned staging for results copied back to the host
  void* h_stage = nullptr;
  void* h_small = nullptr;
  std::size_t h_stage_cap = 0;

  // NCCL communicator of a partitioned solve (dopf_cuda_comm_init) and the
  // solve's CUDA graph (kernels + ncclAllGather, dopf_cuda_solve_part)
  ncclComm_t comm = nullptr;
  int comm_nranks = 0, comm_rank = -1;
  int64_t layout_epoch = 0;          // bumped by every structural streaming upload
  cudaGraphExec_t part_graph = nullptr;
  int part_graph_mode = 0;           // 1 device while-node, 2 unrolled bodies + lazy host poll
  double part_key[6] = {0, 0, 0, 0, 0, 0};
  cudaEvent_t poll_ev[2] = {nullptr, nullptr};
  // second stream: the direct-load chunk kernel beside the staged one (fork / join)
  cudaStream_t aux = nullptr;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  int32_t* h_flags = nullptr;        // pinned: done flags of the last two unrolled launches

  int64_t launches = 0;
  double last_kernel_s = 0;
  bool profiling = false;
  long long* d_prof = nullptr;  // [blocks][8] phase cycles
  std::size_t prof_cap = 0;

  void drop_graph() {
    if (graph) cudaGraphExecDestroy(graph);
    graph = nullptr;
    if (part_graph) cudaGraphExecDestroy(part_graph);
    part_graph = nullptr;
    part_graph_mode = 0;
  }

  void free_model() {
    drop_graph();
    for (Buf& b : bufs) {
      if (b.p) cudaFree(b.p);
      b = Buf{};
    }
    if (d_trace) cudaFree(d_trace);
    d_trace = nullptr;
    trace_cap = 0;
    uploaded = false;
  }

  void* ensure(int slot, std::size_t bytes) {
    Buf& b = bufs.at(slot);
    // 64 bytes of slack: bulk copies round slice ends up to 16 bytes
    bytes = std::max<std::size_t>(bytes, 16) + 64;
    if (b.cap < bytes) {
      if (b.p) cudaFree(b.p);
      b.p = nullptr;
      b.cap = 0;
      ck(cudaMalloc(&b.p, bytes), "cudaMalloc");
      b.cap = bytes;
    }
    return b.p;
  }

  template <typename T>
  T* put(int slot, const std::vector<T>& h) {
    T* p = static_cast<T*>(ensure(slot, h.size() * sizeof(T)));
    if (!h.empty()) ck(cudaMemcpyAsync(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, stream), "upload");
    return p;
  }

  template <typename T>
  T* scratch(int slot, std::size_t count) {
    return static_cast<T*>(ensure(slot, count * sizeof(T)));
  }

  void* small_stage() {  // 256 pinned bytes for packed scalar results
    if (!h_small) ck(cudaMallocHost(&h_small, 256), "cudaMallocHost");
    return h_small;
  }

  void* stage(std::size_t bytes) {
    if (h_stage_cap < bytes) {
      if (h_stage) cudaFreeHost(h_stage);
      h_stage = nullptr;
      h_stage_cap = 0;
      ck(cudaMallocHost(&h_stage, bytes), "cudaMallocHost");
      h_stage_cap = bytes;
    }
    return h_stage;
  }
};

namespace {

int fail(dopf_cuda_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

// Makes the context's device current for one entry point and restores the
// caller's device afterwards (contexts on several devices may share a thread).
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(const dopf_cuda_ctx* c) {
    if (!c || c->sm_count == 0) return;  // not created yet (dopf_cuda_create sets it)
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != c->device) ck(cudaSetDevice(c->device), "cudaSetDevice");
    else prev = -1;
  }
  ~DeviceScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

template <typename F>
int guarded(dopf_cuda_ctx* ctx, F&& body) {
  try {
    DeviceScope scope(ctx);
    body();
    return DOPF_OK;
  } catch (const CudaFailure& e) {
    return fail(ctx, e.code == cudaErrorMemoryAllocation ? DOPF_ERR_OUT_OF_MEMORY : DOPF_ERR_CUDA,
                e.what());
  } catch (const SingularFailure& e) {
    return fail(ctx, DOPF_ERR_SINGULAR, e.what());
  } catch (const nccl::NcclFailure& e) {
    return fail(ctx, DOPF_ERR_NCCL, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(ctx, DOPF_ERR_INVALID_ARGUMENT, e.what());
  } catch (const std::bad_alloc&) {
    return fail(ctx, DOPF_ERR_OUT_OF_MEMORY, "out of host memory");
  } catch (const std::exception& e) {
    return fail(ctx, DOPF_ERR_RUNTIME, e.what());
  }
}

void check_settings(const dopf_settings* s) {
  if (!s) throw std::invalid_argument("null settings");
  if (!(s->rho > 0)) throw std::invalid_argument("rho must be positive");
  if (!(s->eps_rel > 0)) throw std::invalid_argument("eps_rel must be positive");
  if (s->max_iter < 1) throw std::invalid_argument("max_iter must be positive");
}

void upload_layout(dopf_cuda_ctx* c) {
  HostLayout& L = c->L;
  int k = 0;
  c->d_blocks = c->put(k++, L.blocks);
  c->d_inst = c->put(k++, L.inst);
  c->d_P = c->put(k++, L.P);
  c->d_A = c->put(k++, L.A);
  c->d_copies = c->put(k++, L.copies);
  c->d_rmeta = c->put(k++, L.rmeta);
  c->d_v = c->put(k++, L.v);
  c->d_z0 = c->put(k++, L.z0);
  c->d_cmeta = c->put(k++, L.cmeta);
  c->d_cc = c->put(k++, L.cc);
  c->d_cinv = c->put(k++, L.cinv);
  c->d_clo = c->put(k++, L.clo);
  c->d_chi = c->put(k++, L.chi);
  c->d_ameta = c->put(k++, L.ameta);
  c->d_ab = c->put(k++, L.ab);
  c->d_nbrs = c->put(k++, L.nbrs);
  const std::size_t I = L.inst.size();
  const std::size_t R = static_cast<std::size_t>(L.rows_total);
  c->d_u = c->scratch<double>(k++, 4 * R);    // tagged records {t, u}, two buffers
  c->d_z = c->scratch<double>(k++, kZRing * R);    // [t % kZRing][row]
  c->d_lam = c->scratch<double>(k++, kZRing * R);
  c->d_x = c->scratch<double>(k++, L.x_total);
  c->d_part = c->scratch<double>(k++, I * kSlotRing * L.blocks_per_instance * kPartials);
  c->d_flags = c->scratch<unsigned long long>(k++, I * L.blocks_per_instance * 16);
  c->d_ctl = c->scratch<unsigned long long>(k++, I * kCtlWords);
  c->d_iters = c->scratch<int32_t>(k++, I);
  c->d_status = c->scratch<int32_t>(k++, I);
  c->d_maxinf = c->scratch<double>(k++, I);
  c->d_obj = c->scratch<double>(k++, I);
  c->d_ties = c->scratch<int32_t>(k++, 2 * I);
  c->d_phase = c->scratch<long long>(k++, 8);
  ck(cudaStreamSynchronize(c->stream), "upload sync");
}

// CTAs of the resident kernel per SM (register budget: kThreads x 128 regs
// each); DOPF_CTAS_PER_SM overrides for experiments
int ctas_per_sm() {
  const char* e = std::getenv("DOPF_CTAS_PER_SM");
  if (e && (e[0] == '1' || e[0] == '2')) return e[0] - '0';
  return kThreads <= 256 ? 2 : 1;
}

void choose_sync(dopf_cuda_ctx* c) {
  const int G = c->L.blocks_per_instance;
  c->num_blocks = static_cast<int>(c->L.blocks.size());
  if (G == 1) {
    c->mode = SyncMode::block;
    c->cluster = 1;
  } else if (G <= 8) {
    c->mode = SyncMode::cluster;
    c->cluster = G;
  } else {
    if (c->L.inst.size() != 1)
      throw std::invalid_argument("batched instances must fit a cluster of <= 8 CTAs");
    if (G > c->sm_count * ctas_per_sm()) throw std::invalid_argument("instance needs more CTAs than fit the GPU");
    c->mode = SyncMode::grid;
    c->cluster = 1;
  }
}

LayoutOptions options_for(const dopf_cuda_ctx* c) {
  LayoutOptions o;
  const int cps = ctas_per_sm();
  o.smem_limit = cps == 1 ? static_cast<std::size_t>(c->smem_optin)
                          : static_cast<std::size_t>(c->smem_per_sm) / cps - 1024;  // 1 KB reserved per CTA
  o.max_blocks = c->sm_count * cps;
  o.block_weights = c->block_weights;
  if (const char* e = std::getenv("DOPF_BLOCK_WEIGHTS"); e && o.block_weights.empty()) {  // experiments
    for (const char* q = e; *q;) {
      char* end = nullptr;
      const double v = std::strtod(q, &end);
      if (end == q) break;
      o.block_weights.push_back(v);
      q = *end == ',' ? end + 1 : end;
    }
  }
  return o;
}

// FNV-1a (32-bit words) over a model's structure (sizes, z_offsets, l2g): tuned split shares
// only apply to the structure they were measured on.
uint64_t structure_sig(const dopf_model_view& m) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](const void* p, std::size_t bytes) {  // 32-bit words (all inputs are int32 arrays)
    const uint32_t* w = static_cast<const uint32_t*>(p);
    for (std::size_t i = 0; i < bytes / 4; ++i) h = (h ^ w[i]) * 1099511628211ull;
  };
  mix(&m.S, sizeof m.S);
  mix(&m.n, sizeof m.n);
  mix(&m.N_z, sizeof m.N_z);
  if (m.S > 0 && m.z_offsets) mix(m.z_offsets, (m.S + 1) * sizeof(int32_t));
  if (m.N_z > 0 && m.l2g) mix(m.l2g, m.N_z * sizeof(int32_t));
  return h | 1ull;  // never 0
}

// Limits of the resident kernel a single-instance plan must meet (the same
// ones finish_upload / choose_sync enforce), checked before any upload.
void check_resident(const dopf_cuda_ctx* c, const InstancePlan& P) {
  if (P.K > kMaxK) throw std::invalid_argument("model too large for the resident kernel");
  if (P.max_neighbours > 32) throw std::invalid_argument("a block shares columns with more than 32 other blocks");
  if (static_cast<int>(P.blocks.size()) > c->sm_count * ctas_per_sm())
    throw std::invalid_argument("instance needs more CTAs than fit the GPU");
}

void finish_upload(dopf_cuda_ctx* c) {
  if (c->L.K > kMaxK)
    throw std::invalid_argument("model too large for the resident kernel (" +
                                std::to_string(c->L.rows_total) + " rows)");
  if (c->L.max_neighbours > 32)
    throw std::invalid_argument("a block shares columns with more than 32 other blocks (" +
                                std::to_string(c->L.max_neighbours) + ")");
  choose_sync(c);
  upload_layout(c);
  c->uploaded = true;
}

// PhaseTimings (reference admm.hpp:104-106, measured at admm.cpp:182-217) of
// a resident solve: the loop's device time split by the phase clock that
// block 0 samples every kSampleEvery-th iteration -- local = consensus target
// + GEMV (admm.cpp:131-138), dual = dual update + exchange value
// (admm.cpp:140-143), global = column updates incl. the neighbour wait
// (admm.cpp:118-129). The equality check runs on its own warp, beside them.
void resident_timings(dopf_result_view& r, const long long* ph, double total_s) {
  double sum = 0;
  for (int q = 0; q < 6; ++q) sum += static_cast<double>(ph[q]);
  if (!(sum > 0)) {
    r.time_global = r.time_local = r.time_dual = 0.0;
    return;
  }
  r.time_local = total_s * static_cast<double>(ph[0] + ph[1]) / sum;
  r.time_dual = total_s * static_cast<double>(ph[2]) / sum;
  r.time_global = total_s * static_cast<double>(ph[3] + ph[4] + ph[5]) / sum;
}

// Runs the kernel; copies scalars (and optionally vectors/trace) back.
// Results of a single-instance solve (the resident path's common case).
void finish_single(dopf_cuda_ctx* c, const dopf_settings* s, dopf_result_view& r, bool copy_vectors,
                   std::chrono::steady_clock::time_point t_up0) {
  const HostLayout& L = c->L;
  const std::size_t R = static_cast<std::size_t>(L.rows_total);
  double* d_res = c->scratch<double>(122, 2 * R + 8);
  ck(launch_final_single(c->d_z, c->d_lam, L.rows_total, c->d_refdev, c->d_iters, kZRing, c->d_status,
                         c->d_maxinf, c->d_obj, c->d_ties, d_res, d_res + R, d_res + 2 * R, c->sm_count,
                         c->stream),
     "final iterate");
  ++c->kernels;
  double* scal = static_cast<double*>(c->small_stage());
  ck(cudaMemcpyAsync(scal, d_res + 2 * R, 6 * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "d2h");
  long long* ph = reinterpret_cast<long long*>(scal + 8);
  ck(cudaMemcpyAsync(ph, c->d_phase, 8 * sizeof(long long), cudaMemcpyDeviceToHost, c->stream), "d2h");
  if (copy_vectors) {
    const InstDesc& id = L.inst[0];
    if (r.x)
      ck(cudaMemcpyAsync(r.x, c->d_x + id.x_off, sizeof(double) * id.n, cudaMemcpyDeviceToHost, c->stream), "d2h");
    if (r.z) ck(cudaMemcpyAsync(r.z, d_res, R * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "d2h");
    if (r.lambda)
      ck(cudaMemcpyAsync(r.lambda, d_res + R, R * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "d2h");
  }
  ck(cudaStreamSynchronize(c->stream), "solve");
  ck(cudaGetLastError(), "kernel");
  float ms = 0;
  ck(cudaEventElapsedTime(&ms, c->ev0, c->ev1), "elapsed");
  c->last_kernel_s = ms * 1e-3;
  const auto t_dn0 = std::chrono::steady_clock::now();
  r.iterations = static_cast<int32_t>(scal[0]);
  r.status = static_cast<int32_t>(scal[1]);
  r.max_local_infeasibility = scal[2];
  r.objective = scal[3];
  r.near_ties = static_cast<int32_t>(scal[4]);
  r.first_near_tie = static_cast<int32_t>(scal[5]);
  r.time_solve = c->last_kernel_s;
  resident_timings(r, ph, c->last_kernel_s);
  if (r.trace && r.iterations > 0) {
    ck(cudaMemcpyAsync(r.trace, c->d_trace, static_cast<std::size_t>(r.iterations) * 6 * sizeof(double),
                       cudaMemcpyDeviceToHost, c->stream),
       "trace d2h");
    ck(cudaStreamSynchronize(c->stream), "trace d2h");
  }
  r.time_download = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_dn0).count();
  r.time_upload = std::chrono::duration<double>(t_dn0 - t_up0).count() - c->last_kernel_s;
  (void)s;
}

void run(dopf_cuda_ctx* c, const dopf_settings* s, dopf_result_view* results, int count,
         bool copy_vectors) {
  check_settings(s);
  if (!c->uploaded) throw std::invalid_argument("no model uploaded");
  HostLayout& L = c->L;
  const std::size_t I = L.inst.size();
  if (static_cast<std::size_t>(count) != I) throw std::invalid_argument("result count mismatch");
  bool want_trace = false;
  for (int i = 0; i < count; ++i) want_trace = want_trace || results[i].trace;
  const std::size_t need = want_trace ? I * static_cast<std::size_t>(s->max_iter) * 6 : 0;
  if (need > c->trace_cap) {
    if (c->d_trace) cudaFree(c->d_trace);
    c->d_trace = nullptr;
    ck(cudaMalloc(&c->d_trace, need * sizeof(double)), "trace alloc");
    c->trace_cap = need;
  }
  const auto t_up0 = std::chrono::steady_clock::now();
  ck(cudaMemsetAsync(c->d_flags, 0, I * L.blocks_per_instance * 16 * sizeof(unsigned long long),
                     c->stream),
     "memset");
  ck(cudaMemsetAsync(c->d_ctl, 0, I * kCtlWords * sizeof(unsigned long long), c->stream), "memset");
  ck(cudaMemsetAsync(c->d_maxinf, 0, I * sizeof(double), c->stream), "memset");
  ck(cudaMemsetAsync(c->d_part, 0, I * kSlotRing * L.blocks_per_instance * kPartials * sizeof(double), c->stream),
     "memset");
  // u^0 records {tag 0, z^0} in buffer 0 (tags of buffer 1 = 0 never match t = 1)
  ck(cudaMemsetAsync(c->d_u, 0, 4 * L.rows_total * sizeof(double), c->stream), "memset");
  ck(cudaMemcpy2DAsync(c->d_u + 1, 2 * sizeof(double), c->d_z0, sizeof(double), sizeof(double),
                       L.rows_total, cudaMemcpyDeviceToDevice, c->stream),
     "u0");

  KernelParams p{};
  p.blocks = c->d_blocks;
  p.inst = c->d_inst;
  p.P = c->d_P;
  p.A = c->d_A;
  p.copies = c->d_copies;
  p.rmeta = c->d_rmeta;
  p.v = c->d_v;
  p.z0 = c->d_z0;
  p.cmeta = c->d_cmeta;
  p.cc = c->d_cc;
  p.cinv = c->d_cinv;
  p.clo = c->d_clo;
  p.chi = c->d_chi;
  p.ameta = c->d_ameta;
  p.ab = c->d_ab;
  p.nbrs = c->d_nbrs;
  p.ux = reinterpret_cast<unsigned long long*>(c->d_u);
  p.z_out = c->d_z;
  p.lam_out = c->d_lam;
  p.x_out = c->d_x;
  p.part = c->d_part;
  p.flags = c->d_flags;
  p.ctl = c->d_ctl;
  p.trace = want_trace ? c->d_trace : nullptr;
  if (c->profiling && c->prof_cap < static_cast<std::size_t>(c->num_blocks) * 8) {
    if (c->d_prof) cudaFree(c->d_prof);
    c->d_prof = nullptr;
    c->prof_cap = static_cast<std::size_t>(c->num_blocks) * 8;
    ck(cudaMalloc(&c->d_prof, c->prof_cap * sizeof(long long)), "cudaMalloc");
    ck(cudaMemset(c->d_prof, 0, c->prof_cap * sizeof(long long)), "memset");
  }
  p.prof = c->profiling ? c->d_prof : nullptr;
  if (c->profiling) {
    const std::size_t need = static_cast<std::size_t>(c->num_blocks) * kTimelineIters * 3;
    c->d_timeline = c->scratch<unsigned long long>(127, need);
    ck(cudaMemsetAsync(c->d_timeline, 0, need * 8, c->stream), "memset");
    c->timeline_len = need;
  }
  p.timeline = c->profiling ? c->d_timeline : nullptr;
  p.iters = c->d_iters;
  p.status = c->d_status;
  p.maxinf = c->d_maxinf;
  p.objective = c->d_obj;
  p.ties = c->d_ties;
  p.phase_sample = c->d_phase;
  p.rho = s->rho;
  p.rho_inv = rho_reciprocal(s->rho);
  p.eps_rel = s->eps_rel;
  p.rows_total = L.rows_total;
  p.trace_stride = s->max_iter;
  p.max_iter = s->max_iter;
  p.blocks_per_instance = L.blocks_per_instance;
  p.sync_mode = static_cast<int32_t>(c->mode);
  p.snap = c->snap_dev;
  p.snap_stride = 2 * L.rows_total + L.x_total;
  p.snap_iters = c->snap_dev ? c->snap_iters : 0;

  // scenario batches: persistent CTA groups over the instances (every SM
  // busy) unless DOPF_BATCH_CLUSTERS=1 asks for one cluster per instance
  const bool groups = I > 1 && c->mode != SyncMode::grid && !std::getenv("DOPF_BATCH_CLUSTERS");
  p.group_size = groups ? L.blocks_per_instance : 0;
  p.instances = static_cast<int32_t>(I);
  ck(cudaEventRecord(c->ev0, c->stream), "event");
  if (groups) {
    const int G = L.blocks_per_instance;
    const int ng = std::max(1, std::min<int>(static_cast<int>(I), c->sm_count * ctas_per_sm() / G));
    ck(launch_admm_groups(p, ng, L.K, L.smem_bytes, L.all_ops_in_smem, c->stream), "launch");
  } else {
    ck(launch_admm(p, c->num_blocks, L.K, L.smem_bytes, c->mode, c->cluster, L.all_ops_in_smem, c->stream),
       "launch");
  }
  ck(cudaEventRecord(c->ev1, c->stream), "event");
  ++c->launches;
  ++c->kernels;
  if (count == 1 && I == 1 && c->dev_plan) {
    // one instance: everything comes back with the kernel still in the stream
    // order -- device permutation to reference order, direct copies into the
    // caller's arrays, one synchronisation (plus one for the trace)
    finish_single(c, s, results[0], copy_vectors, t_up0);
    return;
  }
  ck(cudaEventSynchronize(c->ev1), "kernel");
  ck(cudaGetLastError(), "kernel");
  float ms = 0;
  ck(cudaEventElapsedTime(&ms, c->ev0, c->ev1), "elapsed");
  c->last_kernel_s = ms * 1e-3;
  const auto t_dn0 = std::chrono::steady_clock::now();

  std::vector<int32_t> iters(I), status(I);
  std::vector<double> maxinf(I), obj(I);
  std::vector<int32_t> ties(2 * I);
  ck(cudaMemcpy(iters.data(), c->d_iters, I * sizeof(int32_t), cudaMemcpyDeviceToHost), "d2h");
  ck(cudaMemcpy(status.data(), c->d_status, I * sizeof(int32_t), cudaMemcpyDeviceToHost), "d2h");
  ck(cudaMemcpy(maxinf.data(), c->d_maxinf, I * sizeof(double), cudaMemcpyDeviceToHost), "d2h");
  ck(cudaMemcpy(obj.data(), c->d_obj, I * sizeof(double), cudaMemcpyDeviceToHost), "d2h");
  ck(cudaMemcpy(ties.data(), c->d_ties, 2 * I * sizeof(int32_t), cudaMemcpyDeviceToHost), "d2h");
  long long ph[8];
  ck(cudaMemcpy(ph, c->d_phase, sizeof ph, cudaMemcpyDeviceToHost), "d2h");
  bool any_vec = false;
  for (int i = 0; i < count; ++i)
    any_vec = any_vec || results[i].x || results[i].z || results[i].lambda;
  // results: a single instance needs only ring buffer iters % kZRing; a
  // batch gathers every instance's slot on the device first (instances stop
  // at different iterations), so one compact copy comes back
  const std::size_t R = static_cast<std::size_t>(L.rows_total);
  const bool one = I == 1;
  double *zdev = nullptr, *ldev = nullptr, *xall = nullptr;
  if (copy_vectors && any_vec) {
    double* st = static_cast<double*>(c->stage((2 * R + L.x_total) * sizeof(double)));
    zdev = st;
    ldev = st + R;
    xall = st + 2 * R;
    const double *zsrc = c->d_z + (one ? (iters[0] % kZRing) * R : 0);
    const double *lsrc = c->d_lam + (one ? (iters[0] % kZRing) * R : 0);
    if (!one) {
      std::vector<int32_t> row0(I), rows(I);
      for (std::size_t i = 0; i < I; ++i) {
        row0[i] = L.inst[i].row0;
        rows[i] = L.inst[i].rows;
      }
      int32_t* d_meta = c->scratch<int32_t>(120, 2 * I);
      double* d_out = c->scratch<double>(121, 2 * R);
      ck(cudaMemcpyAsync(d_meta, row0.data(), I * sizeof(int32_t), cudaMemcpyHostToDevice, c->stream), "h2d");
      ck(cudaMemcpyAsync(d_meta + I, rows.data(), I * sizeof(int32_t), cudaMemcpyHostToDevice, c->stream), "h2d");
      ck(launch_final_iterates(c->d_z, c->d_lam, L.rows_total, d_meta, d_meta + I, c->d_iters,
                               static_cast<int>(I), kZRing, d_out, d_out + R, c->stream),
         "final iterates");
      ++c->kernels;
      zsrc = d_out;
      lsrc = d_out + R;
    }
    ck(cudaMemcpyAsync(zdev, zsrc, R * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "d2h");
    ck(cudaMemcpyAsync(ldev, lsrc, R * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "d2h");
    ck(cudaMemcpyAsync(xall, c->d_x, L.x_total * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "d2h");
    ck(cudaStreamSynchronize(c->stream), "d2h");
  }
  for (int i = 0; i < count; ++i) {
    dopf_result_view& r = results[i];
    const InstDesc& id = L.inst[i];
    r.status = status[i];
    r.iterations = iters[i];
    r.objective = obj[i];
    r.max_local_infeasibility = maxinf[i];
    r.near_ties = ties[2 * i];
    r.first_near_tie = ties[2 * i + 1];
    r.time_solve = c->last_kernel_s;
    resident_timings(r, ph, c->last_kernel_s);  // instance 0's split (same kernel for all)
    if (copy_vectors && any_vec) {
      if (r.x) std::memcpy(r.x, xall + id.x_off, sizeof(double) * id.n);
      const std::size_t base = 0;
      for (int32_t d = id.row0; d < id.row0 + id.rows; ++d) {
        const int32_t ref = L.ref_of_dev[d];
        if (r.z) r.z[ref] = zdev[base + d];
        if (r.lambda) r.lambda[ref] = ldev[base + d];
      }
    }
    if (r.trace && iters[i] > 0)
      ck(cudaMemcpyAsync(r.trace, c->d_trace + static_cast<std::size_t>(i) * s->max_iter * 6,
                         static_cast<std::size_t>(iters[i]) * 6 * sizeof(double), cudaMemcpyDeviceToHost,
                         c->stream),
         "trace d2h");
  }
  ck(cudaStreamSynchronize(c->stream), "trace d2h");
  const double t_dn = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_dn0).count();
  for (int i = 0; i < count; ++i) {
    results[i].time_download = t_dn;
    results[i].time_upload = std::chrono::duration<double>(t_dn0 - t_up0).count() - c->last_kernel_s;
  }
}

}  // namespace

namespace {
int prepare_models(dopf_cuda_ctx* c, const dopf_model_view* ms, int count, double tol, bool reduce,
                   dopf_prepare_out* out, int32_t* fail_model, int32_t* fail_subsystem, double* seconds);
}  // namespace

extern "C" {

int dopf_cuda_create(int device, dopf_cuda_ctx** out) {
  if (!out) return DOPF_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  auto* c = new (std::nothrow) dopf_cuda_ctx();
  if (!c) return DOPF_ERR_OUT_OF_MEMORY;
  const int rc = guarded(c, [&] {
    int count = 0;
    ck(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
    if (device < 0 || device >= count) throw std::invalid_argument("no such CUDA device");
    struct Restore {  // the caller's current device is left as it was
      int prev = -1;
      ~Restore() {
        if (prev >= 0) cudaSetDevice(prev);
      }
    } restore;
    if (cudaGetDevice(&restore.prev) != cudaSuccess) restore.prev = -1;
    ck(cudaSetDevice(device), "cudaSetDevice");
    c->device = device;
    ck(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device), "attr");
    c->smem_optin = max_dynamic_smem(device);
    ck(cudaDeviceGetAttribute(&c->smem_per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device), "attr");
    ck(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking), "stream");
    c->stream = c->own_stream;
    ck(cudaEventCreate(&c->ev0), "event");
    ck(cudaEventCreate(&c->ev1), "event");
    ck(cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&c->join_ev, cudaEventDisableTiming), "event");
  });
  if (rc != DOPF_OK) {
    // keep the message reachable for the caller through a leaked-free path
    static thread_local std::string last;
    last = c->err;
    delete c;
    return rc;
  }
  *out = c;
  return DOPF_OK;
}

namespace {

bool needs_streaming(const dopf_model_view& m, const LayoutOptions& opt) {
  // resident kernel: <= 148 CTAs x 480 threads x kMaxK rows, operators in smem
  const int64_t cap_rows = static_cast<int64_t>(opt.max_blocks) * (opt.threads - 64) * kMaxK;
  if (m.N_z > cap_rows) return true;
  double bytes = 0;
  for (int s = 0; s < m.S; ++s) {
    const double n = m.z_offsets[s + 1] - m.z_offsets[s];
    bytes += 8.0 * (n * n + m.m_s[s] * n);
  }
  return bytes > 0.8 * static_cast<double>(opt.max_blocks) * static_cast<double>(opt.smem_limit);
}

// PhaseTimings of a streaming solve: the loop's device time split by the
// %globaltimer stamps of the kernels -- global = the boundary-column kernel
// (admm.cpp:118-129, interior columns run inside the chunk kernels), local =
// the chunk kernels, whose local update and dual update (admm.cpp:131-143)
// are one fused pass per row, so the dual share is reported inside local.
// (Partitioned: the exchange sits between them and counts in neither.)
void stream_timings(dopf_result_view& r, const StreamCtl& h, double total_s) {
  const double g = static_cast<double>(h.t_global), l = static_cast<double>(h.t_local);
  r.time_dual = 0.0;
  if (!(g + l > 0)) {
    r.time_global = r.time_local = 0.0;
    return;
  }
  r.time_global = total_s * g / (g + l);
  r.time_local = total_s * l / (g + l);
}

void upload_stream(dopf_cuda_ctx* c, const dopf_model_view& m, int nparts = 1, int part = 0,
                   const int32_t* part_of_s = nullptr) {
  c->SL = nparts > 1 ? build_stream_layout_part(m, nparts, part, part_of_s) : build_stream_layout(m);
  ++c->layout_epoch;  // captured graphs bake in the layout's kernel parameters
  const StreamLayout& L = c->SL;
  if (L.chunks.empty()) throw std::invalid_argument("streaming layout without rows");
  auto& d = c->sd;
  int k = 32;  // slots 32.. (the resident path uses 0..31)
  d.chunks = c->put(k++, L.chunks);
  d.blob = reinterpret_cast<unsigned char*>(c->put(k++, L.blob));
  d.z0 = c->put(k++, L.z0);
  d.col_ptr = c->put(k++, L.col_ptr);
  d.copies = c->put(k++, L.copies);
  d.cost = c->put(k++, L.c);
  d.inv = c->put(k++, L.inv);
  d.lo = c->put(k++, L.lo);
  d.hi = c->put(k++, L.hi);
  d.owner = c->put(k++, L.owner);
  d.x = c->scratch<double>(k++, L.cols);
  d.z = c->scratch<double>(k++, L.rows);
  d.lam = c->scratch<double>(k++, L.rows);
  d.u = c->scratch<double>(k++, L.rows);
  d.u_remote = c->scratch<double>(k++, std::max(1, L.remote_slots));
  // persistent staged CTAs per SM; the direct-load chunks get SMs of their own
  // (kBigCtasPerSm each) so they run beside the staged kernel
  c->staged_ctas = kDefaultStagedCtasPerSm;
  if (const char* e = std::getenv("DOPF_STAGED_CTAS")) c->staged_ctas = std::atoi(e) >= 3 ? 3 : 2;
  c->local_threads = kStreamRows;
  for (int32_t q : L.big_ids) {
    const StreamChunk& ch = L.chunks[q];
    if (std::max(ch.rows, std::max(ch.arows, ch.icols)) > kStreamRows) c->local_threads = kWideRows;
  }
  const int big_per_sm = c->local_threads > kStreamRows ? 1 : kBigCtasPerSm;
  const int big_sms = static_cast<int>((L.big_ids.size() + big_per_sm - 1) / big_per_sm);
  // (0 when every chunk takes the direct path: the partial slots and the fold
  // count then cover the direct-load CTAs only)
  c->staged_grid = L.staged_ids.empty()
                       ? 0
                       : std::max(1, std::min<int>(c->staged_ctas * std::max(1, c->sm_count - big_sms),
                                                   static_cast<int>(L.staged_ids.size())));
  d.part = c->scratch<double>(k++, std::max<std::size_t>(1, c->staged_grid + L.big_ids.size()) * 8);
  d.objp = c->scratch<double>(k++, std::max(1, (L.bcols + kStreamRows - 1) / kStreamRows));
  k++;  // (slot of the former separate partials buffer)
  d.ctl = c->scratch<StreamCtl>(k++, 1);
  k++;  // (slot of the former level-2 partials)
  d.final_count = c->scratch<unsigned>(k++, 1);
  d.export_rows = c->put(k++, L.export_rows);
  d.send = c->scratch<double>(k++, L.xstride());  // [exports | partials] record of this rank
  k++;  // (slot of the former separate partial gather)
  d.staged_ids = c->put(k++, L.staged_ids);
  d.big_ids = c->put(k++, L.big_ids);
  d.imp_ptr = c->put(k++, L.imp_ptr);
  d.imp_slot = c->put(k++, L.imp_slot);
  d.ximp = c->scratch<double>(k++, L.bimp.size());
  ck(stream_prepare(), "staged kernel attributes");
  if (const char* vb = std::getenv("DOPF_VERBOSE"); vb && vb[0] == '1')
    std::fprintf(stderr,
                 "stream layout: %zu chunks (%zu staged, %zu direct), %d rows, %d cols (%d boundary), %zu imports, "
                 "%.1f MB of chunk images\n",
                 L.chunks.size(), L.staged_ids.size(), L.big_ids.size(), L.rows, L.cols, L.bcols, L.bimp.size(),
                 8e-6 * static_cast<double>(L.blob.size()));
  ck(cudaStreamSynchronize(c->stream), "upload sync");
  c->drop_graph();
}

StreamParams stream_params(dopf_cuda_ctx* c, const dopf_settings* s, double* trace) {
  const StreamLayout& L = c->SL;
  auto& d = c->sd;
  StreamParams p{};
  p.chunks = d.chunks;
  p.blob = d.blob;
  p.staged_ids = d.staged_ids;
  p.big_ids = d.big_ids;
  p.imp_ptr = d.imp_ptr;
  p.imp_slot = d.imp_slot;
  p.ximp = d.ximp;
  p.n_staged = static_cast<int32_t>(L.staged_ids.size());
  p.n_big = static_cast<int32_t>(L.big_ids.size());
  p.staged_grid = c->staged_grid;
  p.npart = c->staged_grid + p.n_big;
  p.stages = L.stages;
  p.stage_bytes = L.stage_bytes;
  p.staged_ctas = c->staged_ctas;
  p.prof = nullptr;

  if (const char* e = std::getenv("DOPF_STREAM_PROF"); e && e[0] == '1') {
    p.prof = c->scratch<long long>(126, static_cast<std::size_t>(c->staged_grid) * 8);
    ck(cudaMemsetAsync(p.prof, 0, static_cast<std::size_t>(c->staged_grid) * 8 * sizeof(long long), c->stream),
       "prof");
  }
  p.col_ptr = d.col_ptr;
  p.copies = d.copies;
  p.cost = d.cost;
  p.inv = d.inv;
  p.lo = d.lo;
  p.hi = d.hi;
  p.owner = d.owner;
  p.x = d.x;
  p.z = d.z;
  p.lam = d.lam;
  p.u = d.u;
  p.u_remote = d.u_remote;
  p.part = d.part;
  p.objp = d.objp;
  p.final_count = d.final_count;
  p.trace = trace;
  p.ctl = d.ctl;
  p.partials_out = nullptr;
  p.export_rows = d.export_rows;
  p.send = d.send;
  p.n_export = static_cast<int32_t>(L.export_rows.size());
  p.max_export = L.max_export;
  p.rho = s->rho;
  p.rho_inv = rho_reciprocal(s->rho);
  p.eps = s->eps_rel;
  p.max_iter = s->max_iter;
  p.nchunks = static_cast<int32_t>(L.chunks.size());
  p.cols = L.cols;
  p.bcols = L.bcols;
  p.col_blocks = std::max(1, (L.bcols + kStreamRows - 1) / kStreamRows);
  p.local_threads = c->local_threads;
  return p;
}

// state of iteration 0: z = z^0, lambda = 0, u = z^0 - 0/rho = z^0, loop counters cleared
void stream_reset(dopf_cuda_ctx* c) {
  const StreamLayout& L = c->SL;
  auto& d = c->sd;
  ck(cudaMemcpyAsync(d.z, d.z0, L.rows * sizeof(double), cudaMemcpyDeviceToDevice, c->stream), "z0");
  ck(cudaMemcpyAsync(d.u, d.z0, L.rows * sizeof(double), cudaMemcpyDeviceToDevice, c->stream), "u0");
  ck(cudaMemsetAsync(d.lam, 0, L.rows * sizeof(double), c->stream), "lambda0");
  ck(cudaMemsetAsync(d.ctl, 0, sizeof(StreamCtl), c->stream), "ctl");
  ck(cudaMemsetAsync(d.final_count, 0, sizeof(unsigned), c->stream), "counter");
}

// The chunk kernels of one iteration on c->stream, the direct-load kernel on
// the auxiliary stream beside the staged one (a fork / join: under stream
// capture these become parallel graph branches), then the export pack.
void launch_chunks(dopf_cuda_ctx* c, const StreamParams& p) {
  if (p.n_big > 0 && p.n_staged > 0) {
    ck(cudaEventRecord(c->fork_ev, c->stream), "fork");
    ck(cudaStreamWaitEvent(c->aux, c->fork_ev, 0), "fork");
    stream_launch_direct(p, c->aux);
    ck(cudaEventRecord(c->join_ev, c->aux), "join");
    stream_launch_staged(p, c->stream);
    ck(cudaStreamWaitEvent(c->stream, c->join_ev, 0), "join");
  } else {
    stream_launch_direct(p, c->stream);
    stream_launch_staged(p, c->stream);
  }
  stream_launch_pack(p, c->stream);
}

void run_stream(dopf_cuda_ctx* c, const dopf_settings* s, dopf_result_view* r, bool copy_vectors) {
  check_settings(s);
  if (!c->uploaded) throw std::invalid_argument("no model uploaded");
  if (c->partitioned)
    throw std::invalid_argument("partitioned upload: solve through the dopf_cuda_part_* loop or dopf_cuda_solve_part");
  const StreamLayout& L = c->SL;
  auto& d = c->sd;
  const std::size_t need = r->trace ? static_cast<std::size_t>(s->max_iter) * 6 : 0;
  if (need > c->trace_cap) {
    if (c->d_trace) cudaFree(c->d_trace);
    c->d_trace = nullptr;
    ck(cudaMalloc(&c->d_trace, need * sizeof(double)), "trace alloc");
    c->trace_cap = need;
    c->drop_graph();
  }
  double* trace = r->trace ? c->d_trace : nullptr;
  if (!c->graph || c->graph_key[0] != s->rho || c->graph_key[1] != s->eps_rel ||
      c->graph_key[2] != s->max_iter || c->graph_trace != trace) {
    c->drop_graph();
    ck(stream_build_graph(stream_params(c, s, trace), &c->graph), "graph build");
    c->graph_key[0] = s->rho;
    c->graph_key[1] = s->eps_rel;
    c->graph_key[2] = s->max_iter;
    c->graph_trace = trace;
  }
  const auto t_up0 = std::chrono::steady_clock::now();
  stream_reset(c);
  // DOPF_STREAM_NOGRAPH=1: stream-ordered launches with a host stop check per
  // iteration (profilers that do not descend into conditional graph nodes)
  const char* nograph = std::getenv("DOPF_STREAM_NOGRAPH");
  ck(cudaEventRecord(c->ev0, c->stream), "event");
  if (nograph && nograph[0] == '1') {
    const StreamParams p = stream_params(c, s, trace);
    StreamCtl h{};
    do {
      stream_launch_iteration(p, c->stream);
      ck(cudaMemcpyAsync(&h, d.ctl, sizeof(StreamCtl), cudaMemcpyDeviceToHost, c->stream), "ctl");
      ck(cudaStreamSynchronize(c->stream), "iteration");
    } while (!h.done);
  } else {
    ck(cudaGraphLaunch(c->graph, c->stream), "graph launch");
  }
  ck(cudaEventRecord(c->ev1, c->stream), "event");
  ++c->launches;
  // results follow in stream order: loop state, then (single rank, value maps
  // on the device) z / lambda / x permuted to reference order on the device
  // and copied straight into the caller's arrays
  StreamCtl* ctl_h = static_cast<StreamCtl*>(c->small_stage());
  ck(cudaMemcpyAsync(ctl_h, d.ctl, sizeof(StreamCtl), cudaMemcpyDeviceToHost, c->stream), "d2h");
  const bool vectors = copy_vectors && (r->x || r->z || r->lambda);
  const bool direct = vectors && c->stream_maps && !c->partitioned && L.rows == L.N_z && L.cols == L.n;
  if (direct) {
    const std::size_t Nz = static_cast<std::size_t>(L.N_z), n = static_cast<std::size_t>(L.n);
    double* out = c->scratch<double>(123, 2 * Nz + n);
    ck(stream_launch_results(d.z, d.lam, d.x, c->d_refdev, c->d_gcol, L.rows, L.cols, out, out + Nz, out + 2 * Nz,
                             c->sm_count, c->stream),
       "results");
    if (r->z) ck(cudaMemcpyAsync(r->z, out, Nz * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "d2h");
    if (r->lambda)
      ck(cudaMemcpyAsync(r->lambda, out + Nz, Nz * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "d2h");
    if (r->x) ck(cudaMemcpyAsync(r->x, out + 2 * Nz, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "d2h");
  }
  ck(cudaStreamSynchronize(c->stream), "graph");
  ck(cudaGetLastError(), "graph");
  float ms = 0;
  ck(cudaEventElapsedTime(&ms, c->ev0, c->ev1), "elapsed");
  c->last_kernel_s = ms * 1e-3;
  const auto t_dn0 = std::chrono::steady_clock::now();
  const StreamCtl ctl = *ctl_h;
  // per iteration: k_global and the staged and/or direct chunk kernels
  const long long per_it = 1 + (c->SL.staged_ids.empty() ? 0 : 1) + (c->SL.big_ids.empty() ? 0 : 1);
  const char* ng = std::getenv("DOPF_STREAM_NOGRAPH");
  const long long unroll = (ng && ng[0] == '1') ? 1 : stream_graph_unroll();  // whole bodies run
  c->kernels += per_it * ((ctl.t + unroll - 1) / unroll) * unroll + (direct ? 1 : 0);
  if (const char* e = std::getenv("DOPF_STREAM_PROF"); e && e[0] == '1' && ctl.t > 0) {
    std::vector<long long> h(static_cast<std::size_t>(c->staged_grid) * 8);
    ck(cudaMemcpy(h.data(), c->bufs.at(126).p, h.size() * sizeof(long long), cudaMemcpyDeviceToHost), "prof");
    double sum[6] = {0, 0, 0, 0, 0, 0};
    for (int b = 0; b < c->staged_grid; ++b)
      for (int q = 0; q < 6; ++q) sum[q] += static_cast<double>(h[b * 8 + q]);
    const double per = static_cast<double>(c->SL.staged_ids.size());  // the last iteration's chunks
    std::fprintf(stderr, "staged phases (cycles per chunk): wait %.0f rows %.0f icol %.0f tgt %.0f gemv %.0f A %.0f\n",
                 sum[0] / per, sum[1] / per, sum[2] / per, sum[3] / per, sum[4] / per, sum[5] / per);
    std::vector<double> tot(c->staged_grid, 0.0);  // per-CTA busy cycles of the last iteration
    for (int b = 0; b < c->staged_grid; ++b)
      for (int q = 0; q < 6; ++q) tot[b] += static_cast<double>(h[b * 8 + q]);
    std::sort(tot.begin(), tot.end());
    if (!tot.empty())
      std::fprintf(stderr, "staged CTA cycles (last iteration): min %.0f median %.0f max %.0f\n", tot.front(),
                   tot[tot.size() / 2], tot.back());
  }
  r->status = ctl.status;
  r->iterations = ctl.t;
  r->objective = ctl.objective;
  r->max_local_infeasibility = ctl.maxinf;
  r->near_ties = ctl.ties;
  r->first_near_tie = ctl.first_tie;
  r->time_solve = c->last_kernel_s;
  stream_timings(*r, ctl, c->last_kernel_s);
  if (vectors && !direct) {
    const std::size_t R = static_cast<std::size_t>(L.rows);
    double* st = static_cast<double*>(c->stage((2 * R + L.cols) * sizeof(double)));
    ck(cudaMemcpyAsync(st, d.z, R * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "d2h");
    ck(cudaMemcpyAsync(st + R, d.lam, R * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "d2h");
    ck(cudaMemcpyAsync(st + 2 * R, d.x, L.cols * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "d2h");
    ck(cudaStreamSynchronize(c->stream), "d2h");
    if (r->x)
      for (int32_t q = 0; q < L.cols; ++q) r->x[L.gcol[q]] = st[2 * R + q];
    for (std::size_t dd = 0; dd < R; ++dd) {
      const int32_t ref = L.ref_of_dev[dd];
      if (r->z) r->z[ref] = st[dd];
      if (r->lambda) r->lambda[ref] = st[R + dd];
    }
  }
  if (r->trace && ctl.t > 0) {
    ck(cudaMemcpyAsync(r->trace, c->d_trace, static_cast<std::size_t>(ctl.t) * 6 * sizeof(double),
                       cudaMemcpyDeviceToHost, c->stream),
       "trace d2h");
    ck(cudaStreamSynchronize(c->stream), "trace d2h");
  }
  r->time_download = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_dn0).count();
  r->time_upload = std::chrono::duration<double>(t_dn0 - t_up0).count() - c->last_kernel_s;
}

// index maps of the plan (instance 0 layout) -> device, once per plan
void upload_plan_maps(dopf_cuda_ctx* c, const dopf_model_view& m) {
  const InstancePlan& P = *c->plan;
  int k = 64;  // slots 64.. (resident 0..31, streaming 32..62)
  c->d_psrc = c->put(k++, P.p_src);
  c->d_asrc = c->put(k++, P.a_src);
  c->d_absrc = c->put(k++, P.ab_src);
  c->d_refdev = c->put(k++, P.ref_of_dev);
  std::vector<int32_t> gcol(P.cmeta.size());
  for (std::size_t q = 0; q < gcol.size(); ++q) gcol[q] = P.cmeta[q].gcol;
  c->d_gcol = c->put(k++, gcol);
  c->d_rawP = c->scratch<double>(k++, static_cast<std::size_t>(m.p_offsets[m.S]));
  c->d_rawA = c->scratch<double>(k++, static_cast<std::size_t>(m.a_offsets[m.S]));
  c->d_rawb = c->scratch<double>(k++, static_cast<std::size_t>(m.b_offsets[m.S]));
  c->d_rawv = c->scratch<double>(k++, m.N_z);
  c->d_rawz0 = c->scratch<double>(k++, m.N_z);
  c->d_rawc = c->scratch<double>(k++, m.n);
  c->d_rawinv = c->scratch<double>(k++, m.n);
  c->d_rawlo = c->scratch<double>(k++, m.n);
  c->d_rawhi = c->scratch<double>(k++, m.n);
  ck(cudaStreamSynchronize(c->stream), "plan maps");
  c->dev_plan = c->plan.get();
}

void upload_values(dopf_cuda_ctx* c, const dopf_model_view& m) {
  auto h2d = [&](double* d, const double* h, std::size_t n) {
    if (n) ck(cudaMemcpyAsync(d, h, n * sizeof(double), cudaMemcpyHostToDevice, c->stream), "upload");
  };
  h2d(c->d_rawP, m.P, static_cast<std::size_t>(m.p_offsets[m.S]));
  h2d(c->d_rawA, m.A, static_cast<std::size_t>(m.a_offsets[m.S]));
  h2d(c->d_rawb, m.b, static_cast<std::size_t>(m.b_offsets[m.S]));
  h2d(c->d_rawv, m.v, m.N_z);
  h2d(c->d_rawz0, m.z0, m.N_z);
  h2d(c->d_rawc, m.c, m.n);
  h2d(c->d_rawinv, m.inv_copy, m.n);
  h2d(c->d_rawlo, m.x_lo, m.n);
  h2d(c->d_rawhi, m.x_hi, m.n);
  const InstancePlan& P = *c->plan;
  GatherParams g{};
  g.np = static_cast<int64_t>(P.p_src.size());
  g.na = static_cast<int64_t>(P.a_src.size());
  g.rows = static_cast<int64_t>(P.ref_of_dev.size());
  g.cols = static_cast<int64_t>(P.cmeta.size());
  g.nab = static_cast<int64_t>(P.ab_src.size());
  g.p_src = c->d_psrc;
  g.a_src = c->d_asrc;
  g.ref_of_dev = c->d_refdev;
  g.gcol = c->d_gcol;
  g.ab_src = c->d_absrc;
  g.rawP = c->d_rawP;
  g.rawA = c->d_rawA;
  g.rawb = c->d_rawb;
  g.rawv = c->d_rawv;
  g.rawz0 = c->d_rawz0;
  g.rawc = c->d_rawc;
  g.rawinv = c->d_rawinv;
  g.rawlo = c->d_rawlo;
  g.rawhi = c->d_rawhi;
  g.P = c->d_P;
  g.A = c->d_A;
  g.ab = c->d_ab;
  g.v = c->d_v;
  g.z0 = c->d_z0;
  g.cc = c->d_cc;
  g.cinv = c->d_cinv;
  g.clo = c->d_clo;
  g.chi = c->d_chi;
  ck(launch_gather(g, c->sm_count, c->stream), "gather");
  ++c->kernels;
  ck(cudaStreamSynchronize(c->stream), "upload sync");
}

void upload_stream_maps(dopf_cuda_ctx* c, const dopf_model_view& m) {
  const StreamLayout& L = c->SL;
  (void)m;
  int k = 96;  // slots 96.. (resident 0..31, streaming 32..70, resident maps 64..78 unused here)
  c->d_blobsrc = c->put(k++, L.blob_src);
  c->d_refdev = c->put(k++, L.ref_of_dev);
  c->d_gcol = c->put(k++, L.gcol);
  c->d_raw = c->scratch<double>(k++, static_cast<std::size_t>(L.raw_off[kRawEnd]));
  ck(cudaStreamSynchronize(c->stream), "stream maps");
  c->stream_maps = true;
}

void upload_stream_values(dopf_cuda_ctx* c, const dopf_model_view& m) {
  const StreamLayout& L = c->SL;
  const double* sec[kRawEnd] = {m.P, m.A, m.b, m.v, m.z0, m.c, m.inv_copy, m.x_lo, m.x_hi};
  for (int i = 0; i < kRawEnd; ++i) {
    const std::size_t n = static_cast<std::size_t>(L.raw_off[i + 1] - L.raw_off[i]);
    if (n)
      ck(cudaMemcpyAsync(c->d_raw + L.raw_off[i], sec[i], n * sizeof(double), cudaMemcpyHostToDevice, c->stream),
         "upload");
  }
  auto& d = c->sd;
  StreamRegather g{};
  g.raw = c->d_raw;
  g.blob_src = c->d_blobsrc;
  g.blob = reinterpret_cast<double*>(d.blob);
  g.nblob = static_cast<int64_t>(L.blob.size());
  g.ref_of_dev = c->d_refdev;
  g.z0 = d.z0;
  g.rows = L.rows;
  g.gcol = c->d_gcol;
  g.cost = d.cost;
  g.inv = d.inv;
  g.lo = d.lo;
  g.hi = d.hi;
  g.bcols = L.bcols;
  g.off_z0 = L.raw_off[kRawZ0];
  g.off_c = L.raw_off[kRawC];
  g.off_inv = L.raw_off[kRawInv];
  g.off_lo = L.raw_off[kRawLo];
  g.off_hi = L.raw_off[kRawHi];
  ck(stream_launch_regather(g, c->sm_count, c->stream), "regather");
  ++c->kernels;
  ck(cudaStreamSynchronize(c->stream), "upload sync");
}

}  // namespace

int dopf_cuda_upload(dopf_cuda_ctx* c, const dopf_model_view* m) {
  if (!c || !m) return DOPF_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    c->uploaded = false;
    // shares tuned for another structure do not apply (the cheap plan
    // comparison first: the common re-upload of the same model skips the hash)
    if (!c->block_weights.empty() && c->weights_sig &&
        !(c->plan && c->plan->same_structure(*m, options_for(c))) && c->weights_sig != structure_sig(*m)) {
      c->block_weights.clear();
      c->weights_sig = 0;
    }
    const LayoutOptions opt = options_for(c);
    if (!m->has_pre) throw std::invalid_argument("model view lacks precomputed operators");
    c->streaming = c->path_request == 2 || (c->path_request == 0 && needs_streaming(*m, opt));
    c->inst_nz = {m->N_z};
    c->inst_n = {m->n};
    const bool was_partitioned = c->partitioned;
    c->partitioned = false;
    if (was_partitioned) c->stream_maps = false;
    auto stream_upload = [&] {
      c->streaming = true;
      c->dev_plan = nullptr;
      c->L.reset();
      if (c->stream_maps && !c->partitioned && c->SL.same_structure(*m)) {
        upload_stream_values(c, *m);  // raw values + device gather (structure unchanged)
      } else {
        c->stream_maps = false;
        upload_stream(c, *m);
        upload_stream_maps(c, *m);
      }
      c->L.bytes_per_iteration = c->SL.bytes_per_iteration;
      c->uploaded = true;
    };
    if (c->streaming) {
      stream_upload();
      return;
    }
    const bool same = c->plan && c->plan->same_structure(*m, opt);
    if (same && c->dev_plan == c->plan.get() && c->L.inst.size() == 1) {
      // fast path: structure and index maps already on the device; copy the
      // raw value arrays and scatter them on the GPU (no host repacking)
      upload_values(c, *m);
      c->uploaded = true;
      return;
    }
    // the resident plan, checked against every limit of the resident kernel
    // before any device state changes; the automatic path falls back to the
    // streaming path when the model exceeds one (a forced resident path
    // reports it as std::invalid_argument)
    std::shared_ptr<InstancePlan> plan = same ? c->plan : nullptr;
    try {
      if (!plan) plan = std::make_shared<InstancePlan>(plan_instance(*m, choose_blocks(*m, opt), opt));
      check_resident(c, *plan);
    } catch (const std::invalid_argument& e) {
      if (c->path_request != 0) throw;
      if (std::getenv("DOPF_VERBOSE")) std::fprintf(stderr, "dopf: resident path unavailable (%s): streaming\n", e.what());
      stream_upload();
      return;
    }
    c->stream_maps = false;  // the map pointers are about to hold the resident plan's
    c->plan = plan;
    c->L.reset();
    append_instance(c->L, *c->plan, *m);
    finish_upload(c);
    upload_plan_maps(c, *m);
  });
}

int dopf_cuda_upload_batch(dopf_cuda_ctx* c, const dopf_model_view* ms, int32_t count) {
  if (!c || !ms || count < 1) return DOPF_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    c->uploaded = false;
    c->dev_plan = nullptr;
    c->stream_maps = false;
    c->streaming = false;
    c->partitioned = false;
    LayoutOptions opt = options_for(c);
    opt.max_blocks = 8;  // one cluster per scenario
    if (!c->batch_plan || !c->batch_plan->same_structure(ms[0], opt))
      c->batch_plan = std::make_shared<InstancePlan>(plan_instance(ms[0], choose_blocks(ms[0], opt), opt));
    c->inst_nz.clear();
    c->inst_n.clear();
    for (int i = 0; i < count; ++i) {
      if (!c->batch_plan->same_structure(ms[i], opt))
        throw std::invalid_argument("batched scenarios must share the subsystem structure");
      c->inst_nz.push_back(ms[i].N_z);
      c->inst_n.push_back(ms[i].n);
    }
    build_batch(c->L, *c->batch_plan, ms, count);
    finish_upload(c);
  });
}

int dopf_cuda_solve(dopf_cuda_ctx* c, const dopf_settings* s, dopf_result_view* r) {
  if (!c || !r) return DOPF_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    if (c->streaming) run_stream(c, s, r, true);
    else run(c, s, r, 1, true);
  });
}

int dopf_cuda_solve_device(dopf_cuda_ctx* c, const dopf_settings* s, dopf_result_view* r) {
  if (!c || !r) return DOPF_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    if (c->streaming) run_stream(c, s, r, false);
    else run(c, s, r, 1, false);
  });
}

int dopf_cuda_solve_snapshots(dopf_cuda_ctx* c, const dopf_settings* s, dopf_result_view* r,
                              double* snaps, int32_t T) {
  if (!c || !r || !snaps || T < 1) return DOPF_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    if (c->streaming && !c->partitioned) {
      // streaming path: the iteration's kernels launched stream-ordered with a
      // snapshot copy after each (test facility), then the regular solve
      check_settings(s);
      const StreamLayout& L = c->SL;
      auto& d = c->sd;
      const int64_t R = L.rows, X = L.cols, stride = 2 * R + X;
      double* dev = c->scratch<double>(118, static_cast<std::size_t>(T) * stride);
      stream_reset(c);
      const StreamParams p = stream_params(c, s, nullptr);
      StreamCtl h{};
      int rec = 0;
      do {
        stream_launch_iteration(p, c->stream);
        ck(cudaMemcpyAsync(&h, d.ctl, sizeof(StreamCtl), cudaMemcpyDeviceToHost, c->stream), "ctl");
        ck(cudaStreamSynchronize(c->stream), "iteration");
        if (h.t >= 1 && h.t <= T && h.t > rec) {
          double* sn = dev + static_cast<int64_t>(h.t - 1) * stride;
          ck(cudaMemcpyAsync(sn, d.z, R * sizeof(double), cudaMemcpyDeviceToDevice, c->stream), "snap");
          ck(cudaMemcpyAsync(sn + R, d.lam, R * sizeof(double), cudaMemcpyDeviceToDevice, c->stream), "snap");
          ck(cudaMemcpyAsync(sn + 2 * R, d.x, X * sizeof(double), cudaMemcpyDeviceToDevice, c->stream), "snap");
          rec = h.t;
        }
      } while (!h.done);
      run_stream(c, s, r, true);
      if (r->iterations != h.t) throw std::runtime_error("parity-mode rerun diverged");
      std::vector<double> hs(static_cast<std::size_t>(rec) * stride), z0(R);
      ck(cudaMemcpy(hs.data(), dev, hs.size() * sizeof(double), cudaMemcpyDeviceToHost), "d2h");
      ck(cudaMemcpy(z0.data(), d.z0, R * sizeof(double), cudaMemcpyDeviceToHost), "d2h");
      const int64_t n = L.n, out = n + 3 * R;
      std::vector<double> prev(R);
      for (int64_t q = 0; q < R; ++q) prev[L.ref_of_dev[q]] = z0[q];
      for (int t = 0; t < rec; ++t) {
        const double* sn = hs.data() + static_cast<int64_t>(t) * stride;
        double* o = snaps + static_cast<int64_t>(t) * out;
        for (int64_t cl = 0; cl < X; ++cl) o[L.gcol[cl]] = sn[2 * R + cl];
        for (int64_t q = 0; q < R; ++q) {
          o[n + L.ref_of_dev[q]] = sn[q];
          o[n + 2 * R + L.ref_of_dev[q]] = sn[R + q];
        }
        std::copy(prev.begin(), prev.end(), o + n + R);
        std::copy(o + n, o + n + R, prev.begin());
      }
      return;
    }
    if (c->streaming || c->partitioned || !c->dev_plan || c->L.inst.size() != 1)
      throw std::invalid_argument("iterate snapshots need a single model (resident or streaming path)");
    const InstancePlan& P = *c->dev_plan;
    const int64_t R = c->L.rows_total, X = c->L.x_total;
    const int64_t stride = 2 * R + X;
    c->snap_dev = c->scratch<double>(118, static_cast<std::size_t>(T) * stride);
    c->snap_iters = T;
    struct Off {
      dopf_cuda_ctx* c;
      ~Off() { c->snap_dev = nullptr; }
    } off{c};
    run(c, s, r, 1, true);
    const int rec = std::min<int>(T, r->iterations);
    std::vector<double> dev(static_cast<std::size_t>(rec) * stride), z0(R);
    ck(cudaMemcpy(dev.data(), c->snap_dev, dev.size() * sizeof(double), cudaMemcpyDeviceToHost), "d2h");
    ck(cudaMemcpy(z0.data(), c->d_z0, R * sizeof(double), cudaMemcpyDeviceToHost), "d2h");
    // reference order: [x (n) | z (N_z) | z_prev (N_z) | lambda (N_z)] per iteration
    const int64_t n = X, out = n + 3 * R;
    std::vector<double> prev(R);
    for (int64_t d = 0; d < R; ++d) prev[P.ref_of_dev[d]] = z0[d];
    for (int t = 0; t < rec; ++t) {
      const double* sn = dev.data() + static_cast<int64_t>(t) * stride;
      double* o = snaps + static_cast<int64_t>(t) * out;
      std::copy(sn + 2 * R, sn + 2 * R + n, o);
      for (int64_t d = 0; d < R; ++d) {
        const int32_t ref = P.ref_of_dev[d];
        o[n + ref] = sn[d];
        o[n + 2 * R + ref] = sn[R + d];
      }
      std::copy(prev.begin(), prev.end(), o + n + R);
      std::copy(o + n, o + n + R, prev.begin());
    }
  });
}

int dopf_cuda_precompute(dopf_cuda_ctx* c, const dopf_model_view* m, double* P, double* v,
                         int32_t* first_singular) {
  if (!c || !m || !P || !v) return DOPF_ERR_INVALID_ARGUMENT;
  if (first_singular) *first_singular = -1;
  dopf_prepare_out out{nullptr, nullptr, nullptr, P, v};
  int32_t fm = -1, fs = -1;
  const int rc = prepare_models(c, m, 1, 0.0, false, &out, &fm, &fs, nullptr);
  if (rc == DOPF_ERR_SINGULAR && first_singular) *first_singular = fs;
  return rc;
}

int dopf_cuda_prepare(dopf_cuda_ctx* c, const dopf_model_view* models, int32_t count, double tol,
                      dopf_prepare_out* out, int32_t* fail_model, int32_t* fail_subsystem,
                      double* seconds) {
  if (!c || !models || count < 1 || !out || !out->A || !out->b || !out->m || !out->P || !out->v ||
      !(tol >= 0))
    return DOPF_ERR_INVALID_ARGUMENT;
  return prepare_models(c, models, count, tol, true, out, fail_model, fail_subsystem, seconds);
}

}  // extern "C"

namespace {

template <typename T>
T* dev_copy(dopf_cuda_ctx* c, std::vector<void*>& owned, const T* h, std::size_t n) {
  void* d = nullptr;
  ck(cudaMalloc(&d, std::max<std::size_t>(n * sizeof(T), 16)), "cudaMalloc");
  owned.push_back(d);
  if (h && n) ck(cudaMemcpyAsync(d, h, n * sizeof(T), cudaMemcpyHostToDevice, c->stream), "h2d");
  return static_cast<T*>(d);
}

struct Owned {
  std::vector<void*> p;
  ~Owned() {
    for (void* d : p) cudaFree(d);
  }
};

// Batched row reduction + operators over every subsystem of `count` models
// (precompute_kernels.cu): inputs packed into one pinned staging buffer and
// copied once, two launches, outputs copied once into the caller's
// concatenated arrays. Errors as the host: the first infeasible subsystem
// (model order, then subsystem order) after the whole reduction, else the
// first singular one.
int prepare_models(dopf_cuda_ctx* c, const dopf_model_view* ms, int count, double tol, bool reduce,
                   dopf_prepare_out* out, int32_t* fail_model, int32_t* fail_subsystem, double* seconds) {
  if (fail_model) *fail_model = -1;
  if (fail_subsystem) *fail_subsystem = -1;
  int32_t code_model = -1, code_sub = -1, code = 0;
  const int rc = guarded(c, [&] {
    using clock = std::chrono::steady_clock;
    const auto t0 = clock::now();
    std::vector<PrepSub> subs;
    std::vector<int32_t> sub_model, sub_index;
    int64_t na = 0, nb = 0, np = 0, nz = 0, red_words = 0, prj_words = 0, big_words = 0;
    const int64_t smem_cap = c->smem_optin / static_cast<int64_t>(sizeof(double)) - 16;
    for (int k = 0; k < count; ++k) {
      const dopf_model_view& m = ms[k];
      if (m.S < 0 || (m.S > 0 && (!m.z_offsets || !m.m_s || !m.a_offsets || !m.b_offsets)))
        throw std::invalid_argument("bad model view");
      for (int s = 0; s < m.S; ++s) {
        PrepSub d{};
        d.m = m.m_s[s];
        d.n = m.z_offsets[s + 1] - m.z_offsets[s];
        if (d.m < 0 || d.n < 0 || m.a_offsets[s + 1] - m.a_offsets[s] != static_cast<int64_t>(d.m) * d.n)
          throw std::invalid_argument("inconsistent subsystem sizes");
        d.a_off = na + m.a_offsets[s];
        d.b_off = nb + m.b_offsets[s];
        d.p_off = np;
        d.v_off = nz + m.z_offsets[s];
        np += static_cast<int64_t>(d.n) * d.n;
        const int64_t rw = reduce ? reduce_words(d.m, d.n) : 0, pw = project_words(d.m, d.n);
        red_words = std::max(red_words, rw);
        prj_words = std::max(prj_words, pw);
        subs.push_back(d);
        sub_model.push_back(k);
        sub_index.push_back(s);
      }
      na += m.S ? m.a_offsets[m.S] : 0;
      nb += m.S ? m.b_offsets[m.S] : 0;
      nz += m.N_z;
    }
    const int64_t S = static_cast<int64_t>(subs.size());
    if (S == 0) return;
    if (S > 0x7fffffff) throw std::invalid_argument("too many subsystems");
    // subsystems beyond shared memory: every subsystem on global scratch
    const bool global_work = std::max(red_words, prj_words) > smem_cap;
    std::vector<int64_t> woff;
    if (global_work) {
      woff.resize(S);
      for (int64_t q = 0; q < S; ++q) {
        woff[q] = big_words;
        big_words += std::max(reduce ? reduce_words(subs[q].m, subs[q].n) : 0,
                              project_words(subs[q].m, subs[q].n));
      }
    }
    // pinned staging: [A | b] in, [A | b | rank | status | P | v] out
    const std::size_t in_bytes = (na + nb) * sizeof(double);
    const std::size_t out_bytes = (na + nb + np + nz) * sizeof(double) + 2 * S * sizeof(int32_t);
    auto* st = static_cast<unsigned char*>(c->stage(std::max(in_bytes, out_bytes)));
    {
      double* hA = reinterpret_cast<double*>(st);
      double* hb = hA + na;
      for (int k = 0; k < count; ++k) {
        const dopf_model_view& m = ms[k];
        if (!m.S) continue;
        const int64_t a = m.a_offsets[m.S], b = m.b_offsets[m.S];
        if ((a && !m.A) || (b && !m.b)) throw std::invalid_argument("model view without A / b");
        std::memcpy(hA, m.A, a * sizeof(double));
        std::memcpy(hb, m.b, b * sizeof(double));
        hA += a;
        hb += b;
      }
    }
    Owned o;
    auto dalloc = [&](std::size_t bytes) {
      void* d = nullptr;
      ck(cudaMalloc(&d, std::max<std::size_t>(bytes, 16)), "cudaMalloc");
      o.p.push_back(d);
      return d;
    };
    PrepParams p{};
    p.count = S;
    p.tol = tol;
    p.reduce = reduce ? 1 : 0;
    auto* dsubs = static_cast<PrepSub*>(dalloc(S * sizeof(PrepSub)));
    p.subs = dsubs;
    p.A = static_cast<double*>(dalloc((na + nb) * sizeof(double)));
    p.b = p.A + na;
    p.rank = static_cast<int32_t*>(dalloc(2 * S * sizeof(int32_t)));
    p.status = p.rank + S;
    p.P = static_cast<double*>(dalloc((np + nz) * sizeof(double)));
    p.v = p.P + np;
    if (global_work) {
      p.scratch = static_cast<double*>(dalloc(big_words * sizeof(double)));
      auto* d = static_cast<int64_t*>(dalloc(S * sizeof(int64_t)));
      ck(cudaMemcpyAsync(d, woff.data(), S * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream), "h2d");
      p.scratch_off = d;
    }
    ck(cudaMemcpyAsync(dsubs, subs.data(), S * sizeof(PrepSub), cudaMemcpyHostToDevice, c->stream), "h2d");
    ck(cudaMemcpyAsync(p.A, st, in_bytes, cudaMemcpyHostToDevice, c->stream), "h2d");
    if (!reduce) {
      std::vector<int32_t> r(2 * S, 0);
      for (int64_t q = 0; q < S; ++q) r[q] = subs[q].m;
      ck(cudaMemcpyAsync(p.rank, r.data(), 2 * S * sizeof(int32_t), cudaMemcpyHostToDevice, c->stream), "h2d");
    }
    ck(cudaEventRecord(c->ev0, c->stream), "event");
    const auto t1 = clock::now();
    if (reduce) {
      ck(launch_row_reduce(p, global_work ? 0 : red_words, c->stream), "row_reduce launch");
      ++c->kernels;
      // the host reports infeasibility before computing any operator
      std::vector<int32_t> stat(S);
      ck(cudaMemcpyAsync(stat.data(), p.status, S * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream), "d2h");
      ck(cudaStreamSynchronize(c->stream), "row_reduce");
      for (int64_t q = 0; q < S; ++q)
        if (stat[q] == kPrepInfeasible) {
          code = DOPF_ERR_INFEASIBLE;
          code_model = sub_model[q];
          code_sub = sub_index[q];
          return;
        }
    }
    ck(launch_project(p, global_work ? 0 : prj_words, c->stream), "project launch");
    ++c->kernels;
    ck(cudaEventRecord(c->ev1, c->stream), "event");
    // one copy back: [A | b] (reduced in place), [P | v], [rank | status]
    double* hA = reinterpret_cast<double*>(st);
    double* hP = hA + na + nb;
    auto* hr = reinterpret_cast<int32_t*>(hP + np + nz);
    if (reduce) ck(cudaMemcpyAsync(hA, p.A, (na + nb) * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "d2h");
    ck(cudaMemcpyAsync(hP, p.P, (np + nz) * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "d2h");
    ck(cudaMemcpyAsync(hr, p.rank, 2 * S * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream), "d2h");
    ck(cudaStreamSynchronize(c->stream), "prepare");
    float kms = 0.f;
    cudaEventElapsedTime(&kms, c->ev0, c->ev1);
    const auto t2 = clock::now();
    for (int64_t q = 0; q < S; ++q)
      if (hr[S + q] == kPrepSingular) {
        code = DOPF_ERR_SINGULAR;
        code_model = sub_model[q];
        code_sub = sub_index[q];
        return;
      }
    if (reduce) {
      std::memcpy(out->A, hA, na * sizeof(double));
      std::memcpy(out->b, hA + na, nb * sizeof(double));
      std::memcpy(out->m, hr, S * sizeof(int32_t));
    }
    std::memcpy(out->P, hP, np * sizeof(double));
    std::memcpy(out->v, hP + np, nz * sizeof(double));
    if (seconds) {
      seconds[0] = std::chrono::duration<double>(t1 - t0).count();  // pack + upload issue
      seconds[1] = kms * 1e-3;                                       // both kernels (events)
      seconds[2] = std::chrono::duration<double>(clock::now() - t2).count() +
                   std::max(0.0, std::chrono::duration<double>(t2 - t1).count() - kms * 1e-3);
    }
  });
  if (rc != DOPF_OK) return rc;
  if (code) {
    if (fail_model) *fail_model = code_model;
    if (fail_subsystem) *fail_subsystem = code_sub;
    return fail(c, code, std::string(code == DOPF_ERR_INFEASIBLE ? "infeasible" : "numerically singular") +
                             " subsystem #" + std::to_string(code_sub) + " of model " +
                             std::to_string(code_model));
  }
  return DOPF_OK;
}

}  // namespace

extern "C" {

int dopf_cuda_certify(dopf_cuda_ctx* c, const dopf_lp_view* lp, const double* x, dopf_certificate* out) {
  if (!c || !lp || !x || !out) return DOPF_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    Owned o;
    CertifyParams p{};
    p.rows = lp->rows;
    p.cols = lp->cols;
    p.row_blocks = std::max(1, (lp->rows + 255) / 256);
    p.col_blocks = std::max(1, (lp->cols + 255) / 256);
    p.row_ptr = dev_copy(c, o.p, lp->row_ptr, static_cast<std::size_t>(lp->rows) + 1);
    p.col_idx = dev_copy(c, o.p, lp->col_idx, static_cast<std::size_t>(lp->nnz));
    p.values = dev_copy(c, o.p, lp->values, static_cast<std::size_t>(lp->nnz));
    p.b = dev_copy(c, o.p, lp->b, static_cast<std::size_t>(lp->rows));
    p.lo = dev_copy(c, o.p, lp->x_lo, static_cast<std::size_t>(lp->cols));
    p.hi = dev_copy(c, o.p, lp->x_hi, static_cast<std::size_t>(lp->cols));
    p.x = dev_copy(c, o.p, x, static_cast<std::size_t>(lp->cols));
    p.blk_v = dev_copy<double>(c, o.p, nullptr, p.row_blocks + p.col_blocks);
    p.blk_i = dev_copy<int32_t>(c, o.p, nullptr, p.row_blocks + p.col_blocks);
    p.out = dev_copy<double>(c, o.p, nullptr, 2);
    p.out_idx = dev_copy<int32_t>(c, o.p, nullptr, 2);
    ck(launch_certify(p, c->stream), "certify");
    c->kernels += 3;
    double v[2];
    int32_t idx[2];
    ck(cudaMemcpyAsync(v, p.out, sizeof v, cudaMemcpyDeviceToHost, c->stream), "d2h");
    ck(cudaMemcpyAsync(idx, p.out_idx, sizeof idx, cudaMemcpyDeviceToHost, c->stream), "d2h");
    ck(cudaStreamSynchronize(c->stream), "certify");
    out->max_equality_violation = v[0];
    out->max_bound_violation = v[1];
    out->worst_row = idx[0];
    out->worst_col = idx[1];
    double obj = 0.0;  // c'x in column order (the host check's sequence)
    for (int j = 0; j < lp->cols; ++j) obj += lp->c[j] * x[j];
    out->objective = obj;
  });
}

int dopf_cuda_reconstruct(dopf_cuda_ctx* c, const dopf_model_view* m, const double* x, const double* z,
                          double* out) {
  if (!c || !m || !x || !z || !out || !m->has_pre) return DOPF_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    Owned o;
    ReconstructParams p{};
    p.n = m->n;
    p.csr_ptr = dev_copy(c, o.p, m->csr_ptr, static_cast<std::size_t>(m->n) + 1);
    p.csr_copy = dev_copy(c, o.p, m->csr_copy, static_cast<std::size_t>(m->N_z));
    p.z = dev_copy(c, o.p, z, static_cast<std::size_t>(m->N_z));
    p.x = dev_copy(c, o.p, x, static_cast<std::size_t>(m->n));
    p.lo = dev_copy(c, o.p, m->x_lo, static_cast<std::size_t>(m->n));
    p.hi = dev_copy(c, o.p, m->x_hi, static_cast<std::size_t>(m->n));
    double* d_out = dev_copy<double>(c, o.p, nullptr, static_cast<std::size_t>(m->n));
    p.out = d_out;
    ck(launch_reconstruct(p, c->stream), "reconstruct");
    ++c->kernels;
    ck(cudaMemcpyAsync(out, d_out, m->n * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "d2h");
    ck(cudaStreamSynchronize(c->stream), "reconstruct");
  });
}

int dopf_cuda_set_stream(dopf_cuda_ctx* c, void* stream) {
  if (!c) return DOPF_ERR_INVALID_ARGUMENT;
  c->stream = stream ? static_cast<cudaStream_t>(stream) : c->own_stream;
  return DOPF_OK;
}

int dopf_cuda_upload_part(dopf_cuda_ctx* c, const dopf_model_view* m, int32_t nparts, int32_t part,
                          const int32_t* part_of_s) {
  if (!c || !m || nparts < 1 || part < 0 || part >= nparts || !part_of_s) return DOPF_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    if (!m->has_pre) throw std::invalid_argument("model view lacks precomputed operators");
    c->uploaded = false;
    c->dev_plan = nullptr;
    c->L.reset();
    const bool same = c->stream_maps && c->streaming && c->partitioned &&
                      c->SL.same_structure(*m, nparts, part, part_of_s);
    c->streaming = true;
    c->partitioned = true;
    if (same) {
      upload_stream_values(c, *m);  // structure and partition unchanged: values only
      c->L.bytes_per_iteration = c->SL.bytes_per_iteration;
      c->uploaded = true;
      return;
    }
    c->stream_maps = false;
    upload_stream(c, *m, nparts, part, part_of_s);
    upload_stream_maps(c, *m);
    c->L.bytes_per_iteration = c->SL.bytes_per_iteration;
    c->inst_nz = {m->N_z};
    c->inst_n = {m->n};
    c->uploaded = true;
  });
}

int dopf_cuda_part_info(const dopf_cuda_ctx* c, dopf_part_info* out) {
  if (!c || !out || !c->partitioned) return DOPF_ERR_INVALID_ARGUMENT;
  out->nparts = c->SL.nparts;
  out->part = c->SL.part;
  out->rows = c->SL.rows;
  out->cols = c->SL.cols;
  out->n_export = static_cast<int32_t>(c->SL.export_rows.size());
  out->max_export = c->SL.max_export;
  out->xstride = c->SL.xstride();
  out->send = c->sd.send;
  out->recv = c->sd.u_remote;
  out->bytes_per_iteration = c->SL.bytes_per_iteration;
  return DOPF_OK;
}

int dopf_cuda_part_begin(dopf_cuda_ctx* c, const dopf_settings* s, int32_t with_trace) {
  if (!c || !c->partitioned) return DOPF_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    check_settings(s);
    const std::size_t need = with_trace ? static_cast<std::size_t>(s->max_iter) * 6 : 0;
    if (need > c->trace_cap) {
      if (c->d_trace) cudaFree(c->d_trace);
      c->d_trace = nullptr;
      ck(cudaMalloc(&c->d_trace, need * sizeof(double)), "trace alloc");
      c->trace_cap = need;
    }
    c->part_trace = with_trace != 0;
    c->part_params = stream_params(c, s, with_trace ? c->d_trace : nullptr);
    c->part_params.partials_out = c->sd.send + c->SL.max_export;  // behind the exports
    stream_reset(c);
    // u^0 of the exported rows for the first global update: pack z^0
    ck(cudaEventRecord(c->ev0, c->stream), "event");
  });
}

int dopf_cuda_part_step(dopf_cuda_ctx* c, int32_t phase) {
  if (!c || !c->partitioned || phase < 0 || phase > 3) return DOPF_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    const StreamParams& p = c->part_params;
    if (phase == 0) {
      stream_launch_global(p, c->stream);
      c->kernels += 1;
    } else if (phase == 1) {
      launch_chunks(c, p);
      c->kernels += (p.n_staged > 0 ? 1 : 0) + (p.n_big > 0 ? 1 : 0) + (p.max_export > 0 ? 1 : 0);
    } else if (phase == 2) {
      stream_launch_decide(p, c->sd.u_remote, c->SL.nparts, c->SL.xstride(), c->stream);
      c->kernels += 1;
    } else {
      stream_launch_pack(p, c->stream);  // exports of the current u (u^0 before iteration 1)
      c->kernels += 1;
    }
    ck(cudaGetLastError(), "launch");
  });
}

int dopf_cuda_part_poll(dopf_cuda_ctx* c, int32_t* done, int32_t* iterations) {
  if (!c || !c->partitioned) return DOPF_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    StreamCtl h{};
    ck(cudaMemcpyAsync(&h, c->sd.ctl, sizeof(StreamCtl), cudaMemcpyDeviceToHost, c->stream), "ctl");
    ck(cudaStreamSynchronize(c->stream), "poll");
    if (done) *done = h.done;
    if (iterations) *iterations = h.t;
  });
}

}  // extern "C"

namespace {

// results of a partitioned solve (this rank's share): scalars, x at owned
// columns, z / lambda at this rank's rows, trace; ev0 was recorded before
// the loop
void part_results(dopf_cuda_ctx* c, dopf_result_view* r, uint8_t* x_mask, uint8_t* z_mask) {
  {
    ck(cudaEventRecord(c->ev1, c->stream), "event");
    ck(cudaEventSynchronize(c->ev1), "solve");
    float ms = 0;
    ck(cudaEventElapsedTime(&ms, c->ev0, c->ev1), "elapsed");
    c->last_kernel_s = ms * 1e-3;
    const StreamLayout& L = c->SL;
    StreamCtl h{};
    ck(cudaMemcpyAsync(&h, c->sd.ctl, sizeof(StreamCtl), cudaMemcpyDeviceToHost, c->stream), "d2h");
    ck(cudaStreamSynchronize(c->stream), "d2h");
    r->status = h.status;
    r->iterations = h.t;
    r->objective = h.objective;
    r->max_local_infeasibility = h.maxinf;
    r->near_ties = h.ties;
    r->first_near_tie = h.first_tie;
    r->time_solve = c->last_kernel_s;
    stream_timings(*r, h, c->last_kernel_s);
    const std::size_t R = static_cast<std::size_t>(L.rows);
    // through the context's page-locked staging buffer (DMA speed), then
    // scattered to reference order on the host
    double* z = static_cast<double*>(c->stage((2 * R + L.cols) * sizeof(double)));
    double* lam = z + R;
    double* x = z + 2 * R;
    ck(cudaMemcpyAsync(z, c->sd.z, R * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "d2h");
    ck(cudaMemcpyAsync(lam, c->sd.lam, R * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "d2h");
    ck(cudaMemcpyAsync(x, c->sd.x, L.cols * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "d2h");
    ck(cudaStreamSynchronize(c->stream), "d2h");
    for (int32_t q = 0; q < L.cols; ++q) {
      if (!L.owner[q]) continue;
      if (r->x) r->x[L.gcol[q]] = x[q];
      if (x_mask) x_mask[L.gcol[q]] = 1;
    }
    for (std::size_t d = 0; d < R; ++d) {
      const int32_t ref = L.ref_of_dev[d];
      if (r->z) r->z[ref] = z[d];
      if (r->lambda) r->lambda[ref] = lam[d];
      if (z_mask) z_mask[ref] = 1;
    }
    if (r->trace && c->part_trace && h.t > 0)
      ck(cudaMemcpy(r->trace, c->d_trace, static_cast<std::size_t>(h.t) * 6 * sizeof(double),
                    cudaMemcpyDeviceToHost),
         "trace d2h");
  }
}

}  // namespace

extern "C" {

int dopf_cuda_part_finish(dopf_cuda_ctx* c, dopf_result_view* r, uint8_t* x_mask, uint8_t* z_mask) {
  if (!c || !c->partitioned || !r) return DOPF_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    ++c->launches;
    part_results(c, r, x_mask, z_mask);
  });
}

namespace {
// the value arrays of a model view and their lengths (doubles)
std::vector<std::pair<const double*, int64_t>> value_ranges(const dopf_model_view& m) {
  return {{m.P, m.p_offsets[m.S]}, {m.A, m.a_offsets[m.S]}, {m.b, m.b_offsets[m.S]}, {m.v, m.N_z},
          {m.z0, m.N_z}, {m.c, m.n}, {m.inv_copy, m.n}, {m.x_lo, m.n}, {m.x_hi, m.n}};
}
}  // namespace

int dopf_cuda_pin_model(dopf_cuda_ctx* c, const dopf_model_view* m) {
  if (!c || !m || !m->has_pre) return DOPF_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    for (auto [ptr, n] : value_ranges(*m)) {
      if (!ptr || n <= 0 || std::find(c->pinned.begin(), c->pinned.end(), ptr) != c->pinned.end()) continue;
      const cudaError_t e = cudaHostRegister(const_cast<double*>(ptr), static_cast<std::size_t>(n) * sizeof(double),
                                             cudaHostRegisterDefault);
      if (e == cudaErrorHostMemoryAlreadyRegistered) {
        cudaGetLastError();
        continue;
      }
      ck(e, "cudaHostRegister");
      c->pinned.push_back(ptr);
    }
  });
}

int dopf_cuda_pin_host(dopf_cuda_ctx* c, const void* ptr, int64_t bytes) {
  if (!c || !ptr || bytes <= 0) return DOPF_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    if (std::find(c->pinned.begin(), c->pinned.end(), ptr) != c->pinned.end()) return;
    const cudaError_t e =
        cudaHostRegister(const_cast<void*>(ptr), static_cast<std::size_t>(bytes), cudaHostRegisterDefault);
    if (e == cudaErrorHostMemoryAlreadyRegistered) {
      cudaGetLastError();
      return;
    }
    ck(e, "cudaHostRegister");
    c->pinned.push_back(ptr);
  });
}

int dopf_cuda_unpin_host(dopf_cuda_ctx* c, const void* ptr) {
  if (!c || !ptr) return DOPF_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    auto it = std::find(c->pinned.begin(), c->pinned.end(), ptr);
    if (it == c->pinned.end()) return;
    ck(cudaHostUnregister(const_cast<void*>(ptr)), "cudaHostUnregister");
    c->pinned.erase(it);
  });
}

int dopf_cuda_unpin_model(dopf_cuda_ctx* c, const dopf_model_view* m) {
  if (!c || !m) return DOPF_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    for (auto [ptr, n] : value_ranges(*m)) {
      (void)n;
      auto it = std::find(c->pinned.begin(), c->pinned.end(), ptr);
      if (it == c->pinned.end()) continue;
      ck(cudaHostUnregister(const_cast<double*>(ptr)), "cudaHostUnregister");
      c->pinned.erase(it);
    }
  });
}

int dopf_cuda_stream_info(const dopf_cuda_ctx* c, int64_t* out) {
  if (!c || !out) return DOPF_ERR_INVALID_ARGUMENT;
  for (int i = 0; i < 7; ++i) out[i] = 0;
  if (!c->streaming) return DOPF_OK;
  const StreamLayout& L = c->SL;
  out[0] = static_cast<int64_t>(L.chunks.size());
  out[1] = static_cast<int64_t>(L.staged_ids.size());
  out[2] = static_cast<int64_t>(L.big_ids.size());
  out[3] = L.bcols;
  out[4] = c->staged_grid;
  out[5] = L.stage_bytes;
  out[6] = L.stages;
  return DOPF_OK;
}

int dopf_cuda_div_rho_check(dopf_cuda_ctx* c, const double* a, int64_t n, double rho, double* out) {
  if (!c || n < 0 || (n > 0 && (!a || !out))) return DOPF_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    // scratch slots of the context (freed with it), not raw allocations that
    // would leak when a step throws
    double* da = c->scratch<double>(124, static_cast<std::size_t>(std::max<int64_t>(n, 1)));
    double* dout = c->scratch<double>(125, static_cast<std::size_t>(std::max<int64_t>(n, 1)));
    ck(cudaMemcpyAsync(da, a, n * sizeof(double), cudaMemcpyHostToDevice, c->stream), "h2d");
    ck(launch_div_rho_check(da, n, rho, rho_reciprocal(rho), dout, c->stream), "div_rho");
    ck(cudaMemcpyAsync(out, dout, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "d2h");
    ck(cudaStreamSynchronize(c->stream), "div_rho");
  });
}

int dopf_cuda_timeline(const dopf_cuda_ctx* c, uint64_t* out, int64_t cap) {
  if (!c || !out || !c->d_timeline) return DOPF_ERR_INVALID_ARGUMENT;
  return guarded(const_cast<dopf_cuda_ctx*>(c), [&] {
    const std::size_t n = std::min<std::size_t>(static_cast<std::size_t>(cap), c->timeline_len);
    ck(cudaMemcpy(out, c->d_timeline, n * 8, cudaMemcpyDeviceToHost), "d2h");
  });
}

int dopf_cuda_set_path(dopf_cuda_ctx* c, int32_t path) {
  if (!c || path < 0 || path > 2) return DOPF_ERR_INVALID_ARGUMENT;
  c->path_request = path;
  return DOPF_OK;
}

int dopf_cuda_solve_batch(dopf_cuda_ctx* c, const dopf_settings* s, dopf_result_view* r,
                          int32_t count) {
  if (!c || !r) return DOPF_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    if (c->streaming) throw std::invalid_argument("no batch uploaded");
    run(c, s, r, count, true);
  });
}

const char* dopf_cuda_last_error(const dopf_cuda_ctx* c) { return c ? c->err.c_str() : ""; }

void dopf_cuda_destroy(dopf_cuda_ctx* c) {
  if (!c) return;
  int prev = -1;
  if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
  cudaSetDevice(c->device);
  for (const void* ptr : c->pinned) cudaHostUnregister(const_cast<void*>(ptr));
  c->free_model();
  if (c->h_stage) cudaFreeHost(c->h_stage);
  if (c->h_small) cudaFreeHost(c->h_small);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->fork_ev) cudaEventDestroy(c->fork_ev);
  if (c->join_ev) cudaEventDestroy(c->join_ev);
  if (c->aux) cudaStreamDestroy(c->aux);
  if (c->poll_ev[0]) cudaEventDestroy(c->poll_ev[0]);
  if (c->poll_ev[1]) cudaEventDestroy(c->poll_ev[1]);
  if (c->h_flags) cudaFreeHost(c->h_flags);
  if (c->comm) {
    try {
      nccl::api().CommDestroy(c->comm);
    } catch (...) {
    }
  }
  if (c->own_stream) cudaStreamDestroy(c->own_stream);
  if (prev >= 0 && prev != c->device) cudaSetDevice(prev);
  delete c;
}

int dopf_cuda_info(const dopf_cuda_ctx* c, dopf_cuda_info_t* out) {
  if (!c || !out) return DOPF_ERR_INVALID_ARGUMENT;
  if (c->streaming) {
    out->instances = 1;
    out->blocks = c->staged_grid;  // persistent CTAs of the staged kernel
    out->threads = kStagedThreads;
    out->smem_bytes = c->SL.stages * c->SL.stage_bytes;
    out->resident = 0;
    out->sync_mode = 3;  // streaming graph (while-node)
    return DOPF_OK;
  }
  out->instances = static_cast<int32_t>(c->L.inst.size());
  out->blocks = c->L.blocks_per_instance;
  out->threads = kThreads;
  out->smem_bytes = static_cast<int32_t>(c->L.smem_bytes);
  out->resident = c->L.all_ops_in_smem ? 1 : 0;
  out->sync_mode = static_cast<int32_t>(c->mode);
  return DOPF_OK;
}

int64_t dopf_cuda_kernel_launches(const dopf_cuda_ctx* c) { return c ? c->launches : 0; }

int64_t dopf_cuda_kernels_executed(const dopf_cuda_ctx* c) { return c ? c->kernels : 0; }

double dopf_cuda_bytes_per_iteration(const dopf_cuda_ctx* c) {
  return c ? c->L.bytes_per_iteration : 0.0;
}

double dopf_cuda_last_kernel_seconds(const dopf_cuda_ctx* c) { return c ? c->last_kernel_s : 0.0; }

int dopf_layout_probe(const dopf_model_view* m, int32_t max_blocks, int64_t smem_limit,
                      dopf_layout_stats* out) {
  if (!m || !out || max_blocks < 1 || smem_limit < 1024) return DOPF_ERR_INVALID_ARGUMENT;
  try {
    LayoutOptions opt;
    opt.smem_limit = static_cast<std::size_t>(smem_limit);
    opt.max_blocks = max_blocks;
    HostLayout L;
    add_instance(L, *m, choose_blocks(*m, opt), opt);
    out->blocks = L.blocks_per_instance;
    out->rows_per_thread = L.K;
    out->resident = L.all_ops_in_smem ? 1 : 0;
    out->max_neighbours = L.max_neighbours;
    out->smem_bytes = static_cast<int64_t>(L.smem_bytes);
    int64_t remote = 0, local = 0, exported = 0;
    for (int32_t c : L.copies) (c < 0 ? remote : local) += 1;
    for (const RowMeta& r : L.rmeta) exported += r.exported ? 1 : 0;
    out->remote_copies = remote;
    out->local_copies = local;
    out->exported_rows = exported;
    out->bytes_per_iteration = L.bytes_per_iteration;
    return DOPF_OK;
  } catch (const std::invalid_argument&) {
    return DOPF_ERR_INVALID_ARGUMENT;
  } catch (const std::exception&) {
    return DOPF_ERR_RUNTIME;
  }
}

int dopf_partition_subsystems(const dopf_model_view* m, int32_t nparts, int32_t* part_of_s) {
  if (!m || nparts < 1 || !part_of_s) return DOPF_ERR_INVALID_ARGUMENT;
  try {
    // contiguous pieces of the depth-first walk, balanced by operator cost:
    // for the tiled feeder every piece is a run of whole tiles (subtrees)
    const std::vector<int> order = locality_order(*m);
    double total = 0;
    std::vector<double> cost(m->S);
    for (int s = 0; s < m->S; ++s) {
      const double n = m->z_offsets[s + 1] - m->z_offsets[s];
      cost[s] = n * n + m->m_s[s] * n + 6.0 * n + 4.0;
      total += cost[s];
    }
    double acc = 0;
    for (int s : order) {
      const int p = std::min<int>(nparts - 1, static_cast<int>(acc * nparts / total));
      part_of_s[s] = p;
      acc += cost[s];
    }
    return DOPF_OK;
  } catch (const std::exception&) {
    return DOPF_ERR_RUNTIME;
  }
}

int dopf_stream_layout_check(const dopf_model_view* m, int64_t* out) {
  if (!m || !out) return DOPF_ERR_INVALID_ARGUMENT;
  try {
    const StreamLayout L = build_stream_layout(*m);
    auto fail_if = [](bool bad, const char* what) {
      if (bad) throw std::logic_error(what);
    };
    const unsigned char* blob = reinterpret_cast<const unsigned char*>(L.blob.data());
    std::vector<int> seen(L.rows, 0);
    int64_t max_stage = 0, icopies = 0, widest = 0;
    std::vector<char> staged(L.chunks.size(), 0);
    for (int32_t q : L.staged_ids) staged[q] = 1;
    for (std::size_t q = 0; q < L.chunks.size(); ++q) {
      const StreamChunk& ch = L.chunks[q];
      widest = std::max<int64_t>(widest, ch.rows);
      for (int r = 0; r < ch.rows; ++r) ++seen[ch.row0 + r];
      ChunkHead h;
      std::memcpy(&h, blob + ch.image_off, sizeof h);
      fail_if(h.rows != ch.rows || h.arows != ch.arows || h.icols != ch.icols || h.row0 != ch.row0 ||
                  h.icol0 != ch.icol0 || h.bimp0 != ch.bimp0 || h.nbimp != ch.nbimp ||
                  h.image_bytes != ch.image_bytes || ch.image_off % 16 || ch.image_bytes % 16,
              "chunk head");
      for (int i = 0; i < kImgSections; ++i) fail_if(h.off[i] % 16 || h.off[i] > h.image_bytes, "section offset");
      StagePlan sp;
      stage_plan(ch, sp);
      if (staged[q]) {
        fail_if(sp.total > static_cast<uint32_t>(L.stage_bytes) || ch.rows > kStagedRows, "stage overflow");
        max_stage = std::max<int64_t>(max_stage, sp.total);
      }
      const StreamRow* rows = reinterpret_cast<const StreamRow*>(blob + ch.image_off + h.off[kImgRows]);
      const uint32_t* cm = reinterpret_cast<const uint32_t*>(blob + ch.image_off + h.off[kImgCmeta]);
      const int16_t* cc = reinterpret_cast<const int16_t*>(blob + ch.image_off + h.off[kImgCopies]);
      std::vector<int> covered(ch.rows, 0);
      for (int e = 0; e < ch.icols; ++e) {
        fail_if(L.owner[ch.icol0 + e] != (cmeta_owner(cm[e]) ? 1 : 0), "owner flag");
        for (int k = 0; k < cmeta_count(cm[e]); ++k) {
          const int row = cc[cmeta_start(cm[e]) + k];
          fail_if(row < 0 || row >= ch.rows || rows[row].xloc != e, "interior copy");
          ++covered[row];
          ++icopies;
        }
      }
      for (int r = 0; r < ch.rows; ++r) {
        const StreamRow& rm = rows[r];
        fail_if((rm.xloc >= 0) == (rm.xin >= 0), "row column kind");
        if (rm.xloc >= 0) fail_if(covered[r] != 1, "row not covered by its interior column");
        if (rm.xin >= 0)
          fail_if(rm.xin >= ch.nbimp || L.bimp[ch.bimp0 + rm.xin] >= L.bcols, "import slot");
        fail_if(rm.base < 0 || rm.base + rm.n > ch.rows || rm.n < 1, "row subsystem range");
      }
    }
    for (int v : seen) fail_if(v != 1, "row coverage");
    const int64_t vals[12] = {static_cast<int64_t>(L.chunks.size()), static_cast<int64_t>(L.staged_ids.size()),
                              static_cast<int64_t>(L.big_ids.size()), L.bcols, static_cast<int64_t>(L.bimp.size()),
                              max_stage, L.stage_bytes, static_cast<int64_t>(8 * L.blob.size()), L.rows, L.cols,
                              icopies, widest};
    for (int i = 0; i < 12; ++i) out[i] = vals[i];
    return DOPF_OK;
  } catch (const std::logic_error&) {
    return DOPF_ERR_LOGIC;
  } catch (const std::invalid_argument&) {
    return DOPF_ERR_INVALID_ARGUMENT;
  } catch (const std::exception&) {
    return DOPF_ERR_RUNTIME;
  }
}

int dopf_layout_probe_part(const dopf_model_view* m, int32_t nparts, int32_t part,
                           const int32_t* part_of_s, dopf_part_info* out) {
  if (!m || !out || !part_of_s) return DOPF_ERR_INVALID_ARGUMENT;
  try {
    const StreamLayout L = build_stream_layout_part(*m, nparts, part, part_of_s);
    *out = dopf_part_info{};
    out->nparts = nparts;
    out->part = part;
    out->rows = L.rows;
    out->cols = L.cols;
    out->n_export = static_cast<int32_t>(L.export_rows.size());
    out->max_export = L.max_export;
    out->xstride = L.xstride();
    out->bytes_per_iteration = L.bytes_per_iteration;
    return DOPF_OK;
  } catch (const std::invalid_argument&) {
    return DOPF_ERR_INVALID_ARGUMENT;
  } catch (const std::exception&) {
    return DOPF_ERR_RUNTIME;
  }
}

int dopf_layout_probe_batch(const dopf_model_view* ms, int32_t count, int64_t smem_limit,
                            dopf_layout_stats* out) {
  if (!ms || count < 1 || !out) return DOPF_ERR_INVALID_ARGUMENT;
  try {
    LayoutOptions opt;
    opt.smem_limit = static_cast<std::size_t>(smem_limit);
    opt.max_blocks = 8;
    const InstancePlan plan = plan_instance(ms[0], choose_blocks(ms[0], opt), opt);
    for (int i = 0; i < count; ++i)
      if (!plan.same_structure(ms[i], opt)) return DOPF_ERR_INVALID_ARGUMENT;
    HostLayout L;
    build_batch(L, plan, ms, count);
    out->blocks = L.blocks_per_instance;
    out->rows_per_thread = L.K;
    out->resident = L.all_ops_in_smem ? 1 : 0;
    out->max_neighbours = L.max_neighbours;
    out->smem_bytes = static_cast<int64_t>(L.smem_bytes);
    out->remote_copies = out->local_copies = out->exported_rows = 0;
    for (int32_t c : L.copies) (c < 0 ? out->remote_copies : out->local_copies) += 1;
    out->bytes_per_iteration = L.bytes_per_iteration;
    return DOPF_OK;
  } catch (const std::exception&) {
    return DOPF_ERR_RUNTIME;
  }
}

}  // extern "C"

namespace {

// Feedback tuning of the resident split (shared by the single-instance and
// the batch entry points). `upload` re-plans with c->block_weights. Single
// grid-wide instance: a CTA's slack is its wait at the iteration's final
// barrier, and CTAs without slack give cost shares away. Cluster / group
// instances (G <= 8 CTAs, all tight): a CTA position's load is its compute
// time without the exchange, and loaded positions give shares away.
double tune_split(dopf_cuda_ctx* c, const std::function<int()>& upload, const dopf_settings* s, int rounds) {
  check_settings(s);
  const bool grid = c->mode == SyncMode::grid;
  const int I = static_cast<int>(c->L.inst.size());
  const int G = c->L.blocks_per_instance;
  const int nb = static_cast<int>(c->L.blocks.size());
  const int K0 = c->L.K;
  std::vector<double> w(G, 1.0), best_w, best_sig(G), best_ref(G);
  double best = 1e300, beta = 0.8;  // first step (measured: 0.3 / 0.5 / 0.8 all reach 5.06-5.17 us on IEEE-8500)
  if (const char* e = std::getenv("DOPF_TUNE_BETA")) beta = std::atof(e);  // experiments
  std::vector<long long> cyc(static_cast<std::size_t>(nb) * 8);
  std::vector<dopf_result_view> res(I);
  auto median = [](std::vector<double> x) {
    std::nth_element(x.begin(), x.begin() + x.size() / 2, x.end());
    return x[x.size() / 2];
  };
  for (int r = 0; r < rounds; ++r) {
    c->block_weights = w;
    bool ok = true;
    try {
      c->plan.reset();  // re-plan with these shares
      c->batch_plan.reset();
      if (upload() != DOPF_OK) throw std::invalid_argument(c->err);
      ok = !c->streaming && c->L.K == K0 && c->L.all_ops_in_smem && c->L.blocks_per_instance == G &&
           static_cast<int>(c->L.blocks.size()) == nb;
    } catch (const std::invalid_argument&) {
      ok = false;
    }
    double per = 1e300;
    if (ok) {
      for (int q = 0; q < 3; ++q) {  // best of three plain runs: kernel time per (instance-)iteration
        for (auto& v : res) v = dopf_result_view{};
        run(c, s, res.data(), I, false);
        long long its = 0;
        for (const auto& v : res) its += std::max(1, v.iterations);
        per = std::min(per, c->last_kernel_s / static_cast<double>(its));
      }
    }
    if (ok && per < best) {
      best = per;
      best_w = w;
      if (c->d_prof) ck(cudaMemset(c->d_prof, 0, c->prof_cap * sizeof(long long)), "memset");
      c->profiling = true;
      for (auto& v : res) v = dopf_result_view{};
      run(c, s, res.data(), I, false);
      c->profiling = false;
      ck(cudaMemcpy(cyc.data(), c->d_prof, cyc.size() * sizeof(long long), cudaMemcpyDeviceToHost), "d2h");
      std::vector<double> sig(G, 0.0), ref(G, 0.0);
      for (int blk = 0; blk < nb; ++blk) {
        const long long* ph = cyc.data() + static_cast<std::size_t>(blk) * 8;
        const double it = std::max(1, res[blk / G].iterations);
        if (grid) {
          sig[blk % G] += static_cast<double>(ph[4]) / it;                                // slack
          ref[blk % G] += static_cast<double>(ph[0] + ph[1] + ph[2] + ph[3] + ph[5]) / it;  // busy
        } else {
          sig[blk % G] += static_cast<double>(ph[0] + ph[1] + ph[2] + ph[3]) / it;  // load
          ref[blk % G] = sig[blk % G];
        }
      }
      best_sig = sig;
      best_ref = ref;
    } else {
      beta *= 0.5;  // rejected: a smaller step from the best split
    }
    if (best_w.empty()) break;
    const double ms = median(best_sig), mr = std::max(1e-9, median(best_ref));
    double sum = 0;
    for (int g = 0; g < G; ++g) {
      const double d = (best_sig[g] - ms) / mr;
      w[g] = best_w[g] * (1.0 + (grid ? beta : -beta) * d);
      w[g] = std::min(1.5, std::max(0.5, w[g]));
      sum += w[g];
    }
    for (double& x : w) x *= G / sum;
  }
  if (best_w.empty()) best_w.assign(G, 1.0);
  c->block_weights = best_w;
  c->plan.reset();
  c->batch_plan.reset();
  if (upload() != DOPF_OK) throw std::runtime_error(c->err);
  return best;
}

}  // namespace

extern "C" {

int dopf_cuda_block_weights(const dopf_cuda_ctx* c, double* out, int32_t cap) {
  if (!c || (cap > 0 && !out)) return -1;
  const int n = static_cast<int>(c->block_weights.size());
  for (int i = 0; i < std::min(n, cap); ++i) out[i] = c->block_weights[i];
  return n;
}

int dopf_cuda_tune_partition(dopf_cuda_ctx* c, const dopf_model_view* m, const dopf_settings* s,
                             int32_t rounds, double* seconds_per_iteration) {
  if (!c || !m || !s || rounds < 1) return DOPF_ERR_INVALID_ARGUMENT;
  if (seconds_per_iteration) *seconds_per_iteration = 0;
  int rc = dopf_cuda_upload(c, m);
  if (rc != DOPF_OK) return rc;
  if (c->streaming || c->L.inst.size() != 1 || c->L.blocks_per_instance < 2) return DOPF_OK;  // nothing to split
  return guarded(c, [&] {
    c->weights_sig = 0;  // tuning re-plans this very structure
    const double per = tune_split(c, [&] { return dopf_cuda_upload(c, m); }, s, rounds);
    c->weights_sig = structure_sig(*m);
    if (seconds_per_iteration) *seconds_per_iteration = per;
  });
}

int dopf_cuda_tune_partition_batch(dopf_cuda_ctx* c, const dopf_model_view* ms, int32_t count,
                                   const dopf_settings* s, int32_t rounds, double* seconds_per_iteration) {
  if (!c || !ms || count < 1 || !s || rounds < 1) return DOPF_ERR_INVALID_ARGUMENT;
  if (seconds_per_iteration) *seconds_per_iteration = 0;
  int rc = dopf_cuda_upload_batch(c, ms, count);
  if (rc != DOPF_OK) return rc;
  if (c->L.blocks_per_instance < 2) return DOPF_OK;
  return guarded(c, [&] {
    const double per = tune_split(c, [&] { return dopf_cuda_upload_batch(c, ms, count); }, s, rounds);
    c->weights_sig = 0;  // per-instance shares (size G): applied to batches of any structure with G CTAs
    if (seconds_per_iteration) *seconds_per_iteration = per;
  });
}

int dopf_cuda_set_profiling(dopf_cuda_ctx* c, int32_t on) {
  if (!c) return DOPF_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    if (c->d_prof) ck(cudaMemset(c->d_prof, 0, c->prof_cap * sizeof(long long)), "memset");
    c->profiling = on != 0;
  });
}

int dopf_cuda_block_stats(const dopf_cuda_ctx* c, int64_t* out, int32_t max_blocks) {
  if (!c || !out || max_blocks < 1) return DOPF_ERR_INVALID_ARGUMENT;
  const HostLayout& L = c->L;
  const int nb = std::min<int>(max_blocks, static_cast<int>(L.blocks.size()));
  const int cw = kComputeThreads;
  for (int g = 0; g < nb; ++g) {
    const BlockDesc& b = L.blocks[g];
    int64_t remote = 0, exported = 0, chain = 0, n2 = 0;
    for (int q = 0; q < b.copy_len; ++q) remote += L.copies[b.copy_off + q] < 0;
    for (int r = 0; r < b.rows; ++r) {
      const RowMeta& rm = L.rmeta[b.row0 + r];
      exported += rm.exported;
      n2 += rm.n;
    }
    for (int t = 0; t < cw; ++t) {  // a thread's rows t, t + cw, ...: its sequential GEMV chain
      int64_t sum = 0;
      for (int r = t; r < b.rows; r += cw) sum += L.rmeta[b.row0 + r].n;
      chain = std::max(chain, sum);
    }
    const int64_t v[12] = {b.rows, b.cols, b.cols_int, b.arows, b.p_len, b.a_len, b.copy_len,
                           b.nbr_cnt, remote, exported, chain, n2};
    for (int q = 0; q < 12; ++q) out[static_cast<int64_t>(g) * 12 + q] = v[q];
  }
  return DOPF_OK;
}

int dopf_cuda_phase_cycles(const dopf_cuda_ctx* c, int64_t* out, int32_t max_blocks) {
  if (!c || !out || max_blocks < 1) return DOPF_ERR_INVALID_ARGUMENT;
  const int nb = std::min<int>(max_blocks, c->num_blocks);
  for (int q = 0; q < 8 * max_blocks; ++q) out[q] = 0;
  if (!c->d_prof) return DOPF_OK;
  return guarded(const_cast<dopf_cuda_ctx*>(c), [&] {
    ck(cudaMemcpy(out, c->d_prof, static_cast<std::size_t>(nb) * 8 * sizeof(long long),
                  cudaMemcpyDeviceToHost),
       "d2h");
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Partitioned solve on the library's own NCCL communicator
// (dopf_cuda_comm_init / dopf_cuda_solve_part). One iteration is
//   k_global -> chunk kernels (their last CTA writes this rank's partials
//   behind the exports) -> k_pack -> ncclAllGather(record) -> k_decide
// and the whole loop is one CUDA graph: a conditional while-node whose body
// is that iteration (k_decide clears the condition at the stop), or -- when
// the collective cannot be captured into a conditional body -- a graph of
// kUnroll iterations relaunched with a lazy, double-buffered host poll
// (kernels after the stop return at once, so the GPU is never starved and
// the result is the same). Every rank takes the same form (agreed by an
// all-reduce), so the collectives always match.

namespace {

constexpr int kPartUnroll = 8;

void require_comm(const dopf_cuda_ctx* c) {
  if (!c->partitioned || !c->uploaded) throw std::invalid_argument("no partitioned model uploaded");
  if (!c->comm) throw std::invalid_argument("no communicator: call dopf_cuda_comm_init first");
  if (c->SL.nparts != c->comm_nranks || c->SL.part != c->comm_rank)
    throw std::invalid_argument("the uploaded partition (" + std::to_string(c->SL.part) + " of " +
                                std::to_string(c->SL.nparts) + ") does not match the communicator (rank " +
                                std::to_string(c->comm_rank) + " of " + std::to_string(c->comm_nranks) + ")");
}

void enqueue_allgather(dopf_cuda_ctx* c) {
  const auto& a = nccl::api();
  nccl::check(a.AllGather(c->sd.send, c->sd.u_remote, static_cast<std::size_t>(c->SL.xstride()), ncclDouble, c->comm,
                          c->stream),
              "ncclAllGather");
}

// one iteration on c->stream (eager or under capture)
void enqueue_part_iteration(dopf_cuda_ctx* c, const StreamParams& p) {
  stream_launch_global(p, c->stream);
  launch_chunks(c, p);  // chunk kernels side by side + k_pack: this rank's record
  enqueue_allgather(c);
  stream_launch_decide(p, c->sd.u_remote, c->SL.nparts, c->SL.xstride(), c->stream);
}

// conditional while-node graph; false (stream left out of capture) if the
// runtime or the collective refuses the capture
bool build_part_graph_cond(dopf_cuda_ctx* c, StreamParams p, cudaGraphExec_t* exec) {
  cudaGraph_t g = nullptr;
  if (cudaGraphCreate(&g, 0) != cudaSuccess) return false;
  cudaGraphConditionalHandle h;
  cudaGraphNodeParams cp = {};
  cudaGraphNode_t node;
  bool ok = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault) == cudaSuccess;
  if (ok) {
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    ok = cudaGraphAddNode(&node, g, nullptr, 0, &cp) == cudaSuccess;
  }
  if (ok) {
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    p.cond = h;
    p.use_cond = 1;
    ok = cudaStreamBeginCaptureToGraph(c->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed) ==
         cudaSuccess;
    if (ok) {
      bool enq = true;
      try {
        enqueue_part_iteration(c, p);
      } catch (const std::exception&) {
        enq = false;
      }
      cudaGraph_t out = nullptr;
      const cudaError_t e = cudaStreamEndCapture(c->stream, &out);
      ok = enq && e == cudaSuccess && cudaGetLastError() == cudaSuccess;
    }
  }
  if (ok) ok = cudaGraphInstantiate(exec, g, 0) == cudaSuccess;
  cudaGraphDestroy(g);
  cudaGetLastError();  // a refused capture leaves no sticky error behind
  return ok;
}

void build_part_graph_unrolled(dopf_cuda_ctx* c, StreamParams p, cudaGraphExec_t* exec) {
  p.use_cond = 0;
  ck(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed), "capture");
  try {
    for (int i = 0; i < kPartUnroll; ++i) enqueue_part_iteration(c, p);
  } catch (...) {
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(c->stream, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  cudaGraph_t g = nullptr;
  ck(cudaStreamEndCapture(c->stream, &g), "capture");
  const cudaError_t e = cudaGraphInstantiate(exec, g, 0);
  cudaGraphDestroy(g);
  ck(e, "graph instantiate");
}

// the form every rank can run: min over ranks of this rank's capability
int agree_mode(dopf_cuda_ctx* c, int mine) {
  int32_t* d = c->scratch<int32_t>(119, 2);
  ck(cudaMemcpyAsync(d, &mine, sizeof(int32_t), cudaMemcpyHostToDevice, c->stream), "h2d");
  nccl::check(nccl::api().AllReduce(d, d + 1, 1, ncclInt32, ncclMax, c->comm, c->stream), "ncclAllReduce");
  int32_t all = 0;
  ck(cudaMemcpyAsync(&all, d + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream), "d2h");
  ck(cudaStreamSynchronize(c->stream), "agree");
  return all;  // modes: 1 conditional, 2 unrolled -- the max is the common one
}

void prepare_part_graph(dopf_cuda_ctx* c, const StreamParams& p, const dopf_settings* s, const double* trace) {
  const double key[6] = {s->rho, s->eps_rel, static_cast<double>(s->max_iter),
                         static_cast<double>(reinterpret_cast<uintptr_t>(trace)),
                         static_cast<double>(c->layout_epoch), static_cast<double>(c->comm_nranks)};
  if (c->part_graph && std::equal(key, key + 6, c->part_key)) return;
  if (c->part_graph) cudaGraphExecDestroy(c->part_graph);
  c->part_graph = nullptr;
  int want = 1;  // DOPF_PART_GRAPH=unrolled forces the unrolled form
  if (const char* e = std::getenv("DOPF_PART_GRAPH"); e && std::string(e) == "unrolled") want = 2;
  cudaGraphExec_t exec = nullptr;
  int mine = 2;
  if (want == 1 && build_part_graph_cond(c, p, &exec)) mine = 1;
  const int mode = agree_mode(c, mine);
  if (mode != mine && exec) {
    cudaGraphExecDestroy(exec);
    exec = nullptr;
  }
  if (mode == 2) build_part_graph_unrolled(c, p, &exec);
  c->part_graph = exec;
  c->part_graph_mode = mode;
  std::copy(key, key + 6, c->part_key);
}

// our kernels per partitioned iteration: k_global, chunk kernels, k_pack, k_decide
int part_kernels_per_iteration(const dopf_cuda_ctx* c) {
  return 2 + (c->SL.staged_ids.empty() ? 0 : 1) + (c->SL.big_ids.empty() ? 0 : 1) + (c->SL.max_export > 0 ? 1 : 0);
}

void run_part_graph(dopf_cuda_ctx* c, int max_iter) {
  const int per_it = part_kernels_per_iteration(c);
  if (c->part_graph_mode == 1) {
    ck(cudaGraphLaunch(c->part_graph, c->stream), "graph launch");
    ++c->launches;
    return;  // kernels counted from the iteration count (dopf_cuda_solve_part)
  }
  if (!c->poll_ev[0]) {
    ck(cudaEventCreateWithFlags(&c->poll_ev[0], cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&c->poll_ev[1], cudaEventDisableTiming), "event");
  }
  if (!c->h_flags) ck(cudaMallocHost(&c->h_flags, 2 * sizeof(int32_t)), "cudaMallocHost");
  const int64_t need = (static_cast<int64_t>(max_iter) + kPartUnroll - 1) / kPartUnroll;  // launches covering max_iter
  int64_t issued = 0;
  auto issue = [&] {
    const int b = static_cast<int>(issued & 1);
    ck(cudaGraphLaunch(c->part_graph, c->stream), "graph launch");
    ck(cudaMemcpyAsync(&c->h_flags[b], &c->sd.ctl->done, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream),
       "poll");
    ck(cudaEventRecord(c->poll_ev[b], c->stream), "event");
    ++issued;
    ++c->launches;
    c->kernels += static_cast<int64_t>(per_it) * kPartUnroll;
  };
  issue();
  for (int64_t k = 0;; ++k) {
    if (issued < need) issue();  // one launch stays queued behind the one being checked
    ck(cudaEventSynchronize(c->poll_ev[k & 1]), "poll");
    if (c->h_flags[k & 1]) break;
    if (k + 1 >= need) throw std::logic_error("partitioned loop ended without a stop decision");
  }
}

}  // namespace

extern "C" {

int dopf_nccl_unique_id(void* out) {
  if (!out) return DOPF_ERR_INVALID_ARGUMENT;
  try {
    ncclUniqueId id;
    nccl::check(nccl::api().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof(id));
    return DOPF_OK;
  } catch (const std::exception&) {
    return DOPF_ERR_NCCL;
  }
}

int dopf_cuda_comm_init(dopf_cuda_ctx* c, int32_t nranks, int32_t rank, const void* unique_id) {
  if (!c || nranks < 1 || rank < 0 || rank >= nranks || !unique_id) return DOPF_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    if (c->comm) throw std::invalid_argument("communicator already initialised");
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    nccl::check(nccl::api().CommInitRank(&c->comm, nranks, id, rank), "ncclCommInitRank");
    c->comm_nranks = nranks;
    c->comm_rank = rank;
  });
}

int dopf_cuda_comm_init_all(dopf_cuda_ctx** ctxs, int32_t n) {
  if (!ctxs || n < 1) return DOPF_ERR_INVALID_ARGUMENT;
  for (int i = 0; i < n; ++i)
    if (!ctxs[i] || ctxs[i]->comm) return DOPF_ERR_INVALID_ARGUMENT;
  return guarded(ctxs[0], [&] {
    std::vector<int> devs(n);
    std::vector<ncclComm_t> comms(n);
    for (int i = 0; i < n; ++i) devs[i] = ctxs[i]->device;
    nccl::check(nccl::api().CommInitAll(comms.data(), n, devs.data()), "ncclCommInitAll");
    for (int i = 0; i < n; ++i) {
      ctxs[i]->comm = comms[i];
      ctxs[i]->comm_nranks = n;
      ctxs[i]->comm_rank = i;
    }
  });
}

int dopf_cuda_comm_destroy(dopf_cuda_ctx* c) {
  if (!c) return DOPF_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    if (!c->comm) return;
    if (c->part_graph) cudaGraphExecDestroy(c->part_graph);
    c->part_graph = nullptr;
    nccl::check(nccl::api().CommDestroy(c->comm), "ncclCommDestroy");
    c->comm = nullptr;
    c->comm_nranks = 0;
    c->comm_rank = -1;
  });
}

int dopf_cuda_solve_part(dopf_cuda_ctx* c, const dopf_settings* s, dopf_result_view* r, uint8_t* x_mask,
                         uint8_t* z_mask) {
  if (!c || !r) return DOPF_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    check_settings(s);
    require_comm(c);
    const std::size_t need = r->trace ? static_cast<std::size_t>(s->max_iter) * 6 : 0;
    if (need > c->trace_cap) {
      if (c->d_trace) cudaFree(c->d_trace);
      c->d_trace = nullptr;
      ck(cudaMalloc(&c->d_trace, need * sizeof(double)), "trace alloc");
      c->trace_cap = need;
    }
    double* trace = r->trace ? c->d_trace : nullptr;
    c->part_trace = r->trace != nullptr;
    StreamParams p = stream_params(c, s, trace);
    p.partials_out = c->sd.send + c->SL.max_export;  // the record: [exports | partials]
    prepare_part_graph(c, p, s, trace);
    // iteration 0: state reset, u^0 exports gathered
    stream_reset(c);
    stream_launch_pack(p, c->stream);
    enqueue_allgather(c);
    ck(cudaEventRecord(c->ev0, c->stream), "event");
    run_part_graph(c, s->max_iter);
    part_results(c, r, x_mask, z_mask);
    if (c->part_graph_mode == 1) c->kernels += part_kernels_per_iteration(c) * r->iterations;
  });
}

int dopf_cuda_part_graph_mode(const dopf_cuda_ctx* c) { return c ? c->part_graph_mode : 0; }

const char* dopf_nccl_describe(void) {
  static thread_local std::string s;
  s = nccl::describe();
  return s.c_str();
}

}  // extern "C"
