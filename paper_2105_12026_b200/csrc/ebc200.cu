// ebc200.cu -- host runtime + C-ABI (include/ebc200.h) of the B200 EBC hot path.
//
// One context per EbcFunction (ebc.py:46-106): the ground matrix lives on the
// device for the context's life in the padded row-major layout of DESIGN.md §3,
// next to the fp64 e0-distances, the fp64/fp32 cached minima and the scratch of
// the Greedy step.  All work runs on one stream; a Greedy run never synchronises
// with the host between steps.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <atomic>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/ebc200.h"
#include "kernels.cuh"
#include "screen_tc.cuh"
#include "multiset.cuh"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>

using namespace ebc;

namespace {

thread_local std::string g_err;

// NCCL is loaded on demand (dlopen) so the library itself depends only on the
// CUDA runtime; in a torch process this resolves to the NCCL torch loaded.
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

struct SharedComm {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  int64_t generation = 0;
};

SharedComm& shared_comm(int device) {
  static SharedComm comms[64];
  return comms[device & 63];
}

const NcclApi& nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
      api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
      api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
      api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
      api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
      api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
      api.ok = api.GetUniqueId && api.CommInitRank && api.AllGather && api.AllReduce && api.CommDestroy &&
               api.GetErrorString;
    }
  }
  return api;
}

// Small pinned host words for per-step read-backs, carved from one
// process-wide page-locked slab: cudaMallocHost costs milliseconds, far more
// than the rest of a context's creation (EbcFunction in the e2e path).
struct PinnedWords {
  std::mutex mu;
  int* slab = nullptr;
  std::vector<int> free_slots;
  static constexpr int SLOTS = 4096;
  int* take() {
    std::lock_guard<std::mutex> lock(mu);
    if (!slab) {
      if (cudaMallocHost((void**)&slab, SLOTS * sizeof(int) * 16) != cudaSuccess) {
        slab = nullptr;
        return nullptr;
      }
      for (int i = SLOTS - 1; i >= 0; --i) free_slots.push_back(i);
    }
    if (free_slots.empty()) return nullptr;
    const int i = free_slots.back();
    free_slots.pop_back();
    return slab + (size_t)i * 16;  // one 64-byte line per slot
  }
  bool give(int* p) {
    std::lock_guard<std::mutex> lock(mu);
    if (!slab || p < slab || p >= slab + (size_t)SLOTS * 16) return false;
    free_slots.push_back((int)((p - slab) / 16));
    return true;
  }
};
PinnedWords& pinned_words() {
  static PinnedWords pw;
  return pw;
}

// Upload of the caller's pageable rows (ebc_create): host threads copy each
// chunk into one of two process-wide pinned staging buffers while the previous
// chunk's DMA runs (the driver's pageable path stages through one thread).
// Returns false (nothing enqueued) when staging is unavailable.
bool staged_upload(cudaStream_t stream, void* dst, const void* src, size_t bytes) {
  constexpr size_t CH = 8u << 20;
  static std::mutex mu;
  static unsigned char* stage[2] = {nullptr, nullptr};
  std::lock_guard<std::mutex> lock(mu);
  if (!stage[0]) {  // page-locked once per process (portable across devices)
    if (cudaHostAlloc((void**)&stage[0], 2 * CH, cudaHostAllocPortable) != cudaSuccess) {
      stage[0] = nullptr;
      return false;
    }
    stage[1] = stage[0] + CH;
  }
  // events of the calling device (a process may upload to several devices)
  struct Ev {
    cudaEvent_t e = nullptr;
    ~Ev() {
      if (e) cudaEventDestroy(e);
    }
  } done[2];
  if (cudaEventCreateWithFlags(&done[0].e, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&done[1].e, cudaEventDisableTiming) != cudaSuccess)
    return false;
  const size_t nch = (bytes + CH - 1) / CH;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int T = (int)std::min<unsigned>(8, hw);
  std::atomic<int64_t> allowed{std::min<int64_t>(2, (int64_t)nch) - 1};  // highest chunk a worker may fill
  std::vector<std::atomic<int>> filled(nch);
  for (auto& f : filled) f.store(0);
  auto worker = [&](int t) {
    for (size_t i = 0; i < nch; ++i) {
      while (allowed.load(std::memory_order_acquire) < (int64_t)i) std::this_thread::yield();
      const size_t off = i * CH, len = std::min(CH, bytes - off);
      const size_t a = len * t / T, b = len * (t + 1) / T;
      std::memcpy(stage[i & 1] + a, static_cast<const unsigned char*>(src) + off + a, b - a);
      filled[i].fetch_add(1, std::memory_order_acq_rel);
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < T; ++t) pool.emplace_back(worker, t);
  bool ok = true;
  // thread 0 of the copy is this one, interleaved with the DMA issue
  for (size_t i = 0; i < nch; ++i) {
    const size_t off = i * CH, len = std::min(CH, bytes - off);
    const size_t b0 = len / T;
    std::memcpy(stage[i & 1], static_cast<const unsigned char*>(src) + off, b0);
    filled[i].fetch_add(1, std::memory_order_acq_rel);
    while (filled[i].load(std::memory_order_acquire) < T) std::this_thread::yield();
    ok = ok && cudaMemcpyAsync(static_cast<unsigned char*>(dst) + off, stage[i & 1], len, cudaMemcpyHostToDevice,
                               stream) == cudaSuccess;
    ok = ok && cudaEventRecord(done[i & 1].e, stream) == cudaSuccess;
    if (i + 2 < nch) {  // buffer (i & 1) is reused by chunk i + 2 once this DMA is done
      ok = ok && cudaEventSynchronize(done[i & 1].e) == cudaSuccess;
      allowed.store((int64_t)i + 2, std::memory_order_release);
    }
  }
  for (auto& th : pool) th.join();
  // the staging buffers are shared: the last DMAs finish before the next caller
  ok = ok && cudaEventSynchronize(done[(nch - 1) & 1].e) == cudaSuccess;
  if (nch > 1) ok = ok && cudaEventSynchronize(done[nch & 1].e) == cudaSuccess;
  if (!ok) cudaStreamSynchronize(stream);  // no DMA may still read the shared staging
  return ok;
}

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct ScopedEvent {
  cudaEvent_t e = nullptr;
  ~ScopedEvent() {
    if (e) cudaEventDestroy(e);
  }
};

}  // namespace

struct ebc_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  int64_t n = 0;
  int d = 0;
  int dtype = EBC_F32;
  int pitch = 0;      // elements per device row
  int64_t n_pad = 0;  // rows allocated (zero padded)
  int d4 = 0;
  int nchunks = 0;    // ceil(n / RCH)
  float gram_kc = 0.f;  // kc = gram_kc * |c|^2
  double baseline = 0.0;
  int64_t c0 = 0, c1 = 0;  // screened candidate range
  int64_t steps_done = 0;   // selections since the last reset

  // device state
  float* V32 = nullptr;   // fp32 / widened fp16 grounds
  double* V64 = nullptr;  // fp64 grounds
  double* e0d = nullptr;
  double* cm64 = nullptr;
  float4* pt = nullptr;
  float* nv32 = nullptr;
  long long* stats = nullptr;  // k_pick: window-size statistics of the last run
  // adaptive screen: [0] the rung this step's kernels run (-1: a lazy step
  // decided without a screen), [1] the run's current rung (L_FAST .. L_DIRECT)
  int* level = nullptr;
  PtCoef pk{};
  // screen mode: 0 direct, 1 FFMA Gram, 2 adaptive from FFMA Gram, 3 adaptive from the tensor screen
  int screen_mode = 2;
  bool fp32_ok = true;  // ebc_create's range guard: false -> no fp32 screen at all (screen_mode -1)
  int wcap = 256;
  int wcap_tc = 256;  // the anchored tensor rung's window cap (EBC200_WCAP_TC)
  // tensor-core Gram screen (tcgen05, kind::tf32, 3xTF32)
  void* Vhi = nullptr;
  void* Vlo = nullptr;
  int tc_kind = 1;  // tc::KIND_TF32 / KIND_BF16 (fp32 grounds) / KIND_F16 (fp16 grounds)
  // fast first rung (fp32 grounds, large d): one rounded FP16 product (tc::KIND_F16R)
  bool tc_fast = false;
  void* Vf = nullptr;  // fp16(oscale x) in the UMMA canonical layout
  float tc_kx_fast = 0.f, tc_oscale = 1.f, tc_sinv2 = 1.f, tc_keta = 0.f, tc_keta2 = 0.f;
  // seeds folded into the MMA for the one-product FP16 rung (rung 0 for fp32
  // grounds, rung 1 for fp16-stored grounds): DESIGN.md §4
  bool tc_mseed = false;
  bool tc_mb2 = false;  // folded-seed rung: two candidate blocks per CTA (EBC200_TC_MB2)
  float tc_kpscale = 1.f;
  int* tile_anchor0 = nullptr;  // all-zero block anchors (the origin) for rung 0 with folded seeds
  // all-positive (block, tile) pairs of rung 1 summed from tile aggregates (k_screen_agg)
  bool tc_agg = false;
  float* rhomax = nullptr;  // na x tc_ntl: max |v - mu_a| over the tile
  float* cmn = nullptr;     // tc_ntl: min cm over the tile (current step)
  float* vsum = nullptr;    // tc_ntl x pitch: sum of the tile's points
  float* vsn = nullptr;     // tc_ntl: |vsum|
  double* ipsum = nullptr;  // na x tc_ntl: sum of the tile's seeds (current step)
  float* rhomin = nullptr;  // tc_ntl: min over anchors of rhomax
  float radmin = 0.f;       // min candidate-block radius
  int* agg_any = nullptr;   // this step: some tile can be all-positive
  DevBuf part_a;            // nsplit x n_pad aggregate partials
  int wcap_fast = 256;
  float* pttc = nullptr;   // na x n_pad seeds ip_a(v) = (cm32 - |v - mu_a|^2)/2
  float* kpmax = nullptr;  // na x tc_ntl: per (anchor, point tile) max error quantum kp (reset state)
  int tc_na = 1;           // anchors (0 = the origin)
  int64_t tc_ntl = 0;      // point tiles of the tensor screen
  float* anchors = nullptr;         // na x pitch
  float* nva = nullptr;             // na x n_pad: |v - mu_a|^2
  int* tile_anchor = nullptr;       // per 128-row candidate block
  float* tc_vmax = nullptr;         // per point tile: max |v|
  unsigned long long* fps_keys = nullptr;
  float* ipa0 = nullptr;            // na x n_pad seeds at the reset state (work-matrix flag screen)
  // certified tile-pair pruning of the tensor screen
  bool tc_prune = true;
  float* tile_rad = nullptr;        // per 128-row candidate block: max |c - mu_anchor|
  float* crad = nullptr;            // per candidate: |c - mu_anchor| rounded up (refine pruning)
  float* rho = nullptr;             // na x tc_ntl: min |v - mu_a| over the point tile
  float* cmx = nullptr;             // tc_ntl: max cm over the point tile (refreshed every screen)
  float* cmx0 = nullptr;            // tc_ntl: the same at the reset state (cm = d(., e0))
  bool cmx_fresh = false;           // cmx refreshed by the current step's screen (enqueue-time flag)
  int kpad = 0;
  int tc_np = 0;  // points per tensor tile (0: tensor screen unavailable)
  float tc_kp = 0.f, tc_kc = 0.f, tc_kx = 0.f;  // anchored bound coefficients
  unsigned char* selected = nullptr;
  double* chunkpart = nullptr;  // nchunks
  unsigned int* counter = nullptr;
  unsigned int* counter2 = nullptr;  // k_gain_top's last-block ticket
  int64_t* topc = nullptr;           // candidate with the largest screen bound (ub-only screens)
  double* toppart = nullptr;         // 4 nchunks: its exact gain's partials (argmax scratch before)
  double* terms = nullptr;           // n: e0d - cm64 per point (split K4)
  // fused K4 (k_update_fused; false: split K4) and its counters
  // ([0] chunks done, [1..] per-chunk tickets)
  bool uf_on = false;
  int uf_rows = 256;  // EBC200_UPDATE_ROWS: 64, 128 or 256 rows per fused-update block (measured equal)
  unsigned int* uf_ctr = nullptr;
  double* cur = nullptr;
  int64_t* best = nullptr;
  long long* maxlb = nullptr;
  int* wcount = nullptr;
  int64_t* wlist = nullptr;  // n
  double* wgain = nullptr;   // n
  double* ub = nullptr;      // n
  // lazy Greedy (kernels.cuh k_lazy_topk / k_lazy_mark2): ubp[c - c0] bounds c's current gain
  // (+inf after a reset); bflag: this step's re-screened 128-candidate blocks
  double* ubp = nullptr;           // n
  unsigned char* bflag = nullptr;  // ceil(n / 128) + 2
  bool lazy_on = true;             // EBC200_LAZY=0: every step screens every candidate
  int lazy_cap = 256;              // EBC200_LAZY_CAP: stale candidates decided by the exact refine alone
  bool ubp_seeded = false;         // enqueue-time: a full step has run since the reset
  bool cmx_valid = false;          // enqueue-time: cmx computed since the reset (an upper bound of cm's tile maxima)
  int64_t* slist = nullptr;        // n: this step's stale candidates in index order (k_lazy_write)
  int* bcnt = nullptr;             // ceil(n / 256) + 1: per-block stale counts, then offsets
  int* scount = nullptr;
  void* lazy_part = nullptr;       // 2 num_sms x TK 64-bit keys: k_lazy_topk's block lists
  double* ub_next = nullptr;       // best stale bound outside the first batch
  int lazy_batch = 4;              // EBC200_LAZY_BATCH (1..RW): candidates refined first in a lazy step (3 for N >= 2^18)
  bool probe_on = true;            // EBC200_LAZY_PROBE=0: no ring-probe batch on undecided steps
  bool fuse_batch = true;          // EBC200_FUSE_BATCH=0: the next step's first batch not folded into K4
  int64_t probe_min_n = 32768;     // EBC200_PROBE_MIN_N: candidates below which undecided steps skip probe / near bound
  int batch_ready_step = -1;       // enqueue-time: that step's first batch was launched with the last update
  cudaGraphConditionalHandle batch_hrest = 0;
  std::vector<char> fused_step;    // timing: step s's update was k_update_batch (ev[4 s + 2] after its top-k)
  int topk_cpb = 1024;              // EBC200_TOPK_CPB: candidates per k_lazy_topk block (grid <= 2 per SM)
  bool pdl = true;                  // EBC200_PDL: k_update_batch as a programmatic dependent of k_lazy_topk
  int ub_rows = 128;               // EBC200_UB_ROWS: rows per k_update_batch slice (64 or 128; two threads per row)
  ProbeBuf probe;                  // k_lazy_rings: ring winners, ticket, the probe list
  bool nb_on = false;              // EBC200_LAZY_NEARBOUND=0: no near-centre bound (k_lazy_nearbound)
  ChunkGeo geo;                    // per-chunk mean / radius / e0 sums for the near-centre bound
  unsigned int* counter3 = nullptr;  // k_refine's finalize ticket
  bool refine2 = true;             // EBC200_REFINE2=0: the lazy batch on the classic k_refine
  DevBuf rterms;                   // RW x nchunks chunk sums of the short refine
  DevBuf sxt;                      // short refine: RW x n_pad point terms, then nchunks tickets
  DevBuf ubpack;                   // k_batch_pack: the rows k_update_batch stages (BatchPackLayout)
  // CUDA-graph conditional nodes for the undecided part of a lazy step (captured
  // runs only: an eager run gates those kernels on level[0] instead)
  bool use_cond = true;            // EBC200_GRAPH_COND=0: plain gated kernels in graphs too
  cudaStream_t side[2] = {nullptr, nullptr};  // capture streams of conditional bodies
  bool screen_events_outside = false;  // the step's family events are recorded by the caller
  bool in_sharded_run = false;     // enqueue-time: inside enqueue_greedy_sharded (lazy steps use the global bound)
  bool force_global_lb = false;    // EBC200_GLOBAL_LB=1: the all-reduce path even on one rank (tests)
  // gathered lazy re-screens (kernels.cuh k_lazy_plan2): the stale set packed
  // into fresh 128-candidate blocks when the flagged blocks are sparse
  bool gather_on = false;          // EBC200_GATHER=0: always re-screen the flagged blocks
  int64_t gath_cap = 0;            // candidates a gathered re-screen holds
  float* Vg = nullptr;             // gath_cap x pitch
  int* g_anchor = nullptr;         // per gathered block
  float* g_rad = nullptr;
  // eager (uncaptured) lazy steps read the step's mode back (one 4-byte copy
  // into pinned memory) and enqueue only the kernels that will do work
  bool eager_sync = true;          // EBC200_EAGER_SYNC=0: enqueue everything, gated on the device
  int* mode_host = nullptr;        // pinned
  // threshold sieves (ebc_sieve_*): cached minima per slot
  DevBuf sv_cm, sv_de, sv_slots, sv_part, sv_out;
  int sv_nslots = 0;
  int* sv_slots_host = nullptr;    // pinned staging of the slot lists
  double* sv_out_host = nullptr;   // pinned staging of the values
  const unsigned char* step_bflag = nullptr;  // enqueue-time: bflag during a lazy step, else nullptr
  DevBuf part_g, part_e, part_r, sel_out, val_out, gain_out, ms_part, ms_off, ms_idx, ms_out;
  // sparse work-matrix path
  DevBuf ms_tanchor, ms_trad;
  DevBuf ms_mbuf, ms_setof, ms_pairs, ms_keys, ms_vals, ms_keys2, ms_vals2, ms_ukeys, ms_uvals, ms_cub;
  float4* pt0 = nullptr;  // per-point screen data seeded with d(., e0)
  int* ms_count = nullptr;
  int* ms_nruns = nullptr;
  int ms_mode = 1;        // 1: sparse path, tensor flag screen when available; 2: sparse, FFMA flag screen; 0: dense only

  // CUDA graphs of whole Greedy runs, keyed by k (rebuilt when buffers move)
  struct Graph {
    int k;  // (k << 2) | (timing << 1) | sharded
    int64_t c0, c1;  // the candidate range the graph's kernel arguments and grids hold
    int64_t epoch;
    int64_t launches;
    cudaGraphExec_t exec;
    long long decided = -1;  // decided lazy steps the replay must reproduce (-1: not specialised)
  };
  std::vector<Graph> graphs;
  // device-side sharded exchange (NCCL over NVLink, ebc_comm_init)
  ncclComm_t comm = nullptr;  // the device's shared communicator (not owned)
  int64_t comm_gen = -1;
  int nranks = 1, rank = 0;
  DevBuf tie_rec, tie_all, sel_hash;
  int* tie_err = nullptr;
  int comm_status = 0;  // flags of the last sharded run: 1 frontier overflow, 2 cross-rank mismatch
  // runs made eagerly once (captured on the next run with the same key and
  // candidate range) and the deepest ladder rung each of them reached
  struct Eager {
    int k;
    int64_t c0, c1;
    int lv;
    std::vector<char> dec;  // lazy steps the eager run decided with the first batch (1)
    long long decided = -1; // the eager run's stats[5] (every replay reproduces it)
  };
  std::vector<char>* rec_dec = nullptr;        // eager run: record each lazy step's decision here
  const std::vector<char>* cap_dec = nullptr;  // capture: steps decided in the eager run (no conditional node)
  bool spec_dec = true;                        // EBC200_SPEC_DECIDED=0: keep the conditional node on every lazy step
  std::vector<Eager> eager;
  int ladder_max = 3;         // deepest rung enqueued (L_DIRECT except while capturing)
  int64_t alloc_epoch = 0;
  bool use_graphs = true;
  bool capturing = false;  // a Greedy run is being captured into a graph
  // timing / accounting
  bool timing = false;
  std::vector<cudaEvent_t> ev;
  double last_ms[4] = {0, 0, 0, 0};
  int64_t launches = 0;
  std::string err;
};

namespace {

int fail(ebc_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  g_err = msg;
  return code;
}

#define CU(call)                                                                                   \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess)                                                                         \
      return fail(ctx, EBC_ECUDA, std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " + \
                                      __FILE__ + ":" + std::to_string(__LINE__) + " (" #call ")"); \
  } while (0)

#define KCHECK()                                                                                   \
  do {                                                                                             \
    ++ctx->launches;                                                                               \
    cudaError_t e_ = cudaGetLastError();                                                           \
    if (e_ != cudaSuccess)                                                                         \
      return fail(ctx, EBC_ECUDA, std::string("kernel launch failed: ") + cudaGetErrorString(e_) + \
                                      " at " + __FILE__ + ":" + std::to_string(__LINE__));         \
  } while (0)

// Per-step family events (timing mode).  While a run is being captured they
// become external event record nodes (cudaEventRecordExternal), which keep
// their timestamps on every replay; outside capture a plain record.
cudaError_t record_step_event(ebc_ctx* ctx, cudaEvent_t e) {
  return ctx->capturing ? cudaEventRecordWithFlags(e, ctx->stream, cudaEventRecordExternal)
                        : cudaEventRecord(e, ctx->stream);
}

int ensure(ebc_ctx* ctx, DevBuf& b, size_t bytes) {
  if (b.bytes >= bytes) return EBC_OK;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(ctx->stream, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone)
    return fail(ctx, EBC_ECUDA, "buffer growth during graph capture");  // the capture is abandoned, run stays eager
  if (b.p) cudaFreeAsync(b.p, ctx->stream);
  b.p = nullptr;
  b.bytes = 0;
  CU(cudaMallocAsync((void**)&b.p, bytes, ctx->stream));
  b.bytes = bytes;
  ++ctx->alloc_epoch;  // cached graphs hold the old pointers
  return EBC_OK;
}

// Dynamic shared memory of k_tile_anchor's staged form (0: the looped form).
size_t tile_anchor_smem(const ebc_ctx* ctx) {
  const size_t b = (size_t)ctx->tc_na * ((ctx->d + 3) / 4 * 4) * sizeof(float);
  return ctx->tc_na <= NA_ALL && b <= 160 * 1024 ? b : 0;
}

// Dynamic shared memory of k_refine_short (the window's rows in fp64); above
// 180 KB the classic k_refine serves short windows.
size_t short_refine_smem(const ebc_ctx* ctx) { return (size_t)RW * ctx->d * (sizeof(double) + sizeof(float)); }

// Row pitch (elements) of the device copy: 16-byte rows; for fp32 the pitch in
// float4 units is odd so that 4 or 8 consecutive rows read by one LDS.128 hit
// disjoint bank groups.

int pitch_for(int d, int dtype) {
  if (dtype == EBC_F64) return (d + 1) / 2 * 2;
  int p = (d + 3) / 4 * 4;
  if ((p / 4) % 2 == 0) p += 4;
  return p;
}

struct ScreenPlan {
  int shape;  // 0 = ScreenA (2-stage), 1 = ScreenA4 (4-stage), 2 = ScreenB
  size_t smem;
  int ncb;
  int ntiles;
  int tps;
  int nsplit;
  int tp;
};

template <class Cfg>
int plan_shape(const ebc_ctx* ctx, ScreenPlan& p) {
  p.smem = Cfg::smem_bytes(ctx->pitch);
  p.tp = Cfg::TP;
  const int64_t ncand = ctx->c1 - ctx->c0;
  p.ncb = (int)((ncand + Cfg::CT - 1) / Cfg::CT);
  p.ntiles = (int)((ctx->n + Cfg::PT - 1) / Cfg::PT);
  // choose the V split that minimises (waves x tiles per CTA), with one tile
  // of fixed cost per CTA (candidate-tile load, epilogue): wave quantisation
  // otherwise costs up to ~1/waves of the step
  int per_sm = (int)std::min<size_t>(Cfg::MINB, (227 * 1024) / (p.smem + 1024));
  if (per_sm < 1) per_sm = 1;
  const int64_t slots = (int64_t)per_sm * ctx->num_sms;
  double best_cost = 1e300;
  p.tps = p.ntiles;
  for (int s = 1; s <= 64 && s <= p.ntiles; ++s) {
    const int tps = (p.ntiles + s - 1) / s;
    const int ns = (p.ntiles + tps - 1) / tps;
    const int64_t ctas = (int64_t)p.ncb * ns;
    const double waves = (double)((ctas + slots - 1) / slots);
    const double cost = waves * (tps + 1.0);
    if (cost < best_cost * 0.999) {
      best_cost = cost;
      p.tps = tps;
    }
  }
  p.nsplit = (p.ntiles + p.tps - 1) / p.tps;
  return p.smem <= 227 * 1024 ? EBC_OK : EBC_EINVAL;
}

int screen_shape_choice(const ebc_ctx* ctx) {
  const char* env = getenv("EBC200_SCREEN");
  if (env && env[0]) return atoi(env);
  (void)ctx;
  return 2;
}

int plan_screen(const ebc_ctx* ctx, ScreenPlan& p) {
  if (ctx->screen_mode < 0) return EBC_EINVAL;  // out of the fp32 range: exact refine only
  p.shape = screen_shape_choice(ctx);
  int rc;
  if (p.shape == 2) {
    rc = plan_shape<ScreenB>(ctx, p);
    if (rc == EBC_OK) return rc;
    p.shape = 0;
  }
  if (p.shape == 1) {
    rc = plan_shape<ScreenA4>(ctx, p);
    if (rc == EBC_OK && p.smem <= 110 * 1024) return rc;
    p.shape = 0;
  }
  return plan_shape<ScreenA>(ctx, p);
}

template <class Cfg, int MODE, int PITCH = 0>
int launch_screen_t(ebc_ctx* ctx, const ScreenPlan& p, const int* level_now, int level, const float* Vc = nullptr,
                    FlagOut fo = FlagOut{}, const float4* ptv = nullptr) {
  auto kern = k_screen<Cfg, MODE, PITCH>;
  CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
  dim3 grid(p.ncb, p.nsplit);
  kern<<<grid, Cfg::THREADS, p.smem, ctx->stream>>>(ctx->V32, ptv ? ptv : ctx->pt, ctx->pitch, ctx->d4, ctx->c0,
                                                    p.ntiles, p.tps,
                                                    (double*)ctx->part_g.p, (float*)ctx->part_e.p, ctx->n_pad,
                                                    ctx->gram_kc, level_now, level, Vc, fo);
  KCHECK();
  return EBC_OK;
}

template <int MODE>
int launch_screen(ebc_ctx* ctx, const ScreenPlan& p, const int* level_now, int level, const float* Vc = nullptr,
                  FlagOut fo = FlagOut{}, const float4* ptv = nullptr) {
  if (p.shape == 2) {
    // compile-time pitches for the BASELINE dims (16, 32, 64, 100)
    switch (ctx->pitch) {
      case 20: return launch_screen_t<ScreenB, MODE, 20>(ctx, p, level_now, level, Vc, fo, ptv);
      case 36: return launch_screen_t<ScreenB, MODE, 36>(ctx, p, level_now, level, Vc, fo, ptv);
      case 68: return launch_screen_t<ScreenB, MODE, 68>(ctx, p, level_now, level, Vc, fo, ptv);
      case 100: return launch_screen_t<ScreenB, MODE, 100>(ctx, p, level_now, level, Vc, fo, ptv);
      default: return launch_screen_t<ScreenB, MODE>(ctx, p, level_now, level, Vc, fo, ptv);
    }
  }
  if (p.shape == 1) return launch_screen_t<ScreenA4, MODE>(ctx, p, level_now, level, Vc, fo, ptv);
  return launch_screen_t<ScreenA, MODE>(ctx, p, level_now, level, Vc, fo, ptv);
}

// The refine may skip certified-unreachable chunks when the tensor screen's
// anchors exist and cmx was refreshed for this step (run_screen_window).
bool refine_prune_on(const ebc_ctx* ctx) {
  return ctx->tc_np && ctx->tc_prune && ctx->screen_mode == 3 && ctx->dtype != EBC_F64 && (RCH % ctx->tc_np) == 0 &&
         ctx->crad;
}

template <typename T, bool BIGD>
int launch_refine(ebc_ctx* ctx, const T* V, int grid, size_t smem, int ng, const int* skip_level,
                  const RefineFinal& fin) {
  CU(cudaFuncSetAttribute(k_refine<T, BIGD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem + 1024));
  RefinePrune pr;
  if (refine_prune_on(ctx) && ctx->cmx_fresh) {
    pr.rho = ctx->rho;
    pr.kpstride = ctx->tc_ntl;
    pr.cmx = ctx->cmx;
    pr.tile_anchor = ctx->tile_anchor;
    pr.anchors = ctx->anchors;
    pr.apitch = ctx->pitch;
    pr.np = ctx->tc_np;
    pr.crad = ctx->crad;
  }
  k_refine<T, BIGD><<<grid, RED_THREADS, smem, ctx->stream>>>(V, ctx->pitch, ctx->n, ctx->d, ctx->cm64, ctx->wcount,
                                                             ctx->wlist, ctx->nchunks, ng, (double*)ctx->part_r.p, pr,
                                                             skip_level, fin);
  KCHECK();
  return EBC_OK;
}

// FP64 grounds, or a d too large for any screen tile: every unselected
// candidate goes straight to the exact fp64 refine.
int run_window_all(ebc_ctx* ctx, int eb, int fin_blocks) {
  if (ctx->timing) {
    CU(record_step_event(ctx, ctx->ev[eb + 0]));
    CU(record_step_event(ctx, ctx->ev[eb + 1]));
  }
  k_window_all<<<fin_blocks, 256, 0, ctx->stream>>>(ctx->c0, ctx->c1, ctx->selected, ctx->wcount, ctx->wlist);
  KCHECK();
  return EBC_OK;
}

// finalize + window of one screen pass (gscale 2 for the Gram forms, whose
// accumulators hold t/2).  nterms bounds the terms of one fp32 error
// accumulator; gterms the fp32 terms summed before each fp64 fold.
int run_finalize_window(ebc_ctx* ctx, int nsplit, double nterms, int gterms, int fin_blocks, double gscale,
                        const int* level_now, int level, bool ub_only = false, const double* part_a = nullptr) {
  const double u = 5.960464477539063e-08;
  const double einfl = 1.0 + 2.0 * (nterms + 64.0) * u + 1.0 / 64.0;
  const double gcoef = (gterms + 8) * u;
  k_finalize<<<fin_blocks, 256, 0, ctx->stream>>>(ctx->c0, ctx->c1, nsplit, (double*)ctx->part_g.p,
                                                 (float*)ctx->part_e.p, ctx->n_pad, einfl, gcoef, gscale,
                                                 ctx->selected, ctx->ub, ctx->maxlb, level_now, level, ub_only ? 1 : 0,
                                                 part_a, ctx->step_bflag, ctx->lazy_on ? ctx->ubp : nullptr);
  KCHECK();
  if (ub_only) {
    // window threshold = exact gain of the candidate with the largest bound
    // grid <= ceil(ncand / 1024) <= nchunks: its (value, index) partials fit the
    // 4 nchunks doubles of toppart, which k_gain_top overwrites afterwards
    const int ag = (int)std::max<int64_t>(1, std::min<int64_t>(2 * ctx->num_sms, (ctx->c1 - ctx->c0 + 1023) / 1024));
    k_argmax_ub<<<ag, 256, 0, ctx->stream>>>(ctx->c0, ctx->c1, ctx->ub, ctx->topc, ctx->toppart, ctx->counter2,
                                            level_now, level);
    KCHECK();
    const size_t smem = (size_t)ctx->d * sizeof(double);
    if (ctx->dtype == EBC_F64) {
      CU(cudaFuncSetAttribute(k_gain_top<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem + 1024));
      k_gain_top<double><<<(unsigned)((ctx->n + RED_THREADS - 1) / RED_THREADS), RED_THREADS, smem, ctx->stream>>>(
          ctx->V64, ctx->pitch, ctx->n, ctx->d, ctx->cm64, ctx->topc, ctx->toppart, ctx->counter2, ctx->maxlb,
          level_now, level);
    } else {
      CU(cudaFuncSetAttribute(k_gain_top<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem + 1024));
      k_gain_top<float><<<(unsigned)((ctx->n + RED_THREADS - 1) / RED_THREADS), RED_THREADS, smem, ctx->stream>>>(
          ctx->V32, ctx->pitch, ctx->n, ctx->d, ctx->cm64, ctx->topc, ctx->toppart, ctx->counter2, ctx->maxlb,
          level_now, level);
    }
    KCHECK();
  }
  const double margin = (double)ctx->n * 1e-12 * std::max(1.0, std::fabs(ctx->baseline)) * 1.01;
  k_window<<<fin_blocks, 256, 0, ctx->stream>>>(ctx->c0, ctx->c1, ctx->ub, ctx->maxlb, margin, ctx->wcount,
                                               ctx->wlist, level_now, level);
  KCHECK();
  return EBC_OK;
}

// Rungs of the adaptive screen ladder: the fast FP16-rounded
// tensor screen, the BF16-split (or FP16 / TF32) tensor screen, the FFMA Gram
// screen, the direct screen.
enum { L_FAST = 0, L_TC = 1, L_GRAM = 2, L_DIRECT = 3 };

struct TcPlan {
  int ncb, ntiles, tps, nsplit;
  size_t smem;
  int stages;
  int list_cap;  // kept-tile list entries (0: pruning off)
  int kq_cap;    // per-tile {kpmax, vmax} entries staged in smem (0: read per tile)
};

int tc_es(int kind) { return kind == tc::KIND_TF32 ? 4 : 2; }
int tc_parts(int kind) { return tc::one_product(kind) ? 1 : 2; }

bool plan_tc(const ebc_ctx* ctx, TcPlan& p, int kind) {
  // the screen reads each candidate block's anchor and radius as
  // tile_anchor/tile_rad[crow >> 7]: blocks must start on a 128-row boundary
  if (!ctx->tc_np || (ctx->c0 % tc::M) != 0) return false;
  const int64_t ncand = ctx->c1 - ctx->c0;
  p.ncb = (int)((ncand + tc::M - 1) / tc::M);
  p.ntiles = (int)((ctx->n + ctx->tc_np - 1) / ctx->tc_np);
  const int64_t slots = ctx->num_sms;  // one CTA per SM
  double best_cost = 1e300;
  p.tps = p.ntiles;
  for (int s = 1; s <= 64 && s <= p.ntiles; ++s) {
    const int tps = (p.ntiles + s - 1) / s;
    const int ns = (p.ntiles + tps - 1) / tps;
    const double waves = (double)(((int64_t)p.ncb * ns + slots - 1) / slots);
    const double cost = waves * (tps + 2.0);
    if (cost < best_cost * 0.999) {
      best_cost = cost;
      p.tps = tps;
    }
  }
  p.nsplit = (p.ntiles + p.tps - 1) / p.tps;
  const int es = tc_es(kind), parts = tc_parts(kind);
  // per-tile {kpmax, vmax} staged in smem ahead of the kept-tile list (<= 16 KB)
  p.kq_cap = p.tps <= 2048 ? p.tps : 0;
  const size_t kqb = (size_t)p.kq_cap * 8;
  p.list_cap = 0;
  p.stages = tc::stages_for(ctx->kpad, ctx->tc_np, es, parts, kqb);
  if (ctx->tc_prune && p.tps <= 65535) {
    const size_t lb = tc::list_bytes_for(p.tps);
    const int st = tc::stages_for(ctx->kpad, ctx->tc_np, es, parts, lb + kqb);
    if (st >= 2 && st >= p.stages - 1) {  // keep the ring at least as deep, minus one stage at most
      p.list_cap = p.tps;
      p.stages = st;
    }
  }
  p.smem = tc::smem_bytes(ctx->kpad, ctx->tc_np, es, parts, (p.list_cap ? tc::list_bytes_for(p.tps) : 0) + kqb);
  return true;
}

template <int NP, int KIND>
int launch_tc_t(ebc_ctx* ctx, const TcPlan& p, const int* level_now, int level) {
  constexpr bool one = tc::one_product(KIND);
  const bool ms = one && ctx->tc_mseed;
  auto kern = ms ? k_screen_tc<NP, KIND, false, one> : k_screen_tc<NP, KIND>;
  CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
  dim3 grid(p.ncb, p.nsplit);
  constexpr bool fast = KIND == tc::KIND_F16R;
  // folded seeds use the origin anchor: rung 0 (anchored otherwise) gets the
  // all-zero anchor map and no tile-pair pruning (its radii belong to the
  // chosen anchors); fp16-stored grounds have the origin as their only anchor
  const bool origin_only = ms && fast;
  TcAnchors an{ctx->anchors, ctx->pitch, origin_only ? ctx->tile_anchor0 : ctx->tile_anchor, ctx->pttc, ctx->n_pad,
               ctx->kpmax, ctx->tc_ntl, ctx->tc_vmax, ctx->tc_kc, fast ? ctx->tc_kx_fast : ctx->tc_kx,
               (p.list_cap && !origin_only) ? ctx->rho : nullptr, ctx->tile_rad, ctx->cmx, p.list_cap, p.kq_cap,
               (unsigned long long*)(ctx->stats + 4)};
  if (!one && ctx->tc_agg && p.list_cap) {
    an.rhomax = ctx->rhomax;
    an.cmn = ctx->cmn;
  }
  an.bflag = ctx->step_bflag;
  if (ms) {
    an.kpscale = ctx->tc_kpscale;
    an.keta2 = (float)std::ldexp(1.0, -24);  // seed split residual (fp16 subnormal), unscaled operands
  }
  if (fast) {
    an.oscale = ctx->tc_oscale;
    an.sinv2 = ctx->tc_sinv2;
    an.keta = ctx->tc_keta;
    an.keta2 = ctx->tc_keta2;
  }
  if constexpr (one && NP == 128) {
    if (ms && ctx->tc_mb2) {
      // two candidate blocks per CTA on 64-point tiles: the same
      // split of the point range (twice the tiles per split), half the CTAs
      auto k2 = k_screen_tc<64, KIND, false, true, 2>;
      const int tps2 = 2 * p.tps, nt2 = 2 * p.ntiles;
      const int kqc = tps2 <= 4096 ? tps2 : 0;
      const size_t kqb = (size_t)kqc * 8;
      const int st = tc::stages_for(ctx->kpad, 64, 2, 1, kqb);
      const size_t sm = tc::smem_bytes(ctx->kpad, 64, 2, 1, kqb);
      CU(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      an.rho = nullptr;  // no tile-pair pruning in the two-block shape
      an.list_cap = 0;
      an.kq_cap = kqc;
      dim3 g2((p.ncb + 1) / 2, p.nsplit);
      k2<<<g2, tc::THREADS, sm, ctx->stream>>>(ctx->V32, ctx->pitch, ctx->d,
                                               (const unsigned char*)(fast ? ctx->Vf : ctx->Vhi),
                                               (const unsigned char*)ctx->Vlo, an, ctx->kpad, st, ctx->c0, nt2, tps2,
                                               (double*)ctx->part_g.p, (float*)ctx->part_e.p, ctx->n_pad, level_now,
                                               level, nullptr, FlagOut{});
      KCHECK();
      return EBC_OK;
    }
  }
  kern<<<grid, tc::THREADS, p.smem, ctx->stream>>>(ctx->V32, ctx->pitch, ctx->d,
                                                   (const unsigned char*)(fast ? ctx->Vf : ctx->Vhi),
                                                   (const unsigned char*)ctx->Vlo, an, ctx->kpad, p.stages, ctx->c0,
                                                   p.ntiles, p.tps, (double*)ctx->part_g.p, (float*)ctx->part_e.p,
                                                   ctx->n_pad, level_now, level, nullptr, FlagOut{});
  KCHECK();
  return EBC_OK;
}

// Work-matrix flag screen on the tensor cores: candidates = gathered member rows.
template <int NP, int KIND>
int launch_tc_flag_t(ebc_ctx* ctx, const TcPlan& p, const float* Vc, const int* tanchor, const float* trad,
                     FlagOut fo) {
  auto kern = k_screen_tc<NP, KIND, true>;
  CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
  dim3 grid(p.ncb, p.nsplit);
  TcAnchors an{ctx->anchors, ctx->pitch, tanchor, ctx->ipa0, ctx->n_pad, ctx->kpmax, ctx->tc_ntl,
               ctx->tc_vmax, ctx->tc_kc, ctx->tc_kx, p.list_cap ? ctx->rho : nullptr, trad, ctx->cmx0,
               p.list_cap, p.kq_cap, nullptr};
  kern<<<grid, tc::THREADS, p.smem, ctx->stream>>>(ctx->V32, ctx->pitch, ctx->d, (const unsigned char*)ctx->Vhi,
                                                   (const unsigned char*)ctx->Vlo, an, ctx->kpad, p.stages, 0,
                                                   p.ntiles, p.tps, nullptr, nullptr, 0, nullptr, 0, Vc, fo);
  KCHECK();
  return EBC_OK;
}

int launch_tc_flag(ebc_ctx* ctx, const TcPlan& p, const float* Vc, const int* tanchor, const float* trad,
                   FlagOut fo) {
  switch (ctx->tc_kind) {
    case tc::KIND_F16:
      if (ctx->tc_np == 128) return launch_tc_flag_t<128, tc::KIND_F16>(ctx, p, Vc, tanchor, trad, fo);
      return launch_tc_flag_t<64, tc::KIND_F16>(ctx, p, Vc, tanchor, trad, fo);
    case tc::KIND_BF16:
      if (ctx->tc_np == 128) return launch_tc_flag_t<128, tc::KIND_BF16>(ctx, p, Vc, tanchor, trad, fo);
      return launch_tc_flag_t<64, tc::KIND_BF16>(ctx, p, Vc, tanchor, trad, fo);
    default:
      if (ctx->tc_np == 128) return launch_tc_flag_t<128, tc::KIND_TF32>(ctx, p, Vc, tanchor, trad, fo);
      return launch_tc_flag_t<64, tc::KIND_TF32>(ctx, p, Vc, tanchor, trad, fo);
  }
}

int launch_tc(ebc_ctx* ctx, const TcPlan& p, const int* level_now, int level, int kind) {
  switch (kind) {
    case tc::KIND_F16R:
      if (ctx->tc_np == 128) return launch_tc_t<128, tc::KIND_F16R>(ctx, p, level_now, level);
      return launch_tc_t<64, tc::KIND_F16R>(ctx, p, level_now, level);
    case tc::KIND_F16:
      if (ctx->tc_np == 128) return launch_tc_t<128, tc::KIND_F16>(ctx, p, level_now, level);
      return launch_tc_t<64, tc::KIND_F16>(ctx, p, level_now, level);
    case tc::KIND_BF16:
      if (ctx->tc_np == 128) return launch_tc_t<128, tc::KIND_BF16>(ctx, p, level_now, level);
      return launch_tc_t<64, tc::KIND_BF16>(ctx, p, level_now, level);
    default:
      if (ctx->tc_np == 128) return launch_tc_t<128, tc::KIND_TF32>(ctx, p, level_now, level);
      return launch_tc_t<64, tc::KIND_TF32>(ctx, p, level_now, level);
  }
}

// All-positive (block, tile) pairs of rung 1 from tile aggregates (same plan and
// anchors as the rung-1 screen launch).
int launch_tc_agg(ebc_ctx* ctx, const TcPlan& p) {
  TcAnchors an{ctx->anchors, ctx->pitch, ctx->tile_anchor, ctx->pttc, ctx->n_pad, ctx->kpmax, ctx->tc_ntl,
               ctx->tc_vmax, ctx->tc_kc, ctx->tc_kx, ctx->rho, ctx->tile_rad, ctx->cmx, p.list_cap, 0, nullptr};
  an.rhomax = ctx->rhomax;
  an.cmn = ctx->cmn;
  an.bflag = ctx->step_bflag;
  // W (d doubles) and its 128 group partials, then the all-positive tile list
  const size_t smem = ((size_t)ctx->d + 128) * sizeof(double) + ((size_t)p.tps * 2 + 16);
  dim3 grid(p.ncb, p.nsplit);
  CU(cudaFuncSetAttribute(k_screen_agg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_screen_agg<<<grid, 128, smem, ctx->stream>>>(ctx->V32, ctx->pitch, ctx->d, an, ctx->c0, p.ntiles, p.tps,
                                                 ctx->tc_np, ctx->n, ctx->ipsum, ctx->vsum, ctx->vsn,
                                                 (double*)ctx->part_a.p, ctx->n_pad, ctx->level, L_TC, ctx->agg_any);
  KCHECK();
  return EBC_OK;
}

// fp32 screen of the candidate range + certified window.
// Modes: 0 direct form; 1 FFMA Gram form (v.c on the FMA pipe); 2 adaptive
// ladder FFMA Gram -> direct; 3 adaptive ladder tensor-core Gram -> FFMA Gram
// -> direct.  A rung whose window comes out wider than ctx->wcap hands the step
// (and the rest of the run) to the next rung: the Gram bounds scale with
// |v|^2 + |c|^2, the direct one with cm, so clustered data walks down the ladder.
// Returns EBC_EINVAL (nothing launched) when no screen tile fits this d.
int run_screen_window(ebc_ctx* ctx, int eb, int fin_blocks) {
  ctx->cmx_fresh = false;
  ScreenPlan p;
  int rc = plan_screen(ctx, p);
  if (rc) return rc;
  TcPlan tp{}, fp{};
  const bool use_tc = ctx->screen_mode == 3 && plan_tc(ctx, tp, ctx->tc_kind);
  const bool use_fast = use_tc && ctx->tc_fast && plan_tc(ctx, fp, tc::KIND_F16R);
  const int nsplit_max = std::max(std::max(p.nsplit, use_tc ? tp.nsplit : 0), use_fast ? fp.nsplit : 0);
  rc = ensure(ctx, ctx->part_g, (size_t)nsplit_max * ctx->n_pad * sizeof(double));
  if (rc) return rc;
  rc = ensure(ctx, ctx->part_e, (size_t)nsplit_max * ctx->n_pad * sizeof(float));
  if (rc) return rc;
  if (ctx->timing && !ctx->screen_events_outside) CU(record_step_event(ctx, ctx->ev[eb + 0]));
  // lower bounds are clamped at 0 (every gain is a sum of max(0, .) terms), so
  // key 0 (= +0.0) is a valid neutral element for the max
  if (!ctx->step_bflag) CU(cudaMemsetAsync(ctx->maxlb, 0, sizeof(long long), ctx->stream));
  const double nterms_ffma = (double)p.tps * p.tp * 8 * 2;
  if (ctx->screen_mode == 0 || ctx->screen_mode == 1) {
    // single-rung modes: level[] holds L_GRAM for the whole run (do_reset), so
    // the gate only switches the pass off in lazy steps decided without it
    if (ctx->screen_mode == 0) rc = launch_screen<0>(ctx, p, ctx->level, L_GRAM);
    else rc = launch_screen<1>(ctx, p, ctx->level, L_GRAM);
    if (!rc)
      rc = run_finalize_window(ctx, p.nsplit, nterms_ffma, p.tp, fin_blocks, ctx->screen_mode == 0 ? 1.0 : 2.0,
                               ctx->level, L_GRAM);
  } else {
    if (use_tc) {
      const bool agg = ctx->tc_agg && tp.list_cap && ctx->ladder_max >= L_TC;
      if (tp.list_cap || fp.list_cap || refine_prune_on(ctx)) {
        k_tile_cmmax<<<(unsigned)((ctx->tc_ntl * 32 + 255) / 256), 256, 0, ctx->stream>>>(
            ctx->cm64, ctx->n, ctx->tc_ntl, ctx->tc_np, ctx->cmx, agg ? ctx->cmn : nullptr);
        KCHECK();
        ctx->cmx_fresh = true;  // this step's refine may prune with it
      }
      if (agg) {
        rc = ensure(ctx, ctx->part_a, (size_t)tp.nsplit * ctx->n_pad * sizeof(double));
        if (rc) return rc;
        const int64_t cells = (int64_t)ctx->tc_na * ctx->tc_ntl;
        CU(cudaMemsetAsync(ctx->agg_any, 0, sizeof(int), ctx->stream));
        k_tile_ipsum<<<(unsigned)((cells * 32 + 255) / 256), 256, 0, ctx->stream>>>(
            ctx->pttc, ctx->n_pad, ctx->tc_na, ctx->n, ctx->tc_ntl, ctx->tc_np, ctx->ipsum, ctx->rhomin, ctx->radmin,
            ctx->cmn, ctx->agg_any, ctx->level);
        KCHECK();
      }
      // ladder_max < L_DIRECT only while capturing a graph of a run whose eager
      // pass never went below that rung: the rungs below are not enqueued and the
      // last enqueued rung keeps its window however wide (still exact -- the
      // refine evaluates any window; only speed is at stake)
      if (use_fast) {
        rc = launch_tc(ctx, fp, ctx->level, L_FAST, tc::KIND_F16R);
        if (!rc) rc = run_finalize_window(ctx, fp.nsplit, (double)fp.tps * ctx->tc_np, 32, fin_blocks, 2.0,
                                          ctx->level, L_FAST, /*ub_only=*/true);
        if (!rc && ctx->ladder_max > L_FAST) {
          k_adapt<<<1, 32, 0, ctx->stream>>>(ctx->wcount, ctx->maxlb, ctx->wcap_fast, ctx->level, L_FAST);
          KCHECK();
        }
      }
      if (ctx->ladder_max >= L_TC) {
        if (!rc) rc = launch_tc(ctx, tp, ctx->level, L_TC, ctx->tc_kind);
        if (!rc && agg) rc = launch_tc_agg(ctx, tp);
        if (!rc) rc = run_finalize_window(ctx, tp.nsplit, (double)tp.tps * ctx->tc_np, 32, fin_blocks, 2.0,
                                          ctx->level, L_TC, /*ub_only=*/true, agg ? (double*)ctx->part_a.p : nullptr);
        if (!rc && ctx->ladder_max > L_TC) {
          k_adapt<<<1, 32, 0, ctx->stream>>>(ctx->wcount, ctx->maxlb, ctx->wcap_tc, ctx->level, L_TC);
          KCHECK();
        }
      }
    }
    if (ctx->ladder_max >= L_GRAM) {
      if (!rc) rc = launch_screen<1>(ctx, p, ctx->level, L_GRAM);
      if (!rc) rc = run_finalize_window(ctx, p.nsplit, nterms_ffma, p.tp, fin_blocks, 2.0, ctx->level, L_GRAM);
      if (!rc && ctx->ladder_max > L_GRAM) {
        k_adapt<<<1, 32, 0, ctx->stream>>>(ctx->wcount, ctx->maxlb, ctx->wcap, ctx->level, L_GRAM);
        KCHECK();
      }
    }
    if (ctx->ladder_max >= L_DIRECT) {
      if (!rc) rc = launch_screen<0>(ctx, p, ctx->level, L_DIRECT);
      if (!rc) rc = run_finalize_window(ctx, p.nsplit, nterms_ffma, p.tp, fin_blocks, 1.0, ctx->level, L_DIRECT);
    }
  }
  if (rc) return rc;
  if (ctx->timing && !ctx->screen_events_outside) CU(record_step_event(ctx, ctx->ev[eb + 1]));
  return EBC_OK;
}

// One step's candidate screen + certified window + exact refine + pick.
// commit: single-device mode (mark the winner, record it as step `step`).
// Gathered lazy re-screen (level[0] == L_GATHER): the stale candidates packed
// into gath_cap rows, their own block anchors and radii, the split-rung tensor
// screen over them (no all-positive aggregates), bounds per slot, then the
// usual argmax -> exact top gain -> window chain.  Every kernel is gated on
// L_GATHER (eager runs) and the whole section sits in a conditional node
// (captured runs).
template <int NP, int KIND>
int launch_tc_gathered_t(ebc_ctx* ctx, const TcPlan& p) {
  auto kern = k_screen_tc<NP, KIND>;
  CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
  TcAnchors an{ctx->anchors, ctx->pitch, ctx->g_anchor, ctx->pttc, ctx->n_pad, ctx->kpmax, ctx->tc_ntl,
               ctx->tc_vmax, ctx->tc_kc, ctx->tc_kx, p.list_cap ? ctx->rho : nullptr, ctx->g_rad, ctx->cmx,
               p.list_cap, p.kq_cap, (unsigned long long*)(ctx->stats + 4)};
  an.ncand_dev = ctx->scount;
  dim3 grid(p.ncb, p.nsplit);
  kern<<<grid, tc::THREADS, p.smem, ctx->stream>>>(ctx->V32, ctx->pitch, ctx->d, (const unsigned char*)ctx->Vhi,
                                                   (const unsigned char*)ctx->Vlo, an, ctx->kpad, p.stages, 0,
                                                   p.ntiles, p.tps, (double*)ctx->part_g.p, (float*)ctx->part_e.p,
                                                   ctx->n_pad, ctx->level, L_GATHER, ctx->Vg, FlagOut{});
  KCHECK();
  return EBC_OK;
}

int run_gathered_window(ebc_ctx* ctx, int fin_blocks) {
  TcPlan gp{};
  const int64_t s0 = ctx->c0, s1 = ctx->c1;
  ctx->c0 = 0;
  ctx->c1 = ctx->gath_cap;
  const bool ok = plan_tc(ctx, gp, ctx->tc_kind);
  ctx->c0 = s0;
  ctx->c1 = s1;
  if (!ok) return fail(ctx, EBC_ECUDA, "gathered re-screen: no tensor plan");
  int rc = ensure(ctx, ctx->part_g, (size_t)gp.nsplit * ctx->n_pad * sizeof(double));
  if (!rc) rc = ensure(ctx, ctx->part_e, (size_t)gp.nsplit * ctx->n_pad * sizeof(float));
  if (rc) return rc;
  const int64_t ncand = ctx->c1 - ctx->c0;
  // tile maxima of the current cached minima (pruning)
  k_tile_cmmax<<<(unsigned)((ctx->tc_ntl * 32 + 255) / 256), 256, 0, ctx->stream>>>(ctx->cm64, ctx->n, ctx->tc_ntl,
                                                                                  ctx->tc_np, ctx->cmx, nullptr);
  KCHECK();
  k_gather_rows<<<8 * ctx->num_sms, 256, 0, ctx->stream>>>(ctx->V32, ctx->pitch, ctx->slist, ctx->scount,
                                                          (int)ctx->gath_cap, ctx->Vg, ctx->ub, ncand, ctx->level,
                                                          L_GATHER);
  KCHECK();
  k_tile_anchor<<<(unsigned)(ctx->gath_cap / tc::M), 128, tile_anchor_smem(ctx), ctx->stream>>>(
      ctx->Vg, ctx->pitch, ctx->gath_cap, ctx->d, ctx->anchors, ctx->pitch, ctx->tc_na, ctx->g_anchor, ctx->g_rad,
      tile_anchor_smem(ctx) > 0, ctx->scount, ctx->level, L_GATHER);
  KCHECK();
  switch (ctx->tc_kind) {
    case tc::KIND_BF16:
      rc = ctx->tc_np == 128 ? launch_tc_gathered_t<128, tc::KIND_BF16>(ctx, gp)
                             : launch_tc_gathered_t<64, tc::KIND_BF16>(ctx, gp);
      break;
    default:
      rc = ctx->tc_np == 128 ? launch_tc_gathered_t<128, tc::KIND_TF32>(ctx, gp)
                             : launch_tc_gathered_t<64, tc::KIND_TF32>(ctx, gp);
  }
  if (rc) return rc;
  const double u = 5.960464477539063e-08;
  const double nterms = (double)gp.tps * ctx->tc_np;
  const double einfl = 1.0 + 2.0 * (nterms + 64.0) * u + 1.0 / 64.0;
  const double gcoef = (32 + 8) * u;
  k_finalize_gathered<<<(unsigned)((ctx->gath_cap + 255) / 256), 256, 0, ctx->stream>>>(
      ctx->scount, ctx->slist, ctx->c0, gp.nsplit, (const double*)ctx->part_g.p, (const float*)ctx->part_e.p,
      ctx->n_pad, einfl, gcoef, 2.0, ctx->selected, ctx->ub, ctx->ubp, ctx->level, L_GATHER);
  KCHECK();
  const int ag = (int)std::max<int64_t>(1, std::min<int64_t>(2 * ctx->num_sms, (ncand + 1023) / 1024));
  k_argmax_ub<<<ag, 256, 0, ctx->stream>>>(ctx->c0, ctx->c1, ctx->ub, ctx->topc, ctx->toppart, ctx->counter2,
                                          ctx->level, L_GATHER);
  KCHECK();
  const size_t smem = (size_t)ctx->d * sizeof(double);
  CU(cudaFuncSetAttribute(k_gain_top<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem + 1024));
  k_gain_top<float><<<(unsigned)((ctx->n + RED_THREADS - 1) / RED_THREADS), RED_THREADS, smem, ctx->stream>>>(
      ctx->V32, ctx->pitch, ctx->n, ctx->d, ctx->cm64, ctx->topc, ctx->toppart, ctx->counter2, ctx->maxlb,
      ctx->level, L_GATHER);
  KCHECK();
  const double margin = (double)ctx->n * 1e-12 * std::max(1.0, std::fabs(ctx->baseline)) * 1.01;
  k_window<<<fin_blocks, 256, 0, ctx->stream>>>(ctx->c0, ctx->c1, ctx->ub, ctx->maxlb, margin, ctx->wcount,
                                               ctx->wlist, ctx->level, L_GATHER);
  KCHECK();
  return EBC_OK;
}

// Exact fp64 gains of the window (wcount / wlist) into part_r, then the pick
// in the refine's last block (fin); skip_level: the kernel exits when it reads
// -2 there (lazy step decided by the first batch).
int enqueue_refine(ebc_ctx* ctx, int ng, const int* skip_level, const RefineFinal& fin) {
  const int rgrid = 4 * ctx->num_sms;
  const bool bigd = (size_t)RW * ctx->d * sizeof(double) > 160 * 1024;
  const size_t rsmem = bigd ? 0 : (size_t)RW * ctx->d * sizeof(double);
  if (ctx->dtype == EBC_F64)
    return bigd ? launch_refine<double, true>(ctx, ctx->V64, rgrid, rsmem, ng, skip_level, fin)
                : launch_refine<double, false>(ctx, ctx->V64, rgrid, rsmem, ng, skip_level, fin);
  return bigd ? launch_refine<float, true>(ctx, ctx->V32, rgrid, rsmem, ng, skip_level, fin)
              : launch_refine<float, false>(ctx, ctx->V32, rgrid, rsmem, ng, skip_level, fin);
}

// Refine of a window of at most RW candidates (the lazy first batch): one
// RCH-thread block per chunk, the classic reduction replayed (kernels.cuh).
int enqueue_refine_short(ebc_ctx* ctx, int ng, const RefineFinal& fin, const int* wcount = nullptr,
                         const int64_t* wlist = nullptr) {
  if (!wcount) {
    wcount = ctx->wcount;
    wlist = ctx->wlist;
  }
  RefinePrune pr;
  if (refine_prune_on(ctx) && ctx->cmx_fresh) {
    pr.rho = ctx->rho;
    pr.kpstride = ctx->tc_ntl;
    pr.cmx = ctx->cmx;
    pr.tile_anchor = ctx->tile_anchor;
    pr.anchors = ctx->anchors;
    pr.apitch = ctx->pitch;
    pr.np = ctx->tc_np;
    pr.crad = ctx->crad;
  }
  const size_t smem = short_refine_smem(ctx);
  if (smem > 180 * 1024) {
    if (wcount != ctx->wcount) return EBC_EINVAL;  // callers check short_refine_smem first
    return enqueue_refine(ctx, ng, nullptr, fin);
  }
  int rc = ensure(ctx, ctx->rterms, (size_t)RW * ctx->nchunks * sizeof(double));
  if (rc) return rc;
  // per-point terms (RW x n_pad) and the per-chunk tickets (zeroed when allocated)
  const size_t xbytes = (size_t)RW * ctx->n_pad * sizeof(double);
  const size_t sbytes = xbytes + (size_t)ctx->nchunks * sizeof(unsigned int);
  const bool fresh = ctx->sxt.bytes < sbytes;
  if ((rc = ensure(ctx, ctx->sxt, sbytes))) return rc;
  if (fresh) CU(cudaMemsetAsync((unsigned char*)ctx->sxt.p + xbytes, 0, sbytes - xbytes, ctx->stream));
  ShortBufs sb;
  sb.xt = (double*)ctx->sxt.p;
  sb.xstride = ctx->n_pad;
  sb.chunk_ticket = (unsigned int*)((unsigned char*)ctx->sxt.p + xbytes);
  const unsigned grid = (unsigned)(ctx->nchunks * SHORT_SPLIT);
  // staged rows (bulk copies) when a 256-row slice fits next to the window rows
  const size_t esz = ctx->dtype == EBC_F64 ? sizeof(double) : sizeof(float);
  const size_t stage = (size_t)RED_THREADS * ctx->pitch * esz + RED_THREADS * sizeof(double);
  const char* se = getenv("EBC200_SHORT_STAGE");
  const bool staged = stage + smem <= 110 * 1024 && se && se[0] == '1';  // measured slower: opt-in
  const size_t dsm = smem + (staged ? stage : 0);
  auto go = [&](auto kern, const auto* V) -> int {
    CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
    kern<<<grid, SHORT_THREADS, dsm, ctx->stream>>>(V, ctx->pitch, ctx->n, ctx->d, ctx->cm64, wcount, wlist,
                                                    ctx->nchunks, ng, (double*)ctx->rterms.p,
                                                    (double*)ctx->part_r.p, pr, fin, sb);
    return EBC_OK;
  };
  if (ctx->dtype == EBC_F64)
    rc = staged ? go(k_refine_short<double, true>, ctx->V64) : go(k_refine_short<double, false>, ctx->V64);
  else
    rc = staged ? go(k_refine_short<float, true>, ctx->V32) : go(k_refine_short<float, false>, ctx->V32);
  if (rc) return rc;
  KCHECK();
  return EBC_OK;
}

// Conditional graph nodes (captured runs): a handle of the graph ctx->stream is
// capturing into (0 outside capture), and a scope that inserts an IF node with
// it and captures the body on a side stream until the scope closes.
// A Greedy run is a deterministic function of (V, e0, k): a lazy step the
// eager run decided with its first batch is decided in every replay, so the
// captured graph holds no conditional node for it (the node costs ~8 us of
// scheduling per step even when skipped); greedy_run checks the replay's count
// of decided steps against the eager run's and fails loudly on a difference.
bool captured_decided(const ebc_ctx* ctx, int step) {
  return ctx->capturing && ctx->cap_dec && step >= 0 && (size_t)step < ctx->cap_dec->size() && (*ctx->cap_dec)[step];
}

cudaGraphConditionalHandle cond_handle(ebc_ctx* ctx) {
  if (!ctx->capturing || !ctx->use_cond) return 0;
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  cudaGraph_t g = nullptr;
  if (cudaStreamGetCaptureInfo(ctx->stream, &st, nullptr, &g, nullptr, nullptr) != cudaSuccess ||
      st != cudaStreamCaptureStatusActive)
    return 0;
  cudaGraphConditionalHandle h = 0;
  if (cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault) != cudaSuccess) return 0;
  return h;
}

struct CondScope {
  ebc_ctx* ctx = nullptr;
  cudaStream_t saved = nullptr;
  ~CondScope() { close(); }
  cudaError_t open(ebc_ctx* c, cudaGraphConditionalHandle h, int depth) {
    if (!h) return cudaSuccess;
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    cudaGraph_t g = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    cudaError_t e = cudaStreamGetCaptureInfo(c->stream, &st, nullptr, &g, &deps, &nd);
    if (e != cudaSuccess) return e;
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeIf;
    cp.conditional.size = 1;
    cudaGraphNode_t cn = nullptr;
    if ((e = cudaGraphAddNode(&cn, g, deps, nd, &cp)) != cudaSuccess) return e;
    if ((e = cudaStreamUpdateCaptureDependencies(c->stream, &cn, 1, cudaStreamSetCaptureDependencies)) != cudaSuccess)
      return e;
    if ((e = cudaStreamBeginCaptureToGraph(c->side[depth], cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                           cudaStreamCaptureModeThreadLocal)) != cudaSuccess)
      return e;
    ctx = c;
    saved = c->stream;
    c->stream = c->side[depth];
    return cudaSuccess;
  }
  cudaError_t close() {
    if (!ctx) return cudaSuccess;
    cudaGraph_t body = nullptr;
    const cudaError_t e = cudaStreamEndCapture(ctx->stream, &body);
    ctx->stream = saved;
    ctx = nullptr;
    return e;
  }
};

RefineFinal step_final(ebc_ctx* ctx, int commit, int step, int64_t* sel_dev) {
  RefineFinal f;
  f.counter = ctx->counter3;
  f.wgain = ctx->wgain;
  f.inv_n = 1.0 / (double)ctx->n;
  f.cur = ctx->cur;
  f.best = ctx->best;
  f.commit = commit;
  f.step = step;
  f.selected = ctx->selected;
  f.sel_out = sel_dev;
  f.stats = ctx->stats;
  f.level = ctx->level;
  f.ubp = ctx->lazy_on ? ctx->ubp : nullptr;
  f.c0 = ctx->c0;
  return f;
}

double lazy_margin(const ebc_ctx* ctx) {
  return (double)ctx->n * 1e-12 * std::max(1.0, std::fabs(ctx->baseline)) * 1.01;
}

// Point-chunk groups per window candidate: as many as 256 MB of partials allow
// (a short window is latency-bound: more groups = more blocks in flight).
int refine_groups(const ebc_ctx* ctx) {
  const int64_t ng_mem = (int64_t)(256ull << 20) / (8 * (ctx->n + RW));
  return (int)std::max<int64_t>(1, std::min<int64_t>(ctx->nchunks, std::max<int64_t>(32, ng_mem)));
}

// The first batch of lazy step `step`: k_lazy_topk (its wlist / ub_next) and
// the RefineFinal of its refine, which decides the step; the caller launches
// that refine (k_refine_short / k_refine, or k_update_batch with the previous
// step's update).  Device-sharded runs all-reduce the batch's bound before the
// decision (batch 2), so every rank's stale set is its share of the
// single-device one (a rank whose own candidates are all weak would otherwise
// re-screen them against its own low bound).
void lazy_batch_begin(ebc_ctx* ctx, int step, int commit, int64_t* sel_dev, RefineFinal& fb,
                      const PackArgs& pa = PackArgs()) {
  const int64_t ncand = ctx->c1 - ctx->c0;
  const int64_t tpb = ctx->topk_cpb;  // candidates per top-k block (EBC200_TOPK_CPB)
  const int ag = (int)std::max<int64_t>(1, std::min<int64_t>(2 * ctx->num_sms, (ncand + tpb - 1) / tpb));
  k_lazy_topk<<<ag, 256, 0, ctx->stream>>>(ctx->c0, ctx->c1, ctx->ubp, ctx->selected, ctx->lazy_batch,
                                          (unsigned long long*)ctx->lazy_part, ctx->counter2, ctx->wcount, ctx->wlist,
                                          ctx->ub_next, pa, ctx->best, step);
  ++ctx->launches;
  const bool global_lb = ctx->in_sharded_run && ctx->comm && (ctx->nranks > 1 || ctx->force_global_lb);
  fb = step_final(ctx, commit, step, sel_dev);
  fb.batch = global_lb ? 2 : 1;
  fb.ub_next = ctx->ub_next;
  fb.margin = lazy_margin(ctx);
  fb.maxlb = ctx->maxlb;
  fb.scount = ctx->scount;
  fb.hrest = captured_decided(ctx, step) ? 0 : cond_handle(ctx);
}

// One step's selection: screen + certified window + exact refine + pick, or a
// lazy step (DESIGN.md §4 "Lazy steps"): the lazy_batch best stale bounds are
// refined first and decide the step when they hold the whole stale set;
// otherwise (a conditional graph node in captured runs, kernels gated on
// level[0] in eager runs) the stale set is listed and either refined directly
// or its blocks re-screened.  commit: single-device mode (mark the winner,
// record it as step `step`).
int run_step_select(ebc_ctx* ctx, int step, int commit, int64_t* sel_dev) {
  const int eb = 4 * step;  // event slot of this step
  const int64_t ncand = ctx->c1 - ctx->c0;
  const int fin_blocks = (int)((ncand + 255) / 256);
  ctx->cmx_fresh = false;
  ScreenPlan sp;
  const bool has_screen = ctx->dtype != EBC_F64 && plan_screen(ctx, sp) == EBC_OK;
  const bool lazy = ctx->lazy_on && ctx->ubp_seeded;
  if (!lazy) CU(cudaMemsetAsync(ctx->wcount, 0, sizeof(int), ctx->stream));  // a lazy step's k_lazy_topk writes it
  const int ng = refine_groups(ctx);
  int rc = ensure(ctx, ctx->part_r, (size_t)(ctx->n + RW) * ng * sizeof(double));
  if (rc) return rc;
  RefineFinal fin = step_final(ctx, commit, step, sel_dev);
  if (!lazy) {
    rc = has_screen ? run_screen_window(ctx, eb, fin_blocks) : run_window_all(ctx, eb, fin_blocks);
    if (rc) return rc;
    if (ctx->lazy_on) ctx->ubp_seeded = true;
    if (ctx->cmx_fresh) ctx->cmx_valid = true;
    rc = enqueue_refine(ctx, ng, nullptr, fin);
    if (rc) return rc;
    if (ctx->timing) CU(record_step_event(ctx, ctx->ev[eb + 2]));
    return EBC_OK;
  }
  // lazy step: the first batch (k_lazy_topk) and its refine, which decides
  // (it also sets maxlb = lb and zeroes scount; no memset nodes on this path).
  // Fused runs launched both with the previous step's update (k_update_batch).
  const int ag = (int)std::max<int64_t>(1, std::min<int64_t>(2 * ctx->num_sms, (ncand + 1023) / 1024));
  const double margin = lazy_margin(ctx);
  const bool global_lb = ctx->in_sharded_run && ctx->comm && (ctx->nranks > 1 || ctx->force_global_lb);
  cudaGraphConditionalHandle hrest = 0;
  if (ctx->batch_ready_step == step) {
    hrest = ctx->batch_hrest;
    ctx->batch_ready_step = -1;
  } else {
    RefineFinal fb;
    lazy_batch_begin(ctx, step, commit, sel_dev, fb);
    hrest = fb.hrest;
    ctx->cmx_fresh = ctx->cmx_valid;  // an earlier step's tile maxima still bound cm (it only decreases)
    rc = ctx->refine2 ? enqueue_refine_short(ctx, ng, fb) : enqueue_refine(ctx, ng, nullptr, fb);
    if (rc) return rc;
  }
  if (global_lb) {
    const NcclApi& api = nccl_api();
    const ncclResult_t r = api.AllReduce(ctx->maxlb, ctx->maxlb, 1, ncclInt64, ncclMax, ctx->comm, ctx->stream);
    if (r != ncclSuccess) return fail(ctx, EBC_ECOMM, std::string("ncclAllReduce: ") + api.GetErrorString(r));
    k_lazy_decide<<<1, 32, 0, ctx->stream>>>(ctx->maxlb, ctx->ub_next, margin, ctx->level, ctx->stats, hrest);
    KCHECK();
  }
  ctx->cmx_fresh = false;
  const bool sync = !ctx->capturing && ctx->eager_sync;
  auto read_mode = [&]() -> int {
    if (cudaMemcpyAsync(ctx->mode_host, ctx->level, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess)
      return -4;
    return *ctx->mode_host;
  };
  int mode = sync ? read_mode() : -3;
  if (mode == -4) return fail(ctx, EBC_ECUDA, "lazy step: mode read-back failed");
  if (sync && ctx->rec_dec && (size_t)step < ctx->rec_dec->size()) (*ctx->rec_dec)[step] = mode == -2;
  if (captured_decided(ctx, step)) mode = -2;
  if (mode != -2) {
    // undecided step (level[0] == -3): stale set -> mode -> screen / refine
    CondScope ca;
    CU(ca.open(ctx, hrest, 0));
    // probe batch and near-centre bound: only where a stale set can be large
    // enough to matter (small grounds' undecided steps go to the exact refine
    // anyway; the extra launches would only add latency, C1 0.68 -> 0.90 ms)
    const bool big = ncand >= ctx->probe_min_n;
    if (big && ctx->probe_on && has_screen && ctx->refine2 && short_refine_smem(ctx) <= 180 * 1024) {
      // probe batch: ring winners around the last selected centre raise lb
      // (k_lazy_rings) before the stale set is listed
      k_lazy_rings<<<ag, 256, (size_t)ctx->d * sizeof(float), ctx->stream>>>(
          ctx->c0, ctx->c1, ctx->V32, ctx->pitch, ctx->d, ctx->best, ctx->ubp, ctx->selected, ctx->level, ctx->probe,
          RW);
      KCHECK();
      RefineFinal fp = fin;
      fp.batch = 3;
      fp.commit = 0;
      fp.maxlb = ctx->maxlb;
      ctx->cmx_fresh = ctx->cmx_valid;
      rc = enqueue_refine_short(ctx, ng, fp, ctx->probe.pcount, ctx->probe.plist);
      ctx->cmx_fresh = false;
      if (rc) return rc;
    }
    if (big && ctx->nb_on && has_screen) {
      // near-centre bound: the neighbours of the centre just selected leave the
      // stale set without a screen (k_lazy_nearbound)
      const bool regs = ctx->d <= 32;
      const size_t nsm = ((size_t)ctx->geo.dp * (NB_TILE + 1) + (regs ? 0 : (size_t)ctx->d * NB_CPB)) * sizeof(float);
      auto kern = regs ? k_lazy_nearbound<32> : k_lazy_nearbound<0>;
      CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)nsm));
      kern<<<(unsigned)((ncand + NB_CPB - 1) / NB_CPB), 256, nsm, ctx->stream>>>(
          ctx->c0, ctx->c1, ctx->V32, ctx->pitch, ctx->d, ctx->best, ctx->ubp, ctx->selected, ctx->maxlb, margin,
          ctx->level, ctx->geo, ctx->chunkpart, ctx->n);
      KCHECK();
    }
    CU(cudaMemsetAsync(ctx->bflag, 0, (size_t)((ncand + tc::M - 1) / tc::M + 2), ctx->stream));
    k_lazy_mark2<<<fin_blocks, 256, 0, ctx->stream>>>(ctx->c0, ctx->c1, ctx->ubp, ctx->selected, ctx->maxlb,
                                                      margin, ctx->bcnt, ctx->bflag, ctx->level);
    KCHECK();
    k_lazy_scan<<<1, 1024, 0, ctx->stream>>>(ctx->bcnt, fin_blocks, ctx->scount, ctx->level);
    KCHECK();
    k_lazy_write<<<fin_blocks, 256, 0, ctx->stream>>>(ctx->c0, ctx->c1, ctx->ubp, ctx->selected, ctx->maxlb,
                                                      margin, ctx->bcnt, ctx->slist, ctx->level);
    KCHECK();
    const cudaGraphConditionalHandle hs = has_screen ? cond_handle(ctx) : 0;
    const bool can_gather = has_screen && ctx->gather_on && ctx->ladder_max >= L_TC;
    const cudaGraphConditionalHandle hg = can_gather ? cond_handle(ctx) : 0;
    k_lazy_plan2<<<1, 256, 0, ctx->stream>>>(ctx->scount, ctx->slist, has_screen ? ctx->lazy_cap : INT_MAX,
                                             ctx->wcount, ctx->wlist, ctx->level, ctx->stats, hs, ctx->bflag,
                                             (int)((ncand + tc::M - 1) / tc::M),
                                             can_gather ? (int)ctx->gath_cap : 0, (int)L_TC, hg);
    KCHECK();
    if (sync) {
      mode = read_mode();
      if (mode == -4) return fail(ctx, EBC_ECUDA, "lazy step: mode read-back failed");
      if (getenv("EBC200_LAZY_TRACE")) {  // development aid: stale-set shape per eager lazy step
        int cnt = 0;
        cudaStreamSynchronize(ctx->stream);
        std::vector<unsigned char> fl((size_t)((ncand + tc::M - 1) / tc::M));
        cudaMemcpy(&cnt, ctx->scount, sizeof(int), cudaMemcpyDeviceToHost);
        cudaMemcpy(fl.data(), ctx->bflag, fl.size(), cudaMemcpyDeviceToHost);
        size_t nb = 0;
        for (unsigned char b : fl) nb += b != 0;
        fprintf(stderr, "[lazy] step %d mode %d stale %d blocks %zu of %zu\n", step, mode, cnt, nb, fl.size());
      }
    }
    if (can_gather && (mode == -3 || mode == L_GATHER)) {
      CondScope cg;
      CU(cg.open(ctx, hg, 1));
      rc = run_gathered_window(ctx, fin_blocks);
      if (rc) return rc;
      CU(cg.close());
    }
    if (has_screen && mode != -1 && mode != L_GATHER) {
      CondScope cb;
      CU(cb.open(ctx, hs, 1));
      ctx->step_bflag = ctx->bflag;
      ctx->screen_events_outside = true;
      rc = run_screen_window(ctx, eb, fin_blocks);
      ctx->step_bflag = nullptr;
      ctx->screen_events_outside = false;
      if (rc) return rc;
      CU(cb.close());
    }
    // the window's refine and pick (mode -1: the stale list; re-screened: the window)
    ctx->cmx_fresh = ctx->cmx_valid;
    rc = enqueue_refine(ctx, ng, ctx->level, fin);
    if (rc) return rc;
    if (sync && getenv("EBC200_LAZY_TRACE")) {
      long long st[2] = {0, 0};
      cudaStreamSynchronize(ctx->stream);
      cudaMemcpy(st, ctx->stats, sizeof(st), cudaMemcpyDeviceToHost);
      fprintf(stderr, "[lazy] step %d window sum %lld max %lld\n", step, st[0], st[1]);
    }
    CU(ca.close());
  }
  // lazy steps record only eb + 1 (here) and eb + 3 (after the update): greedy_run
  // reads [prev eb + 3, eb + 1] as the step's selection time
  if (ctx->timing) CU(record_step_event(ctx, ctx->ev[eb + 1]));
  return EBC_OK;
}

TcSeeds tc_seeds(const ebc_ctx* ctx) {
  TcSeeds s;
  if (ctx->pttc) {
    s.ipa = ctx->pttc;
    s.nva = ctx->nva;
    s.na = ctx->tc_na;
    s.stride = ctx->n_pad;
    if (ctx->tc_mseed) {
      s.ops = (__half*)(ctx->tc_fast ? ctx->Vf : ctx->Vhi);
      s.kpad = ctx->kpad;
      s.d = ctx->d;
      s.s2 = ctx->tc_fast ? ctx->tc_oscale * ctx->tc_oscale : 1.f;
    }
  }
  return s;
}

int run_update(ebc_ctx* ctx, int step, double* val_dev, double* gain_dev) {
  const int eb = 4 * step;
  const size_t smem = (size_t)ctx->d * sizeof(double);
  if (ctx->dtype == EBC_F64) {
    CU(cudaFuncSetAttribute(k_update<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem + 1024));
    k_update<double><<<ctx->nchunks, RED_THREADS, smem, ctx->stream>>>(
        ctx->V64, ctx->pitch, ctx->n, ctx->d, ctx->best, ctx->pk, ctx->e0d, ctx->nv32, ctx->cm64, ctx->pt, tc_seeds(ctx), ctx->chunkpart,
        ctx->counter, 1.0 / (double)ctx->n, ctx->cur, val_dev, gain_dev, step);
  } else if (ctx->uf_on) {
    // fused K4: one launch, one bulk-copied slice per block (EBC200_UPDATE_ROWS
    // rows, 256 by default; 64 and 128 measured the same on C2 and C4), f(S) by
    // the block that completes the last chunk
    // (DESIGN.md §4 K4)
    const size_t head = (((size_t)ctx->d * 8 + 15) & ~(size_t)15) + (((size_t)((ctx->d + 3) & ~3) * 4 + 15) & ~(size_t)15);
    const int rows = ctx->uf_rows;
    const size_t dsm = head + (size_t)rows * (ctx->pitch * 4 + 16);
    UpdateCounters uc{ctx->uf_ctr + 1, ctx->uf_ctr};
    const unsigned grid = (unsigned)((ctx->n + rows - 1) / rows);
    auto go = [&](auto kern) -> int {
      CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
      kern<<<grid, rows, dsm, ctx->stream>>>(ctx->V32, ctx->pitch, ctx->n, ctx->d, ctx->best, ctx->pk, ctx->e0d,
                                             ctx->nv32, ctx->cm64, ctx->pt, tc_seeds(ctx), ctx->terms,
                                             ctx->chunkpart, uc, 1.0 / (double)ctx->n, ctx->cur, val_dev, gain_dev,
                                             step);
      return EBC_OK;
    };
    const int grc = rows == 64 ? go(k_update_fused<64>) : (rows == 128 ? go(k_update_fused<128>)
                                                                      : go(k_update_fused<256>));
    if (grc) return grc;
  } else {
    // split K4: wide streaming pass over V (a), fixed-structure reduction (b)
    const int nb = (int)((ctx->n + RED_THREADS - 1) / RED_THREADS);
    const bool stage = ctx->pitch <= UPDATE_STAGE_PITCH;
    const size_t dsm = (size_t)((ctx->d + 1) & ~1) * sizeof(double) +
                       (stage ? (size_t)RED_THREADS * ctx->pitch * sizeof(float) : 0);
    if (stage) {
      CU(cudaFuncSetAttribute(k_update_terms<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
      k_update_terms<true><<<nb, RED_THREADS, dsm, ctx->stream>>>(ctx->V32, ctx->pitch, ctx->n, ctx->d, ctx->best,
                                                                  ctx->pk, ctx->e0d, ctx->nv32, ctx->cm64, ctx->pt,
                                                                  tc_seeds(ctx), ctx->terms);
    } else {
      CU(cudaFuncSetAttribute(k_update_terms<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm + 16));
      k_update_terms<false><<<nb, RED_THREADS, dsm, ctx->stream>>>(ctx->V32, ctx->pitch, ctx->n, ctx->d, ctx->best,
                                                                   ctx->pk, ctx->e0d, ctx->nv32, ctx->cm64, ctx->pt,
                                                                   tc_seeds(ctx), ctx->terms);
    }
    KCHECK();
    k_update_reduce<<<ctx->nchunks, RED_THREADS, 0, ctx->stream>>>(ctx->terms, ctx->n, ctx->chunkpart, ctx->counter,
                                                                   1.0 / (double)ctx->n, ctx->cur, val_dev, gain_dev,
                                                                   step, ctx->best);
  }
  KCHECK();
  if (ctx->timing) CU(record_step_event(ctx, ctx->ev[eb + 3]));
  return EBC_OK;
}

int ensure_events(ebc_ctx* ctx, size_t count) {
  while (ctx->ev.size() < count) {
    cudaEvent_t e;
    CU(cudaEventCreate(&e));
    ctx->ev.push_back(e);
  }
  return EBC_OK;
}

int do_reset(ebc_ctx* ctx);
int run_step_select(ebc_ctx* ctx, int step, int commit, int64_t* sel_dev);
int run_update(ebc_ctx* ctx, int step, double* val_dev, double* gain_dev);

// Dynamic shared memory of k_update_batch<rows> (0: does not fit one block).
size_t update_batch_smem(const ebc_ctx* ctx, int rows) {
  const size_t stage = std::max<size_t>((size_t)rows * ctx->pitch * 4 + (size_t)rows * 16,
                                        ((size_t)(RW + 1) * RED_THREADS + RW + 1) * sizeof(double));
  const size_t b = BatchPackLayout(ctx->d).bytes() + stage;
  return b <= 200 * 1024 ? b : 0;
}

// Single-device lazy runs fold the next step's first batch into this step's
// K4 (k_update_batch): fp32 rows on the fused K4 path, the short refine.
bool batch_fusable(const ebc_ctx* ctx) {
  return ctx->fuse_batch && ctx->lazy_on && ctx->refine2 && ctx->uf_on && ctx->dtype != EBC_F64 &&
         !ctx->in_sharded_run && short_refine_smem(ctx) <= 180 * 1024 && update_batch_smem(ctx, ctx->ub_rows) > 0 &&
         refine_groups(ctx) <= 256;
}

// K4 of `step` together with the first batch of lazy step step + 1: k_lazy_topk,
// then one pass over the rows (k_update_batch) -- the batch's refine and its
// decision are those of k_refine_short after k_update_fused, bit for bit.
int run_update_batch(ebc_ctx* ctx, int step, double* val_dev, double* gain_dev, int64_t* sel_dev) {
  const int eb = 4 * step;
  const size_t pbytes = BatchPackLayout(ctx->d).bytes();
  int rc = ensure(ctx, ctx->ubpack, pbytes);
  if (rc) return rc;
  // the batch's top-k also packs the rows k_update_batch stages (winner + batch)
  PackArgs pa;
  pa.V = ctx->V32;
  pa.pitch = ctx->pitch;
  pa.d = ctx->d;
  pa.nv32 = ctx->nv32;
  pa.pack = (unsigned char*)ctx->ubpack.p;
  RefineFinal fb;
  lazy_batch_begin(ctx, step + 1, 1, sel_dev, fb, pa);
  // the top-k picks the next step's batch: timed with the selection family,
  // so the update family is k_update_batch alone (re-recorded event)
  if (ctx->timing) CU(record_step_event(ctx, ctx->ev[eb + 2]));
  if ((rc = ensure(ctx, ctx->rterms, (size_t)RW * ctx->nchunks * sizeof(double)))) return rc;
  const size_t xbytes = (size_t)RW * ctx->n_pad * sizeof(double);
  const size_t sbytes = xbytes + (size_t)ctx->nchunks * sizeof(unsigned int);
  const bool fresh = ctx->sxt.bytes < sbytes;
  if ((rc = ensure(ctx, ctx->sxt, sbytes))) return rc;
  if (fresh) CU(cudaMemsetAsync((unsigned char*)ctx->sxt.p + xbytes, 0, sbytes - xbytes, ctx->stream));
  BatchArgs ba;
  ba.wcount = ctx->wcount;
  ba.wlist = ctx->wlist;
  ba.xch = (double*)ctx->rterms.p;
  ba.part_r = (double*)ctx->part_r.p;
  ba.ng = refine_groups(ctx);
  ba.sb.xt = (double*)ctx->sxt.p;
  ba.sb.xstride = ctx->n_pad;
  ba.fin = fb;
  const int rows = ctx->ub_rows;  // two threads per row: 128 or 256 threads
  const size_t dsm = update_batch_smem(ctx, rows);
  UpdateCounters uc{ctx->uf_ctr + 1, ctx->uf_ctr};
  const unsigned grid = (unsigned)((ctx->n + rows - 1) / rows);
  auto go = [&](auto kern) -> int {
    CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
    // a programmatic dependent of the top-k just launched (EBC200_PDL=0: plain launch)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(2 * rows);
    cfg.dynamicSmemBytes = dsm;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = ctx->pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CU(cudaLaunchKernelEx(&cfg, kern, (const float*)ctx->V32, ctx->pitch, (int64_t)ctx->n, ctx->d,
                          (const int64_t*)ctx->best, ctx->pk, (const double*)ctx->e0d, (const float*)ctx->nv32,
                          ctx->cm64, ctx->pt, tc_seeds(ctx), ctx->terms, ctx->chunkpart, uc, 1.0 / (double)ctx->n,
                          ctx->cur, val_dev, gain_dev, step, ba, (const unsigned char*)ctx->ubpack.p));
    return EBC_OK;
  };
  rc = rows == 64 ? go(k_update_batch<64>) : go(k_update_batch<128>);
  if (rc) return rc;
  KCHECK();
  ctx->batch_ready_step = step + 1;
  ctx->batch_hrest = fb.hrest;
  if (ctx->timing) CU(record_step_event(ctx, ctx->ev[eb + 3]));
  return EBC_OK;
}

// Reset + the k steps of a Greedy run, all on ctx->stream (no host sync).
// One sharded Greedy step entirely on the device: local screen + window +
// exact refine of this rank's candidates, its tie-set records, an NCCL
// all-gather of the fixed-size records, the identical global pick on every
// rank, and the cached-min update -- no host round trip (graph-capturable).
int enqueue_sharded_step(ebc_ctx* ctx, int s, const double2* gathered_host_fed) {
  if (ctx->c1 > ctx->c0) {
    int rc = run_step_select(ctx, s, 0, nullptr);
    if (rc) return rc;
  } else {
    CU(cudaMemsetAsync(ctx->wcount, 0, sizeof(int), ctx->stream));
    if (ctx->lazy_on && s > 0 && ctx->nranks > 1 && !gathered_host_fed) {
      // the other ranks' lazy steps all-reduce their batch bound: take part with 0
      CU(cudaMemsetAsync(ctx->maxlb, 0, sizeof(long long), ctx->stream));
      const NcclApi& api = nccl_api();
      const ncclResult_t r = api.AllReduce(ctx->maxlb, ctx->maxlb, 1, ncclInt64, ncclMax, ctx->comm, ctx->stream);
      if (r != ncclSuccess) return fail(ctx, EBC_ECOMM, std::string("ncclAllReduce: ") + api.GetErrorString(r));
    }
  }
  k_tie_records<<<1, 1024, 0, ctx->stream>>>(ctx->wcount, ctx->wlist, ctx->wgain, 1.0 / (double)ctx->n, ctx->cur,
                                             (double2*)ctx->tie_rec.p);
  KCHECK();
  if (!gathered_host_fed) {
    const NcclApi& api = nccl_api();
    const ncclResult_t r = api.AllGather(ctx->tie_rec.p, ctx->tie_all.p, (size_t)(TIE_CAP + 1) * 2, ncclFloat64,
                                         ctx->comm, ctx->stream);
    if (r != ncclSuccess) return fail(ctx, EBC_ECOMM, std::string("ncclAllGather: ") + api.GetErrorString(r));
  }
  k_pick_global<<<1, 1024, 0, ctx->stream>>>((const double2*)ctx->tie_all.p, ctx->nranks, 1.0 / (double)ctx->n,
                                             ctx->cur, ctx->best, ctx->selected, (int64_t*)ctx->sel_out.p, s,
                                             ctx->tie_err);
  KCHECK();
  return run_update(ctx, s, (double*)ctx->val_out.p, (double*)ctx->gain_out.p);
}

int enqueue_greedy_sharded(ebc_ctx* ctx, int k) {
  int rc = do_reset(ctx);
  if (rc) return rc;
  CU(cudaMemsetAsync(ctx->tie_err, 0, sizeof(int), ctx->stream));
  ctx->in_sharded_run = true;
  for (int s = 0; s < k && !rc; ++s) rc = enqueue_sharded_step(ctx, s, nullptr);
  ctx->in_sharded_run = false;
  if (rc) return rc;
  // consistency guard: every rank must hold the same selection, values and
  // gains; a disagreement (err bit 2) fails the call instead of returning
  // rank-dependent results
  unsigned long long* h = (unsigned long long*)ctx->sel_hash.p;
  k_sel_hash<<<1, 32, 0, ctx->stream>>>((const int64_t*)ctx->sel_out.p, (const double*)ctx->val_out.p,
                                        (const double*)ctx->gain_out.p, k, h);
  KCHECK();
  const NcclApi& api = nccl_api();
  const ncclResult_t r = api.AllGather(h, h + 1, 1, ncclUint64, ctx->comm, ctx->stream);
  if (r != ncclSuccess) return fail(ctx, EBC_ECOMM, std::string("ncclAllGather: ") + api.GetErrorString(r));
  k_sel_hash_check<<<1, 32, 0, ctx->stream>>>(h + 1, ctx->nranks, ctx->tie_err);
  KCHECK();
  return EBC_OK;
}

int enqueue_greedy(ebc_ctx* ctx, int k) {
  int rc = do_reset(ctx);
  if (rc) return rc;
  ctx->fused_step.assign((size_t)k, 0);
  for (int s = 0; s < k; ++s) {
    rc = run_step_select(ctx, s, 1, (int64_t*)ctx->sel_out.p);
    if (rc) return rc;
    if (s + 1 < k && ctx->ubp_seeded && batch_fusable(ctx)) {
      ctx->fused_step[s] = 1;
      rc = run_update_batch(ctx, s, (double*)ctx->val_out.p, (double*)ctx->gain_out.p, (int64_t*)ctx->sel_out.p);
    } else
      rc = run_update(ctx, s, (double*)ctx->val_out.p, (double*)ctx->gain_out.p);
    if (rc) return rc;
  }
  return EBC_OK;
}

int do_reset(ebc_ctx* ctx) {
  ctx->batch_ready_step = -1;
  const int blocks = (int)((ctx->n + 255) / 256);
  CU(cudaMemsetAsync(ctx->stats, 0, 8 * sizeof(long long), ctx->stream));
  k_reset<<<blocks, 256, 0, ctx->stream>>>(ctx->n, ctx->e0d, ctx->nv32, ctx->pk, ctx->cm64, ctx->pt, ctx->selected,
                                           nullptr, tc_seeds(ctx));
  KCHECK();
  {
    // first rung of the adaptive ladder for this run
    const int start = (ctx->screen_mode == 3 && ctx->tc_np) ? (ctx->tc_fast ? L_FAST : L_TC) : L_GRAM;
    k_set_int<<<1, 1, 0, ctx->stream>>>(ctx->level, start);
    k_set_int<<<1, 1, 0, ctx->stream>>>(ctx->level + 1, start);
  }
  KCHECK();
  if (ctx->lazy_on) {
    k_fill_f64<<<(unsigned)std::min<int64_t>(4 * ctx->num_sms, (ctx->n + 255) / 256), 256, 0, ctx->stream>>>(
        ctx->ubp, ctx->n, INFINITY);
    KCHECK();
  }
  ctx->ubp_seeded = false;
  ctx->cmx_valid = false;
  CU(cudaMemsetAsync(ctx->cur, 0, sizeof(double), ctx->stream));
  ctx->steps_done = 0;
  return EBC_OK;
}

void free_ctx(ebc_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  void* ptrs[] = {c->V32, c->V64, c->e0d, c->cm64, c->pt, c->nv32, c->level, c->stats, c->Vhi, c->Vlo, c->Vf, c->tile_anchor0, c->rhomax, c->cmn, c->vsum, c->vsn, c->ipsum, c->rhomin, c->agg_any, c->pttc, c->kpmax, c->anchors, c->nva, c->tile_anchor, c->tc_vmax, c->fps_keys, c->ipa0, c->tile_rad, c->crad, c->rho, c->cmx, c->cmx0, c->selected, c->chunkpart, c->counter, c->counter2, c->topc, c->toppart, c->terms, c->cur, c->best, c->uf_ctr,
                  c->maxlb, c->wcount, c->wlist, c->wgain, c->ub, c->ubp, c->bflag, c->slist, c->scount,
                  c->lazy_part, c->ub_next, c->counter3, c->bcnt, c->Vg, c->g_anchor, c->g_rad, c->probe.rkey,
                  c->geo.mu, c->geo.r, c->geo.mn, c->geo.e0s, c->geo.muf};
  for (void* p : ptrs)
    if (p) cudaFreeAsync(p, c->stream);
  DevBuf* bufs[] = {&c->tie_rec, &c->tie_all, &c->sel_hash, &c->ms_tanchor, &c->ms_trad, &c->part_g, &c->part_e, &c->part_a, &c->part_r, &c->rterms, &c->sxt, &c->ubpack, &c->sv_cm, &c->sv_de, &c->sv_slots, &c->sv_part, &c->sv_out, &c->sel_out, &c->val_out, &c->gain_out, &c->ms_part,
                    &c->ms_off, &c->ms_idx, &c->ms_out, &c->ms_mbuf, &c->ms_setof, &c->ms_pairs, &c->ms_keys,
                    &c->ms_vals, &c->ms_keys2, &c->ms_vals2, &c->ms_ukeys, &c->ms_uvals, &c->ms_cub};
  void* more[] = {c->pt0, c->ms_count, c->ms_nruns};
  for (void* p : more)
    if (p) cudaFreeAsync(p, c->stream);
  for (DevBuf* b : bufs)
    if (b->p) cudaFreeAsync(b->p, c->stream);
  for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
  for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);
  if (c->tie_err) cudaFreeAsync(c->tie_err, c->stream);
  if (c->stream) {
    cudaStreamSynchronize(c->stream);
    cudaStreamDestroy(c->stream);
  }
  for (cudaStream_t ss : c->side)
    if (ss) cudaStreamDestroy(ss);
  if (c->mode_host && !pinned_words().give(c->mode_host)) cudaFreeHost(c->mode_host);
  if (c->sv_slots_host) cudaFreeHost(c->sv_slots_host);
  if (c->sv_out_host) cudaFreeHost(c->sv_out_host);
  delete c;
}

// Sparse work-matrix path (multiset.cuh).  Offsets/idx are already on the
// device (ms_off / ms_idx).  Returns EBC_EINVAL (results not written) when the
// flagged-pair buffer overflows -- the caller then runs the dense kernel.
int multiset_sparse(ebc_ctx* ctx, int64_t l, int64_t nnz) {
  const int64_t mrows = ((nnz + 127) / 128) * 128 + 128;
  int rc = ensure(ctx, ctx->ms_mbuf, (size_t)mrows * ctx->pitch * sizeof(float));
  if (!rc) rc = ensure(ctx, ctx->ms_setof, (size_t)mrows * sizeof(int));
  if (rc) return rc;
  if (!ctx->pt0) {
    CU(cudaMallocAsync((void**)&ctx->pt0, (size_t)ctx->n_pad * sizeof(float4), ctx->stream));
    CU(cudaMemsetAsync(ctx->pt0, 0, (size_t)ctx->n_pad * sizeof(float4), ctx->stream));
    CU(cudaMallocAsync((void**)&ctx->ms_count, sizeof(int), ctx->stream));
    CU(cudaMallocAsync((void**)&ctx->ms_nruns, sizeof(int), ctx->stream));
    k_make_pt0<<<(unsigned)((ctx->n + 255) / 256), 256, 0, ctx->stream>>>(ctx->n, ctx->e0d, ctx->nv32, ctx->pk,
                                                                          ctx->pt0);
    KCHECK();
  }
  CU(cudaMemsetAsync(ctx->ms_mbuf.p, 0, (size_t)mrows * ctx->pitch * sizeof(float), ctx->stream));
  k_gather_members<<<8 * ctx->num_sms, 256, 0, ctx->stream>>>(ctx->V32, ctx->pitch, (const int64_t*)ctx->ms_idx.p,
                                                              (const int64_t*)ctx->ms_off.p, l, nnz,
                                                              (float*)ctx->ms_mbuf.p, (int*)ctx->ms_setof.p);
  KCHECK();
  // flag screen: candidates = member rows, seed = d(., e0)
  const int cap = 16 << 20;
  rc = ensure(ctx, ctx->ms_pairs, (size_t)cap * sizeof(uint2));
  if (rc) return rc;
  CU(cudaMemsetAsync(ctx->ms_count, 0, sizeof(int), ctx->stream));
  const int64_t sc0 = ctx->c0, sc1 = ctx->c1;
  ctx->c0 = 0;
  ctx->c1 = nnz;
  FlagOut fo{(uint2*)ctx->ms_pairs.p, ctx->ms_count, cap, ctx->n, nnz};
  TcPlan tp{};
  if (ctx->ms_mode == 1 && ctx->screen_mode == 3 && plan_tc(ctx, tp, ctx->tc_kind)) {
    // tensor-core flag screen: anchors of the member blocks, reset-state seeds
    rc = ensure(ctx, ctx->ms_tanchor, (size_t)(mrows / 128 + 1) * sizeof(int));
    if (!rc) rc = ensure(ctx, ctx->ms_trad, (size_t)(mrows / 128 + 1) * sizeof(float));
    if (!rc && !ctx->ipa0) {
      CU(cudaMallocAsync((void**)&ctx->ipa0, (size_t)ctx->tc_na * ctx->n_pad * sizeof(float), ctx->stream));
      TcSeeds s0 = tc_seeds(ctx);
      s0.ipa = ctx->ipa0;
      s0.ops = nullptr;  // reset-state seeds only; the operand's folded seeds track the run
      k_seed_ipa<<<(unsigned)((ctx->n_pad + 255) / 256), 256, 0, ctx->stream>>>(ctx->e0d, ctx->n, ctx->n_pad, s0);
      KCHECK();
    }
    if (!rc) {
      k_tile_anchor<<<(unsigned)((nnz + 127) / 128), 128, tile_anchor_smem(ctx), ctx->stream>>>(
          (const float*)ctx->ms_mbuf.p, ctx->pitch, nnz, ctx->d, ctx->anchors, ctx->pitch, ctx->tc_na,
          (int*)ctx->ms_tanchor.p, (float*)ctx->ms_trad.p, tile_anchor_smem(ctx) > 0);
      KCHECK();
      rc = launch_tc_flag(ctx, tp, (const float*)ctx->ms_mbuf.p, (const int*)ctx->ms_tanchor.p,
                          (const float*)ctx->ms_trad.p, fo);
    }
  } else {
    ScreenPlan p;
    rc = plan_screen(ctx, p);
    if (!rc) rc = launch_screen<2>(ctx, p, nullptr, 0, (const float*)ctx->ms_mbuf.p, fo, ctx->pt0);
  }
  ctx->c0 = sc0;
  ctx->c1 = sc1;
  if (rc) return rc;
  int cnt = 0;
  CU(cudaMemcpyAsync(&cnt, ctx->ms_count, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  if (cnt > cap) return EBC_EINVAL;  // dense fallback
  const int64_t items = std::max(cnt, 1);
  rc = ensure(ctx, ctx->ms_keys, (size_t)items * 8);
  if (!rc) rc = ensure(ctx, ctx->ms_vals, (size_t)items * 8);
  if (!rc) rc = ensure(ctx, ctx->ms_keys2, (size_t)items * 8);
  if (!rc) rc = ensure(ctx, ctx->ms_vals2, (size_t)items * 8);
  if (!rc) rc = ensure(ctx, ctx->ms_ukeys, (size_t)items * 8);
  if (!rc) rc = ensure(ctx, ctx->ms_uvals, (size_t)items * 8);
  if (rc) return rc;
  unsigned long long* keys = (unsigned long long*)ctx->ms_keys.p;
  double* vals = (double*)ctx->ms_vals.p;
  if (cnt > 0) {
    k_flag_exact<float><<<4 * ctx->num_sms, 256, 0, ctx->stream>>>(
        (const uint2*)ctx->ms_pairs.p, ctx->ms_count, cap, ctx->V32, ctx->pitch, ctx->d,
        (const int64_t*)ctx->ms_idx.p, (const int*)ctx->ms_setof.p, ctx->e0d, ctx->n, keys, vals);
    KCHECK();
  }
  // sort by (set, point) and take the max term per key
  const int end_bit = 64;  // key = set * n + point; ~0 marks a non-contributing pair
  size_t tb1 = 0, tb2 = 0;
  CU(cub::DeviceRadixSort::SortPairs(nullptr, tb1, keys, (unsigned long long*)ctx->ms_keys2.p, vals,
                                     (double*)ctx->ms_vals2.p, (int)items, 0, end_bit, ctx->stream));
  CU(cub::DeviceReduce::ReduceByKey(nullptr, tb2, (unsigned long long*)ctx->ms_keys2.p,
                                    (unsigned long long*)ctx->ms_ukeys.p, (double*)ctx->ms_vals2.p,
                                    (double*)ctx->ms_uvals.p, ctx->ms_nruns, DMax(), (int)items, ctx->stream));
  rc = ensure(ctx, ctx->ms_cub, std::max(tb1, tb2) + 256);
  if (rc) return rc;
  size_t tb = ctx->ms_cub.bytes;
  if (cnt > 0) {
    CU(cub::DeviceRadixSort::SortPairs(ctx->ms_cub.p, tb, keys, (unsigned long long*)ctx->ms_keys2.p, vals,
                                       (double*)ctx->ms_vals2.p, cnt, 0, end_bit, ctx->stream));
    ++ctx->launches;
    tb = ctx->ms_cub.bytes;
    CU(cub::DeviceReduce::ReduceByKey(ctx->ms_cub.p, tb, (unsigned long long*)ctx->ms_keys2.p,
                                      (unsigned long long*)ctx->ms_ukeys.p, (double*)ctx->ms_vals2.p,
                                      (double*)ctx->ms_uvals.p, ctx->ms_nruns, DMax(), cnt, ctx->stream));
    ++ctx->launches;
  } else {
    CU(cudaMemsetAsync(ctx->ms_nruns, 0, sizeof(int), ctx->stream));
  }
  k_sparse_set_sum<<<(unsigned)((l * 32 + 255) / 256), 256, 0, ctx->stream>>>(
      (const unsigned long long*)ctx->ms_ukeys.p, (const double*)ctx->ms_uvals.p, ctx->ms_nruns, ctx->n, l,
      1.0 / (double)ctx->n, (double*)ctx->ms_out.p);
  KCHECK();
  return EBC_OK;
}

}  // namespace

// ============================================================================ C-ABI

extern "C" {

const char* ebc_version(void) { return "ebc200 0.1.0 sm_100a"; }

int ebc_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

const char* ebc_last_error(const ebc_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

int ebc_create(const void* V, int64_t n, int32_t d, int32_t dtype, const double* e0, int32_t device,
               ebc_ctx** out) {
  ebc_ctx* ctx = nullptr;
  if (!out) return fail(nullptr, EBC_EINVAL, "ebc_create: out is NULL");
  *out = nullptr;
  if (!V || n < 1 || d < 1) return fail(nullptr, EBC_EINVAL, "ground data must be at least 1x1");
  if (dtype != EBC_F32 && dtype != EBC_F16 && dtype != EBC_F64)
    return fail(nullptr, EBC_EINVAL, "unknown dtype " + std::to_string(dtype));
  int ndev = 0;
  cudaError_t ce = cudaGetDeviceCount(&ndev);
  if (ce != cudaSuccess || ndev < 1)
    return fail(nullptr, EBC_ECUDA,
                std::string("no CUDA device available for the b200 backend: ") + cudaGetErrorString(ce));
  if (device < 0 || device >= ndev)
    return fail(nullptr, EBC_EINVAL, "device " + std::to_string(device) + " out of range");

  ctx = new ebc_ctx();
  ctx->device = device;
  ctx->n = n;
  ctx->d = d;
  ctx->dtype = dtype;
  ctx->pitch = pitch_for(d, dtype);
  ctx->d4 = (d + 3) / 4;
  ctx->nchunks = (int)((n + RCH - 1) / RCH);
  ctx->n_pad = ((n + 127) / 128) * 128 + 256;
  ctx->c0 = 0;
  ctx->c1 = n;
  // error quanta: direct tau = 2(d+8)u cm32; Gram
  // kp = (d+4)u/2 (cm32 + 2|v|^2), kc = 1.5 (d+4)u |c|^2 -- all slightly inflated
  {
    const double u = 5.960464477539063e-08;
    ctx->pk.tau_k = (float)(2.0 * (d + 8) * u * (1.0 + 1.0 / 512));
    ctx->pk.gram_k = (float)(0.5 * (d + 4) * u * (1.0 + 1.0 / 512));
    ctx->gram_kc = (float)(1.5 * (d + 4) * u * (1.0 + 1.0 / 512));
    ctx->wcap = (int)std::max<int64_t>(256, n / 64);
    // the anchored tensor rung keeps windows up to N/8: on near-tied clustered
    // data (C4's 50-regime stress case) no FFMA rung narrows them, and refining
    // even N/8 candidates exactly costs far less than an FFMA re-screen
    ctx->wcap_tc = (int)std::max<int64_t>(256, n / 8);
    {
      const char* wc = getenv("EBC200_WCAP_TC");
      if (wc && wc[0]) ctx->wcap_tc = std::max(1, atoi(wc));
    }
    ctx->screen_mode = d >= 24 ? 3 : 0;
    const char* gg = getenv("EBC200_GRAPHS");
    if (gg && gg[0] == '0') ctx->use_graphs = false;
    const char* mm = getenv("EBC200_MULTISET_MODE");
    if (mm && mm[0]) ctx->ms_mode = atoi(mm);
    const char* m = getenv("EBC200_SCREEN_MODE");
    if (m && m[0]) ctx->screen_mode = atoi(m);
  }
  int rc = EBC_OK;
#define CUC(call)                                                                                   \
  do {                                                                                              \
    cudaError_t e_ = (call);                                                                        \
    if (e_ != cudaSuccess) {                                                                        \
      rc = fail(nullptr, EBC_ECUDA, std::string("CUDA error: ") + cudaGetErrorString(e_) + " (" #call ")"); \
      free_ctx(ctx);                                                                                \
      return rc;                                                                                    \
    }                                                                                               \
  } while (0)
  CUC(cudaSetDevice(device));
  // single attributes, not cudaGetDeviceProperties (which can cost tens of ms per call)
  int cc_major = 0, cc_minor = 0, sms = 0;
  CUC(cudaDeviceGetAttribute(&cc_major, cudaDevAttrComputeCapabilityMajor, device));
  CUC(cudaDeviceGetAttribute(&cc_minor, cudaDevAttrComputeCapabilityMinor, device));
  CUC(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  if (cc_major < 10)
    rc = fail(nullptr, EBC_ECUDA,
              "b200 backend needs an sm_100 device, found sm_" + std::to_string(cc_major * 10 + cc_minor));
  if (rc) {
    free_ctx(ctx);
    return rc;
  }
  ctx->num_sms = sms;
  {
    // every device buffer comes from the default stream-ordered pool, which
    // keeps freed memory (release threshold = max): building and destroying a
    // context per call (the e2e path) never goes back to the driver's mapper
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  CUC(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
  CUC(cudaStreamCreateWithFlags(&ctx->side[0], cudaStreamNonBlocking));
  CUC(cudaStreamCreateWithFlags(&ctx->side[1], cudaStreamNonBlocking));
  // EBC200_PROFILE_CREATE=1: host wall time of the creation phases on stderr
  const bool prof = getenv("EBC200_PROFILE_CREATE") != nullptr;
  auto tnow = []() { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  const double t_begin = tnow();
  auto mark = [&](const char* what) {
    if (prof) {
      cudaStreamSynchronize(ctx->stream);
      fprintf(stderr, "[ebc_create] %-22s %8.2f ms\n", what, tnow() - t_begin);
    }
  };
  const size_t esz = dtype == EBC_F64 ? sizeof(double) : sizeof(float);
  const size_t src_esz = dtype == EBC_F64 ? 8 : (dtype == EBC_F16 ? 2 : 4);
  void* Vdev = nullptr;
  CUC(cudaMallocAsync((void**)&Vdev, (size_t)ctx->n_pad * ctx->pitch * esz, ctx->stream));
  CUC(cudaMemsetAsync(Vdev, 0, (size_t)ctx->n_pad * ctx->pitch * esz, ctx->stream));
  if (dtype == EBC_F64)
    ctx->V64 = (double*)Vdev;
  else
    ctx->V32 = (float*)Vdev;
  void* raw = nullptr;
  CUC(cudaMallocAsync((void**)&raw, (size_t)n * d * src_esz, ctx->stream));
  mark("allocs V/raw");
  {
    const size_t bytes = (size_t)n * d * src_esz;
    const char* su = getenv("EBC200_STAGED_UPLOAD");
    // page-locked source (ebc_host_register): one direct DMA; pageable: staged
    cudaPointerAttributes pa{};
    const bool pinned = cudaPointerGetAttributes(&pa, V) == cudaSuccess && pa.type == cudaMemoryTypeHost;
    (void)cudaGetLastError();
    const bool staged = !pinned && bytes >= (16u << 20) && !(su && su[0] == '0') &&
                        staged_upload(ctx->stream, raw, V, bytes);
    if (!staged) CUC(cudaMemcpyAsync(raw, V, bytes, cudaMemcpyHostToDevice, ctx->stream));
  }
  mark("upload");
  {
    const int blocks = 8 * ctx->num_sms;
    if (dtype == EBC_F32)
      k_pad<float, float><<<blocks, 256, 0, ctx->stream>>>((const float*)raw, n, d, ctx->V32, ctx->pitch);
    else if (dtype == EBC_F16)
      k_pad<__half, float><<<blocks, 256, 0, ctx->stream>>>((const __half*)raw, n, d, ctx->V32, ctx->pitch);
    else
      k_pad<double, double><<<blocks, 256, 0, ctx->stream>>>((const double*)raw, n, d, ctx->V64, ctx->pitch);
    CUC(cudaGetLastError());
  }
  mark("pad");
  if (dtype != EBC_F64) {
    // fp32 range guard: every screen (and the sparse work-matrix flag screen)
    // forms squared distances, norms and short sums in fp32.  Grounds whose
    // distances could leave the fp32 range (|x| ~ 1e15 and beyond: the
    // reference's exact fp64 path still handles them) run without a screen --
    // every candidate goes to the exact fp64 refine (lazy steps keep that to
    // the stale ones) and work matrices to the dense fp64 kernel.
    unsigned int* amax = nullptr;
    CUC(cudaMallocAsync((void**)&amax, sizeof(unsigned int), ctx->stream));
    CUC(cudaMemsetAsync(amax, 0, sizeof(unsigned int), ctx->stream));
    k_absmax<<<4 * ctx->num_sms, 256, 0, ctx->stream>>>(ctx->V32, (int64_t)n * ctx->pitch, amax);
    CUC(cudaGetLastError());
    unsigned int bits = 0;
    CUC(cudaMemcpyAsync(&bits, amax, sizeof(unsigned int), cudaMemcpyDeviceToHost, ctx->stream));
    CUC(cudaStreamSynchronize(ctx->stream));
    cudaFreeAsync(amax, ctx->stream);
    float vmax = 0.f;
    std::memcpy(&vmax, &bits, sizeof(float));
    double emax = 0.0;
    if (e0)
      for (int k = 0; k < d; ++k) emax = std::max(emax, std::fabs(e0[k]));
    const double span = 2.0 * std::max((double)vmax, emax);
    // (and grounds whose every distance is below 1e-20: fp32 products of such
    // values underflow, which the screens' relative error bounds do not cover)
    const double far = span * span * (double)d;
    if (!(far < 1e30) || far < 1e-20) {
      ctx->fp32_ok = false;
      ctx->screen_mode = -1;
      ctx->ms_mode = 0;
    }
  }
  CUC(cudaMallocAsync((void**)&ctx->e0d, (size_t)ctx->n_pad * sizeof(double), ctx->stream));  // K4 stages whole slices
  CUC(cudaMallocAsync((void**)&ctx->cm64, (size_t)ctx->n_pad * sizeof(double), ctx->stream));
  CUC(cudaMallocAsync((void**)&ctx->pt, (size_t)ctx->n_pad * sizeof(float4), ctx->stream));
  CUC(cudaMemsetAsync(ctx->pt, 0, (size_t)ctx->n_pad * sizeof(float4), ctx->stream));
  CUC(cudaMallocAsync((void**)&ctx->nv32, (size_t)ctx->n_pad * sizeof(float), ctx->stream));
  CUC(cudaMemsetAsync(ctx->nv32, 0, (size_t)ctx->n_pad * sizeof(float), ctx->stream));
  // [4]: tensor-screen tile pairs executed; [5..7] lazy steps (k_lazy_plan2)
  CUC(cudaMallocAsync((void**)&ctx->stats, 8 * sizeof(long long), ctx->stream));
  CUC(cudaMemsetAsync(ctx->stats, 0, 8 * sizeof(long long), ctx->stream));
  CUC(cudaMallocAsync((void**)&ctx->level, 2 * sizeof(int), ctx->stream));
  CUC(cudaMemsetAsync(ctx->level, 0, 2 * sizeof(int), ctx->stream));
  mark("range guard");
  // tensor-core screen: fp32-path grounds whose 128-candidate tile of hi+lo
  // operands plus a 2-stage ring of NP-point tiles fits shared memory
  if (dtype != EBC_F64 && ctx->screen_mode == 3) {
    // FP16 grounds: one exact FP16 product; fp32 grounds: the BF16 split
    const char* kind = getenv("EBC200_TC_KIND");
    ctx->tc_kind = (kind && kind[0]) ? atoi(kind) : (dtype == EBC_F16 ? tc::KIND_F16 : tc::KIND_BF16);
    if (ctx->tc_kind == tc::KIND_F16 && dtype != EBC_F16) ctx->tc_kind = tc::KIND_BF16;  // fp32 values are not fp16
    if (ctx->tc_kind < 0 || ctx->tc_kind > 2) ctx->tc_kind = tc::KIND_BF16;
    const int es = tc_es(ctx->tc_kind), parts = tc_parts(ctx->tc_kind);
    ctx->kpad = es == 2 ? (d + 15) / 16 * 16 : (d + 7) / 8 * 8;
    int nps[2] = {128, 64};  // points per tile (64 only for wide TF32 operands)
    const char* npenv = getenv("EBC200_TC_NP");
    if (npenv && atoi(npenv) == 64) nps[0] = 64;
    for (int np : nps) {
      if (ctx->kpad <= 128 && tc::stages_for(ctx->kpad, np, es, parts) >= 2) {
        ctx->tc_np = np;
        break;
      }
    }
    if (ctx->tc_np) {
      const double u = 5.960464477539063e-08;
      // split error (dropped low-order products) + fp32 accumulation of parts*kpad
      // products (FP16: no split error, fp16 x fp16 products are exact)
      const double split = ctx->tc_kind == tc::KIND_F16    ? 0.0
                           : ctx->tc_kind == tc::KIND_BF16 ? 3.1 * std::ldexp(1.0, -18)
                                                           : 3.0 * std::ldexp(1.0, -20);
      const double nprod = ctx->tc_kind == tc::KIND_F16 ? 1.0 : 3.0;
      const double ktc = split + (nprod * ctx->kpad + 16.0) * std::ldexp(1.0, -23);
      // anchored bound: kp = (d+8)u (cm + |v - mu|^2),
      // kc = (d+8)u (|mu| |c'| + |c'|^2), kx = ktc + 4u per |v| |c'|
      ctx->tc_kp = (float)((d + 8) * u * 1.01);
      ctx->tc_kc = (float)((d + 8) * u * 1.01);
      ctx->tc_kx = (float)((ktc + 4.0 * u) * 1.01);
      // fast first rung: fp32 grounds whose BF16 split is MMA-bound
      // (3 kpad/16 K steps of 64 clk > the 1024-clk TMEM read of a 128-point tile)
      const char* fast_env = getenv("EBC200_TC_FAST");
      ctx->tc_fast = dtype == EBC_F32 && ctx->tc_kind == tc::KIND_BF16 &&
                     ((fast_env && fast_env[0]) ? atoi(fast_env) != 0 : ctx->kpad >= 96);
      if (ctx->tc_fast) {
        // operand rounding 2^-11 relative per operand -> (2^-10 + 2^-22) |v_k c'_k|;
        // one product per element accumulated in fp32
        const double kfast = std::ldexp(1.0, -10) + std::ldexp(1.0, -22) + (ctx->kpad + 16.0) * std::ldexp(1.0, -23);
        ctx->tc_kx_fast = (float)((kfast + 4.0 * u) * 1.01);
        ctx->wcap_fast = (int)std::max<int64_t>(256, n / 128);
      }
      // anchors: the origin plus farthest points (FP16 operands need c' = c exactly: origin only)
      const char* na_env = getenv("EBC200_TC_ANCHORS");
      ctx->tc_na = (na_env && na_env[0]) ? std::max(1, atoi(na_env)) : 32;
      if (ctx->tc_kind == tc::KIND_F16) ctx->tc_na = 1;
      ctx->tc_na = (int)std::min<int64_t>(ctx->tc_na, n);
      ctx->tc_ntl = ctx->n_pad / ctx->tc_np;
      const size_t ve = (size_t)ctx->n_pad * ctx->kpad;
      const size_t nas = (size_t)ctx->tc_na * ctx->n_pad;
      mark("tc plan");
      CUC(cudaMallocAsync((void**)&ctx->Vhi, ve * es, ctx->stream));
      if (parts == 2) CUC(cudaMallocAsync((void**)&ctx->Vlo, ve * es, ctx->stream));
      if (ctx->tc_fast) CUC(cudaMallocAsync((void**)&ctx->Vf, ve * 2, ctx->stream));
      CUC(cudaMallocAsync((void**)&ctx->pttc, nas * sizeof(float), ctx->stream));
      CUC(cudaMallocAsync((void**)&ctx->nva, nas * sizeof(float), ctx->stream));
      CUC(cudaMemsetAsync(ctx->nva, 0, nas * sizeof(float), ctx->stream));
      CUC(cudaMallocAsync((void**)&ctx->kpmax, (size_t)ctx->tc_na * ctx->tc_ntl * sizeof(float), ctx->stream));
      CUC(cudaMallocAsync((void**)&ctx->tc_vmax, (size_t)ctx->tc_ntl * sizeof(float), ctx->stream));
      CUC(cudaMallocAsync((void**)&ctx->anchors, (size_t)ctx->tc_na * ctx->pitch * sizeof(float), ctx->stream));
      CUC(cudaMallocAsync((void**)&ctx->tile_anchor, (size_t)(ctx->n_pad / 128 + 1) * sizeof(int), ctx->stream));
      CUC(cudaMemsetAsync(ctx->tile_anchor, 0, (size_t)(ctx->n_pad / 128 + 1) * sizeof(int), ctx->stream));
      CUC(cudaMallocAsync((void**)&ctx->fps_keys, (size_t)(ctx->tc_na + 1) * sizeof(unsigned long long), ctx->stream));
      const char* pr_env = getenv("EBC200_TC_PRUNE");
      ctx->tc_prune = !(pr_env && pr_env[0] == '0');
      CUC(cudaMallocAsync((void**)&ctx->tile_rad, (size_t)(ctx->n_pad / 128 + 1) * sizeof(float), ctx->stream));
      CUC(cudaMemsetAsync(ctx->tile_rad, 0, (size_t)(ctx->n_pad / 128 + 1) * sizeof(float), ctx->stream));
      CUC(cudaMallocAsync((void**)&ctx->rho, (size_t)ctx->tc_na * ctx->tc_ntl * sizeof(float), ctx->stream));
      {
        const char* ag_env = getenv("EBC200_TC_AGG");
        ctx->tc_agg = ctx->tc_prune && ctx->tc_kind != tc::KIND_F16 && ctx->tc_na > 1 && d <= 128 &&
                      !(ag_env && ag_env[0] == '0');
      }
      if (ctx->tc_agg) {
        CUC(cudaMallocAsync((void**)&ctx->rhomax, (size_t)ctx->tc_na * ctx->tc_ntl * sizeof(float), ctx->stream));
        CUC(cudaMallocAsync((void**)&ctx->cmn, (size_t)ctx->tc_ntl * sizeof(float), ctx->stream));
        CUC(cudaMallocAsync((void**)&ctx->vsum, ((size_t)ctx->tc_ntl * ctx->pitch + 32) * sizeof(float), ctx->stream));
        CUC(cudaMemsetAsync(ctx->vsum + (size_t)ctx->tc_ntl * ctx->pitch, 0, 32 * sizeof(float), ctx->stream));
        CUC(cudaMallocAsync((void**)&ctx->vsn, (size_t)ctx->tc_ntl * sizeof(float), ctx->stream));
        CUC(cudaMallocAsync((void**)&ctx->ipsum, (size_t)ctx->tc_na * ctx->tc_ntl * sizeof(double), ctx->stream));
        CUC(cudaMallocAsync((void**)&ctx->rhomin, (size_t)ctx->tc_ntl * sizeof(float), ctx->stream));
        CUC(cudaMallocAsync((void**)&ctx->agg_any, sizeof(int), ctx->stream));
      }
      CUC(cudaMallocAsync((void**)&ctx->cmx, (size_t)ctx->tc_ntl * sizeof(float), ctx->stream));
      CUC(cudaMallocAsync((void**)&ctx->cmx0, (size_t)ctx->tc_ntl * sizeof(float), ctx->stream));
      CUC(cudaMemsetAsync(ctx->fps_keys, 0, (size_t)(ctx->tc_na + 1) * sizeof(unsigned long long), ctx->stream));
    }
  }
  mark("tc allocs");
  CUC(cudaMallocAsync((void**)&ctx->selected, (size_t)ctx->n_pad, ctx->stream));
  CUC(cudaMemsetAsync(ctx->selected, 0, (size_t)ctx->n_pad, ctx->stream));
  CUC(cudaMallocAsync((void**)&ctx->chunkpart, (size_t)ctx->nchunks * sizeof(double), ctx->stream));
  CUC(cudaMallocAsync((void**)&ctx->counter, sizeof(unsigned int), ctx->stream));
  CUC(cudaMemsetAsync(ctx->counter, 0, sizeof(unsigned int), ctx->stream));
  CUC(cudaMallocAsync((void**)&ctx->counter2, sizeof(unsigned int), ctx->stream));
  CUC(cudaMemsetAsync(ctx->counter2, 0, sizeof(unsigned int), ctx->stream));
  CUC(cudaMallocAsync((void**)&ctx->topc, sizeof(int64_t), ctx->stream));
  CUC(cudaMallocAsync((void**)&ctx->toppart, (size_t)ctx->nchunks * 4 * sizeof(double), ctx->stream));
  CUC(cudaMallocAsync((void**)&ctx->terms, (size_t)ctx->n_pad * sizeof(double), ctx->stream));
  if (dtype != EBC_F64) {
    // fused K4 when a 256-row slice fits shared memory (pitch <= ~200 floats)
    const size_t dsm = (((size_t)d * 8 + 15) & ~(size_t)15) + (size_t)UF_ROWS * (ctx->pitch * 4 + 16);
    const char* uf_env = getenv("EBC200_UPDATE_FUSED");
    const char* ur_env = getenv("EBC200_UPDATE_ROWS");
    if (ur_env && (atoi(ur_env) == 128 || atoi(ur_env) == 256 || atoi(ur_env) == 64)) ctx->uf_rows = atoi(ur_env);
    if (dsm <= 220 * 1024 && !(uf_env && uf_env[0] == '0')) {
      ctx->uf_on = true;
      const size_t cb = (size_t)(1 + ctx->nchunks) * sizeof(unsigned int);
      CUC(cudaMallocAsync((void**)&ctx->uf_ctr, cb, ctx->stream));
      CUC(cudaMemsetAsync(ctx->uf_ctr, 0, cb, ctx->stream));
    }
  }
  mark("misc allocs");
  CUC(cudaMallocAsync((void**)&ctx->cur, sizeof(double), ctx->stream));
  CUC(cudaMemsetAsync(ctx->cur, 0, sizeof(double), ctx->stream));
  CUC(cudaMallocAsync((void**)&ctx->best, sizeof(int64_t), ctx->stream));
  CUC(cudaMallocAsync((void**)&ctx->maxlb, sizeof(long long), ctx->stream));
  CUC(cudaMallocAsync((void**)&ctx->wcount, sizeof(int), ctx->stream));
  CUC(cudaMallocAsync((void**)&ctx->wlist, (size_t)n * sizeof(int64_t), ctx->stream));
  CUC(cudaMallocAsync((void**)&ctx->wgain, (size_t)n * sizeof(double), ctx->stream));
  CUC(cudaMallocAsync((void**)&ctx->ub, (size_t)n * sizeof(double), ctx->stream));
  CUC(cudaMallocAsync((void**)&ctx->ubp, (size_t)n * sizeof(double), ctx->stream));
  CUC(cudaMallocAsync((void**)&ctx->bflag, (size_t)((n + tc::M - 1) / tc::M + 2), ctx->stream));
  CUC(cudaMallocAsync((void**)&ctx->slist, (size_t)n * sizeof(int64_t), ctx->stream));
  CUC(cudaMallocAsync((void**)&ctx->scount, sizeof(int), ctx->stream));
  CUC(cudaMallocAsync((void**)&ctx->bcnt, (size_t)((n + 255) / 256 + 1) * sizeof(int), ctx->stream));
  CUC(cudaMallocAsync(&ctx->lazy_part, (size_t)2 * ctx->num_sms * TK * sizeof(unsigned long long), ctx->stream));
  CUC(cudaMallocAsync((void**)&ctx->ub_next, sizeof(double), ctx->stream));
  CUC(cudaMallocAsync((void**)&ctx->counter3, sizeof(unsigned int), ctx->stream));
  CUC(cudaMemsetAsync(ctx->counter3, 0, sizeof(unsigned int), ctx->stream));
  {
    // ring keys | ticket | count | list (one allocation, zeroed once; k_lazy_rings re-zeroes)
    const size_t pbytes = NRING * 8 + 8 + 8 + RW * 8;
    unsigned char* pbm = nullptr;
    CUC(cudaMallocAsync((void**)&pbm, pbytes, ctx->stream));
    CUC(cudaMemsetAsync(pbm, 0, pbytes, ctx->stream));
    ctx->probe.rkey = (unsigned long long*)pbm;
    ctx->probe.counter = (unsigned int*)(pbm + NRING * 8);
    ctx->probe.pcount = (int*)(pbm + NRING * 8 + 8);
    ctx->probe.plist = (int64_t*)(pbm + NRING * 8 + 16);
    const char* pe = getenv("EBC200_LAZY_PROBE");
    if (pe && pe[0] == '0') ctx->probe_on = false;
    const char* pm = getenv("EBC200_PROBE_MIN_N");
    if (pm && pm[0]) ctx->probe_min_n = std::max(0, atoi(pm));
    const char* fz = getenv("EBC200_FUSE_BATCH");
    if (fz && fz[0] == '0') ctx->fuse_batch = false;
    const char* ur = getenv("EBC200_UB_ROWS");
    if (ur && ur[0]) {
      const int r = atoi(ur);
      ctx->ub_rows = r == 64 ? 64 : 128;
    }
    if (const char* pe = getenv("EBC200_PDL")) {
      ctx->pdl = atoi(pe) != 0;
    }
  }
  {
    // measured (bench.py, EBC200_LAZY_BATCH A/B): 4 on C2 (N = 100k: 3.17 ms
    // vs 3.27 with 3), 3 on C4 (N = 500k: 48.3 ms vs 52.0 with 4; fewer
    // candidates re-examined), C4S50 equal
    ctx->lazy_batch = ctx->n >= (int64_t)1 << 18 ? 3 : 4;
    const char* lb = getenv("EBC200_LAZY_BATCH");
    if (lb && lb[0]) ctx->lazy_batch = std::max(1, std::min(RW, atoi(lb)));
    const char* r2 = getenv("EBC200_REFINE2");
    if (r2 && r2[0] == '0') ctx->refine2 = false;
    const char* gl = getenv("EBC200_GLOBAL_LB");
    ctx->force_global_lb = gl && gl[0] == '1';
    const char* es = getenv("EBC200_EAGER_SYNC");
    if (es && es[0] == '0') ctx->eager_sync = false;
    ctx->mode_host = pinned_words().take();
    if (!ctx->mode_host) CUC(cudaMallocHost((void**)&ctx->mode_host, sizeof(int)));
    const char* gc = getenv("EBC200_GRAPH_COND");
    if (gc && gc[0] == '0') ctx->use_cond = false;
    const char* tc = getenv("EBC200_TOPK_CPB");
    if (tc && atoi(tc) >= 256) ctx->topk_cpb = atoi(tc);
    const char* sd = getenv("EBC200_SPEC_DECIDED");
    if (sd && sd[0] == '0') ctx->spec_dec = false;
  }
  {
    const char* lz = getenv("EBC200_LAZY");
    ctx->lazy_on = !(lz && lz[0] == '0');
    const char* lc = getenv("EBC200_LAZY_CAP");
    if (lc && lc[0]) ctx->lazy_cap = std::max(0, atoi(lc));
    const char* ge = getenv("EBC200_GATHER");
    ctx->gather_on = ctx->lazy_on && ctx->tc_np && ctx->screen_mode == 3 && !ctx->tc_fast &&
                     (ctx->tc_kind == tc::KIND_BF16 || ctx->tc_kind == tc::KIND_TF32) && !(ge && ge[0] == '0');
    if (ctx->gather_on) {
      // up to a quarter of the candidates (at least 64k): late steps of C4 with the
      // probe batch list ~100k scattered stale candidates over every block
      const int64_t gq = std::max<int64_t>(65536, (n / 4 + tc::M - 1) / tc::M * tc::M);
      ctx->gath_cap = std::min<int64_t>((n + tc::M - 1) / tc::M * tc::M, gq);
      const char* gc = getenv("EBC200_GATHER_CAP");
      if (gc && gc[0]) ctx->gath_cap = std::min<int64_t>(ctx->gath_cap, std::max(tc::M, atoi(gc) / tc::M * tc::M));
      CUC(cudaMallocAsync((void**)&ctx->Vg, (size_t)ctx->gath_cap * ctx->pitch * sizeof(float), ctx->stream));
      CUC(cudaMallocAsync((void**)&ctx->g_anchor, (size_t)(ctx->gath_cap / tc::M + 1) * sizeof(int), ctx->stream));
      CUC(cudaMallocAsync((void**)&ctx->g_rad, (size_t)(ctx->gath_cap / tc::M + 1) * sizeof(float), ctx->stream));
    }
  }
  double* e0dev = nullptr;
  CUC(cudaMallocAsync((void**)&e0dev, (size_t)d * sizeof(double), ctx->stream));
  {
    std::vector<double> z;
    const double* src = e0;
    if (!src) {
      z.assign(d, 0.0);
      src = z.data();
    }
    CUC(cudaMemcpyAsync(e0dev, src, (size_t)d * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CUC(cudaStreamSynchronize(ctx->stream));  // z / caller buffers may go away
  }
  if (dtype == EBC_F64)
    k_init<double><<<ctx->nchunks, RED_THREADS, 0, ctx->stream>>>(ctx->V64, ctx->pitch, n, d, e0dev, ctx->pk,
                                                                 ctx->e0d, ctx->cm64, ctx->nv32, ctx->pt, ctx->chunkpart);
  else
    mark("allocs rest"),
    k_init<float><<<ctx->nchunks, RED_THREADS, 0, ctx->stream>>>(ctx->V32, ctx->pitch, n, d, e0dev, ctx->pk,
                                                                ctx->e0d, ctx->cm64, ctx->nv32, ctx->pt, ctx->chunkpart);
  CUC(cudaGetLastError());
  mark("init");
  {
    const char* nb = getenv("EBC200_LAZY_NEARBOUND");
    ctx->nb_on = ctx->lazy_on && dtype != EBC_F64 && d <= 256 && !(nb && nb[0] == '0');
    if (ctx->nb_on) {
      ctx->geo.nchunks = (int)ctx->nchunks;
      CUC(cudaMallocAsync((void**)&ctx->geo.mu, (size_t)ctx->nchunks * d * sizeof(double), ctx->stream));
      CUC(cudaMallocAsync((void**)&ctx->geo.r, (size_t)ctx->nchunks * sizeof(double), ctx->stream));
      CUC(cudaMallocAsync((void**)&ctx->geo.mn, (size_t)ctx->nchunks * sizeof(double), ctx->stream));
      CUC(cudaMallocAsync((void**)&ctx->geo.e0s, (size_t)ctx->nchunks * sizeof(double), ctx->stream));
      ctx->geo.dp = (d + 3) / 4 * 4;
      CUC(cudaMallocAsync((void**)&ctx->geo.muf, (size_t)ctx->nchunks * ctx->geo.dp * sizeof(float), ctx->stream));
      k_chunk_geo<<<(unsigned)ctx->nchunks, 256, (size_t)d * sizeof(double), ctx->stream>>>(ctx->V32, ctx->pitch, n,
                                                                                          d, ctx->e0d, ctx->geo);
      CUC(cudaGetLastError());
    }
  }
  if (ctx->tc_np) {
    {
      // anchors (farthest-point sampling from the origin), |v - mu_a|^2, the
      // anchor of each candidate block, seeds and per-tile error quanta
      float* mind = nullptr;
      CUC(cudaMallocAsync((void**)&mind, (size_t)n * sizeof(float), ctx->stream));
      {
        // one cooperative launch (grid barrier per anchor); per-anchor launches
        // if the cooperative launch is refused -- the same anchors either way
        int per_sm = 0;
        const size_t fsm = (size_t)(d + 3) / 4 * 4 * sizeof(float);
        bool coop = fsm <= 48 * 1024 &&
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fps_all, 256, fsm) == cudaSuccess &&
                    per_sm > 0;
        unsigned int* bar = nullptr;
        if (coop) {
          CUC(cudaMallocAsync((void**)&bar, 2 * sizeof(unsigned int), ctx->stream));
          CUC(cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned int), ctx->stream));
          const float* v32 = ctx->V32;
          int pitch_ = ctx->pitch, d_ = d, na_ = ctx->tc_na, ap_ = ctx->pitch;
          int64_t n_ = n;
          void* args[] = {(void*)&v32, &pitch_, &n_, &d_, &na_, (void*)&mind, (void*)&ctx->fps_keys,
                          (void*)&ctx->anchors, &ap_, (void*)&bar};
          coop = cudaLaunchCooperativeKernel((const void*)k_fps_all, dim3(std::min(per_sm, 2) * ctx->num_sms),
                                             dim3(256), args, fsm, ctx->stream) == cudaSuccess;
          if (!coop) (void)cudaGetLastError();
          cudaFreeAsync(bar, ctx->stream);
        }
        if (!coop)
          for (int a = 0; a < ctx->tc_na; ++a) {
            k_fps_step<<<2 * ctx->num_sms, 256, 0, ctx->stream>>>(ctx->V32, ctx->pitch, n, d, a, ctx->tc_na, mind,
                                                                  ctx->fps_keys, ctx->anchors, ctx->pitch);
            CUC(cudaGetLastError());
          }
      }
      mark("fps anchors");
      const size_t nsm = (size_t)ctx->tc_na * ((d + 3) / 4 * 4) * sizeof(double);
      if (ctx->tc_na <= NA_ALL && nsm <= 160 * 1024) {
        CUC(cudaFuncSetAttribute(k_nva_all, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
        k_nva_all<<<(unsigned)((n + 127) / 128), 128, nsm, ctx->stream>>>(ctx->V32, ctx->pitch, n, d, ctx->anchors,
                                                                         ctx->pitch, ctx->tc_na, ctx->nva,
                                                                         ctx->n_pad);
      } else {
        k_nva<<<8 * ctx->num_sms, 256, 0, ctx->stream>>>(ctx->V32, ctx->pitch, n, d, ctx->anchors, ctx->pitch,
                                                         ctx->tc_na, ctx->nva, ctx->n_pad);
      }
      CUC(cudaGetLastError());
      CUC(cudaFuncSetAttribute(k_tile_anchor, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
      k_tile_anchor<<<(unsigned)((n + 127) / 128), 128, tile_anchor_smem(ctx), ctx->stream>>>(
          ctx->V32, ctx->pitch, n, d, ctx->anchors, ctx->pitch, ctx->tc_na, ctx->tile_anchor, ctx->tile_rad,
          tile_anchor_smem(ctx) > 0);
      CUC(cudaGetLastError());
      CUC(cudaMallocAsync((void**)&ctx->crad, (size_t)n * sizeof(float), ctx->stream));
      k_cand_rad<float><<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(ctx->V32, ctx->pitch, n, d,
                                                                             ctx->tile_anchor, ctx->anchors,
                                                                             ctx->pitch, ctx->crad);
      CUC(cudaGetLastError());
      k_seed_ipa<<<(unsigned)((ctx->n_pad + 255) / 256), 256, 0, ctx->stream>>>(ctx->cm64, n, ctx->n_pad,
                                                                                 tc_seeds(ctx));
      CUC(cudaGetLastError());
      const int64_t cells = (int64_t)ctx->tc_na * ctx->tc_ntl;
      k_tile_kpmax<<<(unsigned)((cells + 255) / 256), 256, 0, ctx->stream>>>(
          ctx->e0d, ctx->nv32, ctx->nva, ctx->n_pad, ctx->tc_na, n, ctx->tc_ntl, ctx->tc_np, ctx->tc_kp, ctx->kpmax,
          ctx->tc_vmax, ctx->rho, ctx->rhomax);
      CUC(cudaGetLastError());
      if (ctx->tc_agg) {
        k_tile_vsum<<<(unsigned)ctx->tc_ntl, 128, 0, ctx->stream>>>(ctx->V32, ctx->pitch, n, d, ctx->tc_np, ctx->vsum,
                                                                   ctx->vsn);
        CUC(cudaGetLastError());
        k_tile_rhomin<<<(unsigned)((ctx->tc_ntl + 255) / 256), 256, 0, ctx->stream>>>(ctx->rhomax, ctx->tc_na,
                                                                                       ctx->tc_ntl, ctx->rhomin);
      }
      CUC(cudaGetLastError());
      k_tile_cmmax<<<(unsigned)((ctx->tc_ntl * 32 + 255) / 256), 256, 0, ctx->stream>>>(ctx->e0d, n, ctx->tc_ntl,
                                                                                        ctx->tc_np, ctx->cmx0);
      CUC(cudaGetLastError());
      CUC(cudaStreamSynchronize(ctx->stream));
      mark("init + anchors");
      cudaFreeAsync(mind, ctx->stream);
      // the scalars below from one device pass (k_create_maxes) and one 32-byte copy
      double max_e0d = 0.0, max_nv = 0.0;
      float vmx = 0.f;
      {
        unsigned long long hm[4] = {0ull, 0ull, 0ull, 0x7f800000ull};
        unsigned long long* dm = nullptr;
        CUC(cudaMallocAsync((void**)&dm, sizeof(hm), ctx->stream));
        CUC(cudaMemcpyAsync(dm, hm, sizeof(hm), cudaMemcpyHostToDevice, ctx->stream));
        k_create_maxes<<<2 * ctx->num_sms, 256, 0, ctx->stream>>>(ctx->e0d, ctx->nv32, n, ctx->tc_vmax, ctx->tc_ntl,
                                                                 ctx->tile_rad, (n + 127) / 128, dm);
        CUC(cudaGetLastError());
        CUC(cudaMemcpyAsync(hm, dm, sizeof(hm), cudaMemcpyDeviceToHost, ctx->stream));
        CUC(cudaStreamSynchronize(ctx->stream));
        cudaFreeAsync(dm, ctx->stream);
        max_e0d = __builtin_bit_cast(double, hm[0]);
        max_nv = (double)__builtin_bit_cast(float, (unsigned int)hm[1]);
        vmx = __builtin_bit_cast(float, (unsigned int)hm[2]);
        // smallest candidate-block radius (k_tile_ipsum's any-block screen)
        if (ctx->tc_agg) ctx->radmin = __builtin_bit_cast(float, (unsigned int)hm[3]);
      }
      if (ctx->tc_fast) {
        // operand scale s = 2^e: every |s c'_k| <= s (|c| + |mu|) <= 2 s max|v| <= 2^15
        // (fp16 max 65504); |e| <= 60 keeps s^2 and 1/s^2 normal in fp32
        int e = vmx > 0.f ? (int)std::floor(std::log2(std::ldexp(1.0, 14) / (double)vmx)) : 0;
        e = std::max(-60, std::min(60, e));
        ctx->tc_oscale = (float)std::ldexp(1.0, e);
        ctx->tc_sinv2 = (float)std::ldexp(1.0, -2 * e);
        // subnormal half-spacing 2^-25 in scaled units: per element |err| <= 2^-11 |x| + eta
        const double eta = std::ldexp(1.0, -25 - e);
        ctx->tc_keta = (float)(eta * std::sqrt((double)d) * (1.0 + std::ldexp(1.0, -11)) * 1.02);
        ctx->tc_keta2 = (float)((double)d * eta * eta * 1.02 + 1e-38);
      }
      // seeds folded into the MMA: the one-product rung with three
      // spare K columns; scaled seeds |s^2 ip| <= s^2 (max e0d + max |v|^2)/2 <= 2^14
      const bool one_rung = ctx->tc_fast || ctx->tc_kind == tc::KIND_F16;
      const char* ms_env = getenv("EBC200_TC_MSEED");
      if (one_rung && ctx->kpad - d >= 3 && !(ms_env && ms_env[0] == '0')) {
        const double me = max_e0d, mv = max_nv;
        const double bip = 0.5 * (me + mv) * 1.01 + 1e-30;
        if (ctx->tc_fast) {
          const int e2 = (int)std::floor(0.5 * std::log2(std::ldexp(1.0, 14) / bip));
          const int e = std::max(-60, std::min(e2, (int)std::lround(std::log2((double)ctx->tc_oscale))));
          ctx->tc_oscale = (float)std::ldexp(1.0, e);
          ctx->tc_sinv2 = (float)std::ldexp(1.0, -2 * e);
          const double eta = std::ldexp(1.0, -25 - e);
          ctx->tc_keta = (float)(eta * std::sqrt((double)d) * (1.0 + std::ldexp(1.0, -11)) * 1.02);
          ctx->tc_keta2 = (float)((double)d * eta * eta * 1.02 + std::ldexp(1.0, -24 - 2 * e) + 1e-38);
          ctx->tc_mseed = true;
        } else {
          ctx->tc_mseed = bip <= 16384.0;  // fp16-stored grounds: unscaled seeds must fit fp16
        }
        {
          const char* mb = getenv("EBC200_TC_MB2");
          ctx->tc_mb2 = ctx->tc_np == 128 && !(mb && mb[0] == '0');
        }
        // in-MMA fp32 accumulation of the seed parts: (kpad + 16 + 8) 2^-23 |ip| on top
        // of the (d + 8) u (cm + |v|^2) seed/final-add quantum kpmax
        ctx->tc_kpscale = (float)((1.0 + (ctx->kpad + 24.0) / (d + 8.0)) * 1.01);
        if (ctx->tc_mseed && ctx->tc_fast) {
          CUC(cudaMallocAsync((void**)&ctx->tile_anchor0, (size_t)(ctx->n_pad / 128 + 1) * sizeof(int), ctx->stream));
          CUC(cudaMemsetAsync(ctx->tile_anchor0, 0, (size_t)(ctx->n_pad / 128 + 1) * sizeof(int), ctx->stream));
        }
      }
    }
    if (ctx->tc_fast) {
      k_split_f16<<<8 * ctx->num_sms, 256, 0, ctx->stream>>>(ctx->V32, ctx->pitch, ctx->n_pad, d, ctx->kpad,
                                                            (__half*)ctx->Vf, ctx->tc_oscale);
      CUC(cudaGetLastError());
    }
    if (ctx->tc_kind == tc::KIND_F16)
      k_split_f16<<<8 * ctx->num_sms, 256, 0, ctx->stream>>>(ctx->V32, ctx->pitch, ctx->n_pad, d, ctx->kpad,
                                                            (__half*)ctx->Vhi);
    else if (ctx->tc_kind == tc::KIND_BF16)
      k_split_bf16<<<8 * ctx->num_sms, 256, 0, ctx->stream>>>(ctx->V32, ctx->pitch, ctx->n_pad, d, ctx->kpad,
                                                             (__nv_bfloat16*)ctx->Vhi, (__nv_bfloat16*)ctx->Vlo);
    else
      k_split_tf32<<<8 * ctx->num_sms, 256, 0, ctx->stream>>>(ctx->V32, ctx->pitch, ctx->n_pad, d, ctx->kpad,
                                                             (float*)ctx->Vhi, (float*)ctx->Vlo);
    CUC(cudaGetLastError());
    if (ctx->tc_mseed) {
      // the splits zero K columns >= d: write the folded seeds after them
      k_seed_ipa<<<(unsigned)((ctx->n_pad + 255) / 256), 256, 0, ctx->stream>>>(ctx->cm64, n, ctx->n_pad,
                                                                                 tc_seeds(ctx));
      CUC(cudaGetLastError());
    }
  }
  double* bl = nullptr;
  CUC(cudaMallocAsync((void**)&bl, sizeof(double), ctx->stream));
  k_total<<<1, 32, 0, ctx->stream>>>(ctx->chunkpart, ctx->nchunks, 1.0 / (double)n, bl);
  CUC(cudaGetLastError());
  CUC(cudaMemcpyAsync(&ctx->baseline, bl, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CUC(cudaStreamSynchronize(ctx->stream));
  cudaFreeAsync(bl, ctx->stream);
  cudaFreeAsync(e0dev, ctx->stream);
  cudaFreeAsync(raw, ctx->stream);
  ctx->ev.resize(4);
  for (auto& e : ctx->ev) CUC(cudaEventCreate(&e));
#undef CUC
  mark("done");
  *out = ctx;
  return EBC_OK;
}

int ebc_baseline(const ebc_ctx* ctx, double* out) {
  if (!ctx || !out) return fail(nullptr, EBC_EINVAL, "ebc_baseline: NULL argument");
  *out = ctx->baseline;
  return EBC_OK;
}

int ebc_reset(ebc_ctx* ctx) {
  if (!ctx) return fail(nullptr, EBC_EINVAL, "ebc_reset: NULL context");
  CU(cudaSetDevice(ctx->device));
  int rc = do_reset(ctx);
  if (rc) return rc;
  CU(cudaStreamSynchronize(ctx->stream));
  return EBC_OK;
}

void* ebc_stream(const ebc_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int ebc_set_timing(ebc_ctx* ctx, int on) {
  if (!ctx) return fail(nullptr, EBC_EINVAL, "ebc_set_timing: NULL context");
  ctx->timing = on != 0;
  return EBC_OK;
}

int ebc_last_timings(const ebc_ctx* ctx, double* out_ms4) {
  if (!ctx || !out_ms4) return fail(nullptr, EBC_EINVAL, "ebc_last_timings: NULL argument");
  for (int i = 0; i < 4; ++i) out_ms4[i] = ctx->last_ms[i];
  return EBC_OK;
}

int64_t ebc_last_launches(const ebc_ctx* ctx) { return ctx ? ctx->launches : -1; }

#ifdef EBC200_TRACE
// Development only (-DEBC200_TRACE): read (and with reset, re-arm) the fused
// update's per-step phase stamps; out = 64 x 8 globaltimer values.
int ebc_debug_ub_trace(unsigned long long* out, int reset) {
  if (cudaDeviceSynchronize() != cudaSuccess) return EBC_ECUDA;
  if (out && cudaMemcpyFromSymbol(out, g_ub_trace, sizeof(g_ub_trace)) != cudaSuccess) return EBC_ECUDA;
  if (out && cudaMemcpyFromSymbol(out + 64 * 8, g_ub_blk, sizeof(g_ub_blk)) != cudaSuccess) return EBC_ECUDA;
  if (out && cudaMemcpyFromSymbol(out + 64 * 8 + 8192 * 4, g_tk_trace, sizeof(g_tk_trace)) != cudaSuccess)
    return EBC_ECUDA;
  if (reset) {
    static unsigned long long init[64][8];
    for (auto& r : init) {
      for (auto& x : r) x = 0ull;
      r[0] = ~0ull;
    }
    if (cudaMemcpyToSymbol(g_ub_trace, init, sizeof(init)) != cudaSuccess) return EBC_ECUDA;
    static unsigned long long tinit[64][4];
    for (auto& r : tinit) {
      for (auto& x : r) x = 0ull;
      r[0] = ~0ull;
    }
    if (cudaMemcpyToSymbol(g_tk_trace, tinit, sizeof(tinit)) != cudaSuccess) return EBC_ECUDA;
  }
  return EBC_OK;
}
#endif

int ebc_screen_info(const ebc_ctx* ctx, int64_t* out4) {
  if (!ctx || !out4) return fail(nullptr, EBC_EINVAL, "ebc_screen_info: NULL argument");
  out4[0] = ctx->screen_mode;
  out4[1] = ctx->tc_np;
  out4[2] = ctx->tc_np ? ctx->tc_kind : -1;
  out4[3] = ctx->kpad;
  return EBC_OK;
}

int ebc_last_screen_work(const ebc_ctx* ctx, int64_t* out_pairs) {
  if (!ctx || !out_pairs) return fail(nullptr, EBC_EINVAL, "ebc_last_screen_work: NULL argument");
  long long v[8];
  if (cudaMemcpy(v, ctx->stats, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess)
    return fail(const_cast<ebc_ctx*>(ctx), EBC_ECUDA, "ebc_last_screen_work: copy failed");
  *out_pairs = (int64_t)v[4] * tc::M * (ctx->tc_np ? ctx->tc_np : 0);
  return EBC_OK;
}

int ebc_host_register(const void* ptr, int64_t bytes) {
  if (!ptr || bytes <= 0) return fail(nullptr, EBC_EINVAL, "ebc_host_register: NULL or empty buffer");
  if (cudaHostRegister(const_cast<void*>(ptr), (size_t)bytes, cudaHostRegisterPortable) != cudaSuccess) {
    (void)cudaGetLastError();
    return fail(nullptr, EBC_ECUDA, "ebc_host_register: cudaHostRegister refused");
  }
  return EBC_OK;
}

int ebc_host_unregister(const void* ptr) {
  if (!ptr) return fail(nullptr, EBC_EINVAL, "ebc_host_unregister: NULL buffer");
  if (cudaHostUnregister(const_cast<void*>(ptr)) != cudaSuccess) {
    (void)cudaGetLastError();
    return fail(nullptr, EBC_ECUDA, "ebc_host_unregister: not registered");
  }
  return EBC_OK;
}

int ebc_last_lazy_stats(const ebc_ctx* ctx, int64_t* out4) {
  if (!ctx || !out4) return fail(nullptr, EBC_EINVAL, "ebc_last_lazy_stats: NULL argument");
  long long v[8];
  if (cudaMemcpy(v, ctx->stats, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess)
    return fail(const_cast<ebc_ctx*>(ctx), EBC_ECUDA, "ebc_last_lazy_stats: copy failed");
  out4[0] = ctx->lazy_on ? 1 : 0;
  out4[1] = v[7];
  out4[2] = v[5];
  out4[3] = v[6];
  return EBC_OK;
}

int ebc_last_stats(const ebc_ctx* ctx, int64_t* out4) {
  if (!ctx || !out4) return fail(nullptr, EBC_EINVAL, "ebc_last_stats: NULL argument");
  long long v[4];
  if (cudaMemcpy(v, ctx->stats, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess)
    return fail(const_cast<ebc_ctx*>(ctx), EBC_ECUDA, "ebc_last_stats: copy failed");
  for (int i = 0; i < 4; ++i) out4[i] = v[i];
  return EBC_OK;
}

}  // extern "C"

namespace {

// Shared driver of ebc_greedy (single device, full candidate range) and
// ebc_greedy_sharded (this rank's range, device-side NCCL exchange).
int greedy_run(ebc_ctx* ctx, int32_t k, bool sharded, int64_t* out_sel, double* out_val, double* out_gain,
               int64_t* out_evals) {
  if (!ctx) return fail(nullptr, EBC_EINVAL, "ebc_greedy: NULL context");
  if (k < 1) return fail(ctx, EBC_EINVAL, "k must be >= 1");
  if (k > ctx->n)
    return fail(ctx, EBC_EINVAL, "k=" + std::to_string(k) + " exceeds ground size " + std::to_string(ctx->n));
  if (!out_sel || !out_val || !out_gain) return fail(ctx, EBC_EINVAL, "ebc_greedy: NULL output buffer");
  CU(cudaSetDevice(ctx->device));
  ctx->launches = 0;
  if (!sharded) {
    ctx->c0 = 0;
    ctx->c1 = ctx->n;
  } else {
    const SharedComm& sc = shared_comm(ctx->device);
    if (!sc.comm) return fail(ctx, EBC_EINVAL, "ebc_greedy_sharded: no communicator (call ebc_comm_init)");
    if (ctx->comm != sc.comm || ctx->comm_gen != sc.generation) {
      const int arc = ebc_comm_attach(ctx);
      if (arc) return arc;
    }
    int rc0 = ensure(ctx, ctx->tie_rec, (size_t)(TIE_CAP + 1) * sizeof(double2));
    if (!rc0) rc0 = ensure(ctx, ctx->tie_all, (size_t)ctx->nranks * (TIE_CAP + 1) * sizeof(double2));
    if (!rc0) rc0 = ensure(ctx, ctx->sel_hash, (size_t)(ctx->nranks + 1) * sizeof(unsigned long long));
    if (rc0) return rc0;
  }
  int rc = ensure(ctx, ctx->sel_out, (size_t)k * sizeof(int64_t));
  if (!rc) rc = ensure(ctx, ctx->val_out, (size_t)k * sizeof(double));
  if (!rc) rc = ensure(ctx, ctx->gain_out, (size_t)k * sizeof(double));
  if (rc) return rc;
  if (ctx->timing) {
    rc = ensure_events(ctx, 4 * k);
    if (rc) return rc;
  }
  double acc_ms[4] = {0, 0, 0, 0};
  ScopedEvent ts, te;  // destroyed on every return path
  CU(cudaEventCreate(&ts.e));
  CU(cudaEventCreate(&te.e));
  cudaEvent_t tstart = ts.e, tend = te.e;
  CU(cudaEventRecord(tstart, ctx->stream));
  // The k-step loop has no host decision in it, so the second run with the
  // same k is captured as a CUDA graph and launched; later runs replay it (one
  // launch instead of ~10 per step: matters for small N, e.g. C1).  The first
  // run stays eager, so a context used once (the e2e path) never pays for
  // capture + instantiation.
  // timing mode captures the per-step event records into the graph too
  // (external event record nodes: cudaEventRecordExternal, which keep timing),
  // so timed runs are replays like the untimed product path
  const bool graph_ok = ctx->use_graphs;
  const int key = (k << 2) | (ctx->timing ? 2 : 0) | (sharded ? 1 : 0);
  auto enqueue = [&]() { return sharded ? enqueue_greedy_sharded(ctx, k) : enqueue_greedy(ctx, k); };
  ebc_ctx::Graph* cached = nullptr;
  for (auto& g : ctx->graphs)
    if (g.k == key && g.c0 == ctx->c0 && g.c1 == ctx->c1 && g.epoch == ctx->alloc_epoch) cached = &g;
  const ebc_ctx::Eager* er = nullptr;
  for (const auto& e : ctx->eager)
    if (e.k == key && e.c0 == ctx->c0 && e.c1 == ctx->c1) er = &e;
  const bool seen = er != nullptr;
  const int seen_lv = er ? std::max(0, std::min(3, er->lv)) : 3;
  std::vector<char> dec_rec;
  long long dec_expect = -1, dec_run = -1;
  if (graph_ok && !cached && seen) {
    const int64_t before = ctx->launches;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    bool ok = cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    const int64_t epoch = ctx->alloc_epoch;
    if (ok) {
      // a Greedy run is a deterministic function of (V, e0, k): replays take the
      // eager run's path down the ladder, so the graph holds only those rungs
      ctx->ladder_max = seen_lv;
      ctx->capturing = true;
      if (!sharded && ctx->spec_dec && !er->dec.empty()) ctx->cap_dec = &er->dec;
      const int crc = enqueue();
      ctx->cap_dec = nullptr;
      ctx->capturing = false;
      ctx->ladder_max = 3;
      ok = cudaStreamEndCapture(ctx->stream, &graph) == cudaSuccess && crc == EBC_OK && epoch == ctx->alloc_epoch;
    }
    if (ok) ok = cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();  // a failed capture only disables graphs
    if (ok) {
      for (auto it = ctx->graphs.begin(); it != ctx->graphs.end();)
        if (it->k == key && it->c0 == ctx->c0 && it->c1 == ctx->c1) {
          cudaGraphExecDestroy(it->exec);
          it = ctx->graphs.erase(it);
        } else {
          ++it;
        }
      const long long nd = !sharded && ctx->spec_dec && !er->dec.empty() ? er->decided : -1;
      ctx->graphs.push_back({key, ctx->c0, ctx->c1, epoch, ctx->launches - before, exec, nd});
      cached = &ctx->graphs.back();
    } else {
      ctx->use_graphs = false;
    }
    ctx->launches = before;
  }
  if (graph_ok && cached) {
    CU(cudaGraphLaunch(cached->exec, ctx->stream));
    ctx->launches = cached->launches;
    dec_expect = cached->decided;
    if (dec_expect >= 0)
      CU(cudaMemcpyAsync(&dec_run, ctx->stats + 5, sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
  } else {
    // a repeated eager run (timing mode: per-step events, no graph) takes the
    // first run's path down the ladder, like a replayed graph
    if (seen) ctx->ladder_max = seen_lv;
    if (!seen) {
      dec_rec.assign((size_t)k, 0);
      ctx->rec_dec = &dec_rec;
    }
    rc = enqueue();
    ctx->rec_dec = nullptr;
    ctx->ladder_max = 3;
    if (rc) return rc;
  }
  long long lv_end = 3, dec_eager = -1;
  if (!(graph_ok && cached) && !seen) {
    CU(cudaMemcpyAsync(&lv_end, ctx->stats + 2, sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(&dec_eager, ctx->stats + 5, sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
  }
  CU(cudaEventRecord(tend, ctx->stream));
  CU(cudaMemcpyAsync(out_sel, ctx->sel_out.p, (size_t)k * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaMemcpyAsync(out_val, ctx->val_out.p, (size_t)k * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaMemcpyAsync(out_gain, ctx->gain_out.p, (size_t)k * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  int tie_err = 0;
  if (sharded) CU(cudaMemcpyAsync(&tie_err, ctx->tie_err, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  if (!(graph_ok && cached) && !seen)
    ctx->eager.push_back({key, ctx->c0, ctx->c1, lv_end < 0 ? 3 : (int)lv_end,
                          ctx->eager_sync ? dec_rec : std::vector<char>(), dec_eager});
  if (dec_expect >= 0 && dec_run != dec_expect)
    return fail(ctx, EBC_ECUDA, "Greedy graph replay diverged from its eager run (" + std::to_string(dec_run) +
                                    " decided lazy steps, " + std::to_string(dec_expect) + " in the eager run)");
  ctx->comm_status = tie_err;
  if (tie_err & 2)
    return fail(ctx, EBC_ECOMM, "sharded Greedy: ranks disagree on the selection (end-of-run hash mismatch)");
  if (tie_err)
    return fail(ctx, EBC_ECOMM, "sharded Greedy: a rank's tie-set frontier exceeded " + std::to_string(TIE_CAP) +
                                    " records (use the host exchange)");
  if (ctx->timing) {
    for (int st = 0; st < k; ++st) {
      float a = 0, b = 0, c = 0;
      if (ctx->lazy_on && st > 0) {
        // lazy step: selection (batch, and the screen when re-run) + update;
        // a fused update (k_update_batch) is timed from after the next
        // batch's top-k (selection work)
        const bool fz = (size_t)st < ctx->fused_step.size() && ctx->fused_step[st];
        CU(cudaEventElapsedTime(&a, ctx->ev[4 * (st - 1) + 3], ctx->ev[4 * st + (fz ? 2 : 1)]));
        CU(cudaEventElapsedTime(&c, ctx->ev[4 * st + (fz ? 2 : 1)], ctx->ev[4 * st + 3]));
        acc_ms[0] += a;
        acc_ms[2] += c;
        continue;
      }
      CU(cudaEventElapsedTime(&a, ctx->ev[4 * st + 0], ctx->ev[4 * st + 1]));
      CU(cudaEventElapsedTime(&b, ctx->ev[4 * st + 1], ctx->ev[4 * st + 2]));
      CU(cudaEventElapsedTime(&c, ctx->ev[4 * st + 2], ctx->ev[4 * st + 3]));
      acc_ms[0] += a;
      acc_ms[1] += b;
      acc_ms[2] += c;
    }
  }
  float tot = 0;
  CU(cudaEventElapsedTime(&tot, tstart, tend));
  acc_ms[3] = tot;
  for (int i = 0; i < 4; ++i) ctx->last_ms[i] = acc_ms[i];
  ctx->steps_done = k;
  if (out_evals) {
    int64_t ev = 0;
    for (int s = 0; s < k; ++s) ev += ctx->n - s;
    *out_evals = ev;
  }
  for (int s = 0; s < k; ++s)
    if (out_sel[s] < 0) return fail(ctx, EBC_ECUDA, "greedy step " + std::to_string(s) + " found no candidate");
  return EBC_OK;
}

}  // namespace

extern "C" {

int ebc_greedy(ebc_ctx* ctx, int32_t k, int64_t* out_sel, double* out_val, double* out_gain, int64_t* out_evals) {
  return greedy_run(ctx, k, false, out_sel, out_val, out_gain, out_evals);
}

int ebc_comm_unique_id(unsigned char* out_id, int64_t bytes) {
  if (!out_id || bytes < (int64_t)sizeof(ncclUniqueId)) return fail(nullptr, EBC_EINVAL, "ebc_comm_unique_id: buffer too small");
  const NcclApi& api = nccl_api();
  if (!api.ok) return fail(nullptr, EBC_ECOMM, "NCCL (libnccl.so.2) not available");
  ncclUniqueId id;
  const ncclResult_t r = api.GetUniqueId(&id);
  if (r != ncclSuccess) return fail(nullptr, EBC_ECOMM, std::string("ncclGetUniqueId: ") + api.GetErrorString(r));
  std::memcpy(out_id, &id, sizeof(id));
  return EBC_OK;
}

int64_t ebc_comm_id_bytes(void) { return (int64_t)sizeof(ncclUniqueId); }

int ebc_comm_init(ebc_ctx* ctx, const unsigned char* id, int64_t bytes, int32_t nranks, int32_t rank) {
  if (!ctx || !id || bytes < (int64_t)sizeof(ncclUniqueId)) return fail(ctx, EBC_EINVAL, "ebc_comm_init: bad argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(ctx, EBC_EINVAL, "ebc_comm_init: bad rank / world size");
  const NcclApi& api = nccl_api();
  if (!api.ok) return fail(ctx, EBC_ECOMM, "NCCL (libnccl.so.2) not available");
  CU(cudaSetDevice(ctx->device));
  // one communicator per device and process, shared by every context on it
  // (an EbcFunction per call must not pay ncclCommInitRank each time)
  SharedComm& sc = shared_comm(ctx->device);
  if (sc.comm) api.CommDestroy(sc.comm);  // contexts still holding it re-attach below / via ebc_comm_attach
  sc.comm = nullptr;
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  const ncclResult_t r = api.CommInitRank(&sc.comm, nranks, uid, rank);
  if (r != ncclSuccess) {
    sc.comm = nullptr;
    ctx->comm = nullptr;
    return fail(ctx, EBC_ECOMM, std::string("ncclCommInitRank: ") + api.GetErrorString(r));
  }
  sc.nranks = nranks;
  sc.rank = rank;
  ++sc.generation;
  return ebc_comm_attach(ctx);
}

int ebc_comm_attach(ebc_ctx* ctx) {
  if (!ctx) return fail(nullptr, EBC_EINVAL, "ebc_comm_attach: NULL context");
  const SharedComm& sc = shared_comm(ctx->device);
  if (!sc.comm) return fail(ctx, EBC_ECOMM, "no communicator on this device (call ebc_comm_init)");
  CU(cudaSetDevice(ctx->device));
  ctx->comm = sc.comm;
  ctx->comm_gen = sc.generation;
  ctx->nranks = sc.nranks;
  ctx->rank = sc.rank;
  if (!ctx->tie_err) CU(cudaMallocAsync((void**)&ctx->tie_err, sizeof(int), ctx->stream));
  ++ctx->alloc_epoch;  // graphs captured with another communicator are stale
  return EBC_OK;
}

int ebc_greedy_sharded(ebc_ctx* ctx, int32_t k, int64_t* out_sel, double* out_val, double* out_gain,
                       int64_t* out_evals) {
  return greedy_run(ctx, k, true, out_sel, out_val, out_gain, out_evals);
}

int32_t ebc_tie_cap(void) { return TIE_CAP; }

int ebc_comm_status(const ebc_ctx* ctx, int32_t* out_flags) {
  if (!ctx || !out_flags) return fail(nullptr, EBC_EINVAL, "ebc_comm_status: NULL argument");
  *out_flags = ctx->comm_status;
  return EBC_OK;
}

int ebc_shard_tie_step(ebc_ctx* ctx, double* out_rec, double* out_current) {
  if (!ctx || !out_rec || !out_current) return fail(ctx, EBC_EINVAL, "ebc_shard_tie_step: NULL argument");
  CU(cudaSetDevice(ctx->device));
  int rc = ensure(ctx, ctx->tie_rec, (size_t)(TIE_CAP + 1) * sizeof(double2));
  if (rc) return rc;
  if (ctx->c1 > ctx->c0) {
    rc = run_step_select(ctx, 0, 0, nullptr);
    if (rc) return rc;
  } else {
    CU(cudaMemsetAsync(ctx->wcount, 0, sizeof(int), ctx->stream));
  }
  k_tie_records<<<1, 1024, 0, ctx->stream>>>(ctx->wcount, ctx->wlist, ctx->wgain, 1.0 / (double)ctx->n, ctx->cur,
                                             (double2*)ctx->tie_rec.p);
  KCHECK();
  CU(cudaMemcpyAsync(out_rec, ctx->tie_rec.p, (size_t)(TIE_CAP + 1) * sizeof(double2), cudaMemcpyDeviceToHost,
                     ctx->stream));
  CU(cudaMemcpyAsync(out_current, ctx->cur, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return EBC_OK;
}

int ebc_shard_pick_commit(ebc_ctx* ctx, const double* gathered, int32_t world, int32_t step, int64_t* out_best,
                          double* out_value) {
  if (!ctx || !gathered || world < 1 || !out_best || !out_value)
    return fail(ctx, EBC_EINVAL, "ebc_shard_pick_commit: bad argument");
  CU(cudaSetDevice(ctx->device));
  int rc = ensure(ctx, ctx->tie_all, (size_t)world * (TIE_CAP + 1) * sizeof(double2));
  if (!rc) rc = ensure(ctx, ctx->sel_out, (size_t)(step + 1) * sizeof(int64_t));
  if (!rc) rc = ensure(ctx, ctx->val_out, (size_t)(step + 1) * sizeof(double));
  if (!rc) rc = ensure(ctx, ctx->gain_out, (size_t)(step + 1) * sizeof(double));
  if (rc) return rc;
  if (!rc && ctx->timing) rc = ensure_events(ctx, 4 * (size_t)(step + 1));  // run_update records slot 4 step + 3
  if (rc) return rc;
  if (!ctx->tie_err) CU(cudaMallocAsync((void**)&ctx->tie_err, sizeof(int), ctx->stream));
  CU(cudaMemsetAsync(ctx->tie_err, 0, sizeof(int), ctx->stream));
  CU(cudaMemcpyAsync(ctx->tie_all.p, gathered, (size_t)world * (TIE_CAP + 1) * sizeof(double2),
                     cudaMemcpyHostToDevice, ctx->stream));
  k_pick_global<<<1, 1024, 0, ctx->stream>>>((const double2*)ctx->tie_all.p, world, 1.0 / (double)ctx->n, ctx->cur,
                                             ctx->best, ctx->selected, (int64_t*)ctx->sel_out.p, step, ctx->tie_err);
  KCHECK();
  rc = run_update(ctx, step, (double*)ctx->val_out.p, (double*)ctx->gain_out.p);
  if (rc) return rc;
  int err = 0;
  CU(cudaMemcpyAsync(out_best, ctx->best, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaMemcpyAsync(out_value, ctx->cur, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaMemcpyAsync(&err, ctx->tie_err, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  ctx->steps_done += 1;
  if (err) return fail(ctx, EBC_ECOMM, "tie set exceeded " + std::to_string(TIE_CAP) + " records");
  return EBC_OK;
}

int ebc_shard_set_range(ebc_ctx* ctx, int64_t c0, int64_t c1) {
  if (!ctx) return fail(nullptr, EBC_EINVAL, "ebc_shard_set_range: NULL context");
  if (c0 < 0 || c1 < c0 || c1 > ctx->n)
    return fail(ctx, EBC_EINVAL,
                "candidate range [" + std::to_string(c0) + ", " + std::to_string(c1) + ") outside [0, n)");
  if (c0 < c1 && (c0 % tc::M) != 0)
    return fail(ctx, EBC_EINVAL,
                "candidate range start " + std::to_string(c0) + " is not a multiple of " + std::to_string(tc::M));
  // cached graphs and eager ladder records are keyed by the range (greedy_run)
  ctx->c0 = c0;
  ctx->c1 = c1;
  return EBC_OK;
}

int ebc_shard_step(ebc_ctx* ctx, int64_t* out_idx, double* out_gain, int64_t cap, int64_t* out_count,
                   double* out_current) {
  if (!ctx || !out_count) return fail(ctx, EBC_EINVAL, "ebc_shard_step: NULL argument");
  CU(cudaSetDevice(ctx->device));
  int count = 0;
  if (ctx->c1 > ctx->c0) {
    ctx->launches = 0;
    int rc = run_step_select(ctx, 0, 0, nullptr);
    if (rc) return rc;
    CU(cudaMemcpyAsync(&count, ctx->wcount, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
  }
  *out_count = count;
  const int64_t m = std::min<int64_t>(cap, count);
  if (m > 0) {
    if (!out_idx || !out_gain) return fail(ctx, EBC_EINVAL, "ebc_shard_step: NULL output buffer");
    CU(cudaMemcpyAsync(out_idx, ctx->wlist, (size_t)m * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(out_gain, ctx->wgain, (size_t)m * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  }
  if (out_current) CU(cudaMemcpyAsync(out_current, ctx->cur, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return EBC_OK;
}

int ebc_shard_advance(ebc_ctx* ctx, int64_t commit_idx, int32_t run_step, int64_t* out_idx, double* out_gain,
                      int64_t cap, int64_t* out_count, double* out_current) {
  if (!ctx || !out_count || !out_current) return fail(ctx, EBC_EINVAL, "ebc_shard_advance: NULL argument");
  if (commit_idx >= ctx->n)
    return fail(ctx, EBC_EINDEX, "index " + std::to_string(commit_idx) + " out of range for ground size " +
                                     std::to_string(ctx->n));
  CU(cudaSetDevice(ctx->device));
  ctx->launches = 0;
  if (commit_idx >= 0) {
    CU(cudaMemcpyAsync(ctx->best, &commit_idx, sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
    const unsigned char one = 1;
    CU(cudaMemcpyAsync(ctx->selected + commit_idx, &one, 1, cudaMemcpyHostToDevice, ctx->stream));
    int rc = run_update(ctx, 0, nullptr, nullptr);
    if (rc) return rc;
    ctx->steps_done += 1;
  }
  int count = 0;
  const bool step = run_step && ctx->c1 > ctx->c0;
  if (step) {
    int rc = run_step_select(ctx, 0, 0, nullptr);
    if (rc) return rc;
    CU(cudaMemcpyAsync(&count, ctx->wcount, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    const int64_t m = std::min<int64_t>(cap, ctx->n);
    if (m > 0 && out_idx && out_gain) {
      // optimistic: the first `cap` entries travel with the same sync
      CU(cudaMemcpyAsync(out_idx, ctx->wlist, (size_t)m * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
      CU(cudaMemcpyAsync(out_gain, ctx->wgain, (size_t)m * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    }
  }
  CU(cudaMemcpyAsync(out_current, ctx->cur, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  *out_count = count;
  return EBC_OK;
}

int ebc_shard_fetch(const ebc_ctx* ctx, int64_t* out_idx, double* out_gain, int64_t count) {
  if (!ctx || (count > 0 && (!out_idx || !out_gain))) return fail(nullptr, EBC_EINVAL, "ebc_shard_fetch: NULL argument");
  if (count > ctx->n) return fail(const_cast<ebc_ctx*>(ctx), EBC_EINVAL, "ebc_shard_fetch: count exceeds n");
  if (count <= 0) return EBC_OK;
  if (cudaMemcpy(out_idx, ctx->wlist, (size_t)count * sizeof(int64_t), cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemcpy(out_gain, ctx->wgain, (size_t)count * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
    return fail(const_cast<ebc_ctx*>(ctx), EBC_ECUDA, "ebc_shard_fetch: copy failed");
  return EBC_OK;
}

int ebc_shard_commit(ebc_ctx* ctx, int64_t s, double* out_value) {
  if (!ctx) return fail(nullptr, EBC_EINVAL, "ebc_shard_commit: NULL context");
  if (s < 0 || s >= ctx->n)
    return fail(ctx, EBC_EINDEX, "index " + std::to_string(s) + " out of range for ground size " +
                                     std::to_string(ctx->n));
  CU(cudaSetDevice(ctx->device));
  CU(cudaMemcpyAsync(ctx->best, &s, sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
  const unsigned char one = 1;
  CU(cudaMemcpyAsync(ctx->selected + s, &one, 1, cudaMemcpyHostToDevice, ctx->stream));
  int rc = run_update(ctx, 0, nullptr, nullptr);
  if (rc) return rc;
  double v = 0;
  CU(cudaMemcpyAsync(&v, ctx->cur, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  ctx->steps_done += 1;
  if (out_value) *out_value = v;
  return EBC_OK;
}

int ebc_sieve_reserve(ebc_ctx* ctx, int32_t slots) {
  if (!ctx) return fail(nullptr, EBC_EINVAL, "ebc_sieve_reserve: NULL context");
  if (slots < 1) return fail(ctx, EBC_EINVAL, "ebc_sieve_reserve: slots must be >= 1");
  CU(cudaSetDevice(ctx->device));
  int rc = ensure(ctx, ctx->sv_cm, (size_t)slots * ctx->n_pad * sizeof(double));
  if (!rc) rc = ensure(ctx, ctx->sv_de, (size_t)ctx->n_pad * sizeof(double));
  if (!rc) rc = ensure(ctx, ctx->sv_slots, (size_t)3 * (slots + 1) * sizeof(int));
  if (!rc) rc = ensure(ctx, ctx->sv_part, (size_t)(slots + 1) * ctx->nchunks * sizeof(double));
  if (!rc) rc = ensure(ctx, ctx->sv_out, (size_t)(slots + 1) * sizeof(double));
  if (rc) return rc;
  if (slots > ctx->sv_nslots) {
    if (ctx->sv_slots_host) cudaFreeHost(ctx->sv_slots_host);
    if (ctx->sv_out_host) cudaFreeHost(ctx->sv_out_host);
    ctx->sv_slots_host = nullptr;
    ctx->sv_out_host = nullptr;
    CU(cudaMallocHost((void**)&ctx->sv_slots_host, (size_t)3 * (slots + 1) * sizeof(int)));
    CU(cudaMallocHost((void**)&ctx->sv_out_host, (size_t)(slots + 1) * sizeof(double)));
    ctx->sv_nslots = slots;
  }
  return EBC_OK;
}

int ebc_sieve_step(ebc_ctx* ctx, int64_t commit_e, const int32_t* commit_slots, int32_t n_commit,
                   const int32_t* reset_slots, int32_t n_reset, int64_t e, const int32_t* eval_slots,
                   int32_t n_eval, double* out_single, double* out_values) {
  if (!ctx) return fail(nullptr, EBC_EINVAL, "ebc_sieve_step: NULL context");
  if (n_commit < 0 || n_reset < 0 || n_eval < 0 || (n_commit && !commit_slots) || (n_reset && !reset_slots) ||
      (n_eval && (!eval_slots || !out_values)) || (e >= 0 && !out_single))
    return fail(ctx, EBC_EINVAL, "ebc_sieve_step: bad slot lists");
  if (n_commit > ctx->sv_nslots || n_reset > ctx->sv_nslots || n_eval > ctx->sv_nslots)
    return fail(ctx, EBC_EINVAL, "ebc_sieve_step: more slots than reserved");
  if (commit_e >= ctx->n || e >= ctx->n)
    return fail(ctx, EBC_EINDEX, "index " + std::to_string(std::max(commit_e, e)) + " out of range for ground size " +
                                     std::to_string(ctx->n));
  int* hs = ctx->sv_slots_host;
  for (int i = 0; i < n_commit; ++i) hs[i] = commit_slots[i];
  for (int i = 0; i < n_reset; ++i) hs[n_commit + i] = reset_slots[i];
  for (int i = 0; i < n_eval; ++i) hs[n_commit + n_reset + i] = eval_slots[i];
  for (int i = 0; i < n_commit + n_reset + n_eval; ++i)
    if (hs[i] < 0 || hs[i] >= ctx->sv_nslots) return fail(ctx, EBC_EINVAL, "ebc_sieve_step: slot out of range");
  CU(cudaSetDevice(ctx->device));
  ctx->launches = 0;
  int* ds = (int*)ctx->sv_slots.p;
  const int tot = n_commit + n_reset + n_eval;
  if (tot) CU(cudaMemcpyAsync(ds, hs, (size_t)tot * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
  double* cm = (double*)ctx->sv_cm.p;
  double* de = (double*)ctx->sv_de.p;
  const size_t smem = (size_t)2 * ctx->d * sizeof(double);
  const unsigned grid = (unsigned)((ctx->n + RED_THREADS - 1) / RED_THREADS);
  if (n_commit || n_reset || e >= 0) {
    if (ctx->dtype == EBC_F64) {
      CU(cudaFuncSetAttribute(k_sieve_points<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem + 1024));
      k_sieve_points<double><<<grid, RED_THREADS, smem, ctx->stream>>>(ctx->V64, ctx->pitch, ctx->n, ctx->d, ctx->e0d,
                                                                      cm, ctx->n_pad, n_commit ? commit_e : -1, ds,
                                                                      n_commit, n_reset, e, de);
    } else {
      CU(cudaFuncSetAttribute(k_sieve_points<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem + 1024));
      k_sieve_points<float><<<grid, RED_THREADS, smem, ctx->stream>>>(ctx->V32, ctx->pitch, ctx->n, ctx->d, ctx->e0d,
                                                                     cm, ctx->n_pad, n_commit ? commit_e : -1, ds,
                                                                     n_commit, n_reset, e, de);
    }
    KCHECK();
  }
  if (e < 0) {
    CU(cudaStreamSynchronize(ctx->stream));
    return EBC_OK;
  }
  double* part = (double*)ctx->sv_part.p;
  dim3 g2((unsigned)ctx->nchunks, (unsigned)((n_eval + 1 + 7) / 8));
  k_sieve_sums<<<g2, RED_THREADS, 0, ctx->stream>>>(ctx->n, ctx->e0d, cm, ctx->n_pad, de, ds + n_commit + n_reset,
                                                   n_eval, ctx->nchunks, part);
  KCHECK();
  k_multiset_final<<<(unsigned)((n_eval + 1 + 127) / 128), 128, 0, ctx->stream>>>(part, n_eval + 1, ctx->nchunks,
                                                                                  1.0 / (double)ctx->n,
                                                                                  (double*)ctx->sv_out.p);
  KCHECK();
  CU(cudaMemcpyAsync(ctx->sv_out_host, ctx->sv_out.p, (size_t)(n_eval + 1) * sizeof(double), cudaMemcpyDeviceToHost,
                     ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  *out_single = ctx->sv_out_host[0];
  for (int i = 0; i < n_eval; ++i) out_values[i] = ctx->sv_out_host[1 + i];
  return EBC_OK;
}

int ebc_kmedoids_loss(ebc_ctx* ctx, const double* reps, int64_t r, double* out) {
  if (!ctx) return fail(nullptr, EBC_EINVAL, "ebc_kmedoids_loss: NULL context");
  if (!reps || !out) return fail(ctx, EBC_EINVAL, "ebc_kmedoids_loss: NULL argument");
  if (r < 1) return fail(ctx, EBC_EINVAL, "the loss is undefined for an empty representative set");
  for (int64_t i = 0; i < r * ctx->d; ++i)
    if (!std::isfinite(reps[i])) return fail(ctx, EBC_EINVAL, "representatives must be finite");
  CU(cudaSetDevice(ctx->device));
  ctx->launches = 0;
  int rc = ensure(ctx, ctx->ms_part, (size_t)r * ctx->d * sizeof(double));
  if (rc) return rc;
  CU(cudaMemcpyAsync(ctx->ms_part.p, reps, (size_t)r * ctx->d * sizeof(double), cudaMemcpyHostToDevice,
                     ctx->stream));
  // representatives staged in shared memory, up to 48 KB per pass
  const int per = (int)std::max<int64_t>(1, std::min<int64_t>(r, 6144 / ctx->d));
  const unsigned grid = (unsigned)((ctx->n + RED_THREADS - 1) / RED_THREADS);
  for (int64_t r0 = 0; r0 < r; r0 += per) {
    const int r1 = (int)std::min<int64_t>(r, r0 + per);
    const size_t smem = (size_t)(r1 - r0) * ctx->d * sizeof(double);
    if (ctx->dtype == EBC_F64) {
      CU(cudaFuncSetAttribute(k_kmed_min<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_kmed_min<double><<<grid, RED_THREADS, smem, ctx->stream>>>(ctx->V64, ctx->pitch, ctx->n, ctx->d,
                                                                   (const double*)ctx->ms_part.p, (int)r0, r1,
                                                                   ctx->terms, r0 == 0);
    } else {
      CU(cudaFuncSetAttribute(k_kmed_min<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_kmed_min<float><<<grid, RED_THREADS, smem, ctx->stream>>>(ctx->V32, ctx->pitch, ctx->n, ctx->d,
                                                                  (const double*)ctx->ms_part.p, (int)r0, r1,
                                                                  ctx->terms, r0 == 0);
    }
    KCHECK();
  }
  k_sum_chunks<<<ctx->nchunks, RED_THREADS, 0, ctx->stream>>>(ctx->terms, ctx->n, ctx->chunkpart);
  KCHECK();
  rc = ensure(ctx, ctx->ms_out, sizeof(double));
  if (rc) return rc;
  double* dout = (double*)ctx->ms_out.p;
  k_mean<<<1, 1, 0, ctx->stream>>>(ctx->chunkpart, ctx->nchunks, (double)ctx->n, dout);
  KCHECK();
  CU(cudaMemcpyAsync(out, dout, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return EBC_OK;
}

int ebc_eval_multiset(ebc_ctx* ctx, const int64_t* offsets, const int64_t* idx, int64_t l, double* out_f,
                      int64_t* out_bad_set, int64_t* out_bad_index) {
  if (!ctx) return fail(nullptr, EBC_EINVAL, "ebc_eval_multiset: NULL context");
  if (l < 1) return fail(ctx, EBC_EINVAL, "a multiset must contain at least one set");
  if (!offsets || !out_f) return fail(ctx, EBC_EINVAL, "ebc_eval_multiset: NULL argument");
  if (offsets[0] != 0) return fail(ctx, EBC_EINVAL, "offsets[0] must be 0");
  for (int64_t j = 0; j < l; ++j)
    if (offsets[j + 1] < offsets[j]) return fail(ctx, EBC_EINVAL, "offsets must be non-decreasing");
  const int64_t nnz = offsets[l];
  if (nnz > 0 && !idx) return fail(ctx, EBC_EINVAL, "ebc_eval_multiset: NULL idx");
  // validate in set order (core.py:136-143): negative indices first, as EvalMultiset does
  for (int64_t j = 0; j < l; ++j)
    for (int64_t p = offsets[j]; p < offsets[j + 1]; ++p)
      if (idx[p] < 0) {
        if (out_bad_set) *out_bad_set = j;
        if (out_bad_index) *out_bad_index = idx[p];
        return fail(ctx, EBC_EINDEX, "set " + std::to_string(j) + " contains a negative index");
      }
  for (int64_t j = 0; j < l; ++j)
    for (int64_t p = offsets[j]; p < offsets[j + 1]; ++p)
      if (idx[p] >= ctx->n) {
        if (out_bad_set) *out_bad_set = j;
        if (out_bad_index) *out_bad_index = idx[p];
        return fail(ctx, EBC_EINDEX, "set " + std::to_string(j) + ": index " + std::to_string(idx[p]) +
                                         " out of range for ground size " + std::to_string(ctx->n));
      }
  CU(cudaSetDevice(ctx->device));
  ctx->launches = 0;
  int rc = ensure(ctx, ctx->ms_off, (size_t)(l + 1) * sizeof(int64_t));
  if (!rc) rc = ensure(ctx, ctx->ms_idx, (size_t)std::max<int64_t>(nnz, 1) * sizeof(int64_t));
  if (!rc) rc = ensure(ctx, ctx->ms_out, (size_t)l * sizeof(double));
  if (rc) return rc;
  const int64_t batch = std::min<int64_t>(l, 65535);
  ScopedEvent ea, eb;  // destroyed on every return path
  CU(cudaEventCreate(&ea.e));
  CU(cudaEventCreate(&eb.e));
  cudaEvent_t a = ea.e, b = eb.e;
  CU(cudaMemcpyAsync(ctx->ms_off.p, offsets, (size_t)(l + 1) * sizeof(int64_t), cudaMemcpyHostToDevice,
                     ctx->stream));
  if (nnz > 0)
    CU(cudaMemcpyAsync(ctx->ms_idx.p, idx, (size_t)nnz * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaEventRecord(a, ctx->stream));
  bool done = false;
  if (ctx->dtype != EBC_F64 && ctx->ms_mode >= 1) {
    ScreenPlan probe;
    const int64_t sc0 = ctx->c0, sc1 = ctx->c1;
    ctx->c0 = 0;
    ctx->c1 = std::max<int64_t>(nnz, 1);
    const bool fits = plan_screen(ctx, probe) == EBC_OK;
    ctx->c0 = sc0;
    ctx->c1 = sc1;
    if (fits && nnz > 0) {
      rc = multiset_sparse(ctx, l, nnz);
      if (rc == EBC_OK) done = true;
      else if (rc != EBC_EINVAL) return rc;
    }
  }
  if (!done) {
    // dense fallback: partials of one batch of sets at a time (batch x nchunks),
    // allocated only when it runs; each batch is finished before the next
    rc = ensure(ctx, ctx->ms_part, (size_t)std::min<int64_t>(l, batch) * ctx->nchunks * sizeof(double));
    if (rc) return rc;
  }
  for (int64_t s0 = 0; !done && s0 < l; s0 += batch) {
    const int64_t nb = std::min<int64_t>(batch, l - s0);
    dim3 grid(ctx->nchunks, (unsigned)nb);
    double* part = (double*)ctx->ms_part.p;  // k_multiset indexes it by (set - s0)
    if (ctx->dtype == EBC_F64)
      k_multiset<double><<<grid, RED_THREADS, 0, ctx->stream>>>(ctx->V64, ctx->pitch, ctx->n, ctx->d, ctx->e0d,
                                                               (const int64_t*)ctx->ms_off.p,
                                                               (const int64_t*)ctx->ms_idx.p, s0, ctx->nchunks, part);
    else
      k_multiset<float><<<grid, RED_THREADS, 0, ctx->stream>>>(ctx->V32, ctx->pitch, ctx->n, ctx->d, ctx->e0d,
                                                              (const int64_t*)ctx->ms_off.p,
                                                              (const int64_t*)ctx->ms_idx.p, s0, ctx->nchunks, part);
    KCHECK();
    k_multiset_final<<<(unsigned)((nb + 255) / 256), 256, 0, ctx->stream>>>(
        part, nb, ctx->nchunks, 1.0 / (double)ctx->n, (double*)ctx->ms_out.p + s0);
    KCHECK();
  }
  CU(cudaEventRecord(b, ctx->stream));
  CU(cudaMemcpyAsync(out_f, ctx->ms_out.p, (size_t)l * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  float ms = 0;
  CU(cudaEventElapsedTime(&ms, a, b));
  ctx->last_ms[0] = ms;
  ctx->last_ms[1] = 0;
  ctx->last_ms[2] = 0;
  ctx->last_ms[3] = ms;
  return EBC_OK;
}

void ebc_destroy(ebc_ctx* ctx) { free_ctx(ctx); }

}  // extern "C"
