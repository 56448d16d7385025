// Host runtime of the transpose-free slab 3D real FFT: plans, twiddle tables,
// the two exchange transports (NCCL over NVLink; in-process local fabric on
// one device) and the forward / inverse stage orchestration behind the C ABI
// declared in include/tffft.h.
//
// Pipeline (reference dfft.py:148-215, STRIDED strategy):
//   forward: r2c rows (n2) -> c2c columns (n1), epilogue splits self band /
//            peer bands -> exchange (peer chunks land in the vacated bands,
//            exchange.py:263-276) -> in-place c2c along n0 over the
//            STRIDED_INPLACE columns (kernels.py:176-200)
//   inverse: c2c along n0 (epilogue splits peer blocks) -> exchange ->
//            c2c columns (n1) -> c2r rows (n2) with 1/(n0 n1 n2).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/tffft.h"
#include "fourstep.cuh"
#include "stage1_fused.cuh"
#include "fourstep_tma.cuh"
#include "col_tma.cuh"
#include "col_wpc.cuh"
#include "col_wpc2.cuh"
#include "kernels.cuh"
#include "nccl.h"
#include <nvtx3/nvToolsExt.h>

using namespace tffft;

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
static thread_local std::string g_last_error;

static int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                 \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess)                                                             \
      return fail(TFFFT_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), \
                  __FILE__, __LINE__);                                                 \
  } while (0)

#define TRY(expr)               \
  do {                          \
    int _s = (expr);            \
    if (_s != TFFFT_OK) return _s; \
  } while (0)

// ---------------------------------------------------------------------------
// NCCL, loaded lazily so the library loads (and its symbols can be checked)
// on machines without a GPU or without NCCL.
// ---------------------------------------------------------------------------
struct NcclApi {
  bool loaded = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  // optional (NCCL >= 2.28): the COLLECTIVE pattern's single all-to-all
  ncclResult_t (*AlltoAll)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) =
      nullptr;
};

static NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = getenv("TFFFT_NCCL_LIBRARY");
    void* h = nullptr;
    if (env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);  // torch's copy
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.err = dlerror() ? dlerror() : "libnccl.so.2 not found";
      return;
    }
#define LOAD(name)                                                           \
  api.name = reinterpret_cast<decltype(api.name)>(dlsym(h, "nccl" #name));   \
  if (!api.name) { api.err = "missing symbol nccl" #name; return; }
    LOAD(GetUniqueId) LOAD(CommInitRank) LOAD(CommDestroy) LOAD(CommAbort) LOAD(CommGetAsyncError)
    LOAD(Send) LOAD(Recv) LOAD(GroupStart) LOAD(GroupEnd) LOAD(GetErrorString) LOAD(AllReduce)
#undef LOAD
    api.AlltoAll = reinterpret_cast<decltype(api.AlltoAll)>(dlsym(h, "ncclAlltoAll"));
    api.CommInitAll = reinterpret_cast<decltype(api.CommInitAll)>(dlsym(h, "ncclCommInitAll"));
    api.loaded = true;
  });
  return api;
}

#define NCCL_TRY(expr)                                                                   \
  do {                                                                                   \
    ncclResult_t _r = (expr);                                                            \
    if (_r != ncclSuccess)                                                               \
      return fail(TFFFT_ERR_TRANSPORT, "%s failed: %s", #expr, nccl().GetErrorString(_r)); \
  } while (0)

// ---------------------------------------------------------------------------
// local fabric: p ranks in one process on one device (transport.py:188-302)
// ---------------------------------------------------------------------------
struct LocalFabric {
  int p;
  int device;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  bool aborted = false;
  double timeout_s = 600.0;
  // per plan sequence number: every rank's exchange buffers and events, per
  // buffer set (a batched plan at p > 1 pipelines two sets)
  struct Slot {
    std::vector<void*> staging[2], landing[2];
    std::vector<cudaEvent_t> ready[2], done[2];
  };
  // a deque: slot(seq) may grow it while other ranks hold references to
  // earlier slots (growing a deque at the end keeps references valid)
  std::deque<Slot> slots;
  std::atomic<int> refs{0};

  // every rank's exchange events: owned by the fabric, destroyed with it, so a
  // rank that destroys its plan early never frees an event a slower peer is
  // still about to wait on
  std::vector<cudaEvent_t> events;

  explicit LocalFabric(int p_, int dev) : p(p_), device(dev) {}
  ~LocalFabric() {
    for (cudaEvent_t e : events) cudaEventDestroy(e);
  }

  // generation barrier with abort and timeout (transport.py:225-233, 290-302)
  int barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) return fail(TFFFT_ERR_TRANSPORT, "fabric aborted");
    uint64_t gen = generation;
    if (++arrived == p) {
      arrived = 0;
      ++generation;
      cv.notify_all();
      return TFFFT_OK;
    }
    bool ok = cv.wait_for(lk, std::chrono::duration<double>(timeout_s),
                          [&] { return generation != gen || aborted; });
    if (aborted) return fail(TFFFT_ERR_TRANSPORT, "fabric aborted while waiting at barrier");
    if (!ok) {
      aborted = true;
      cv.notify_all();
      return fail(TFFFT_ERR_TRANSPORT, "barrier timed out after %.0f s (a rank did not arrive)", timeout_s);
    }
    return TFFFT_OK;
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    aborted = true;
    cv.notify_all();
  }
  // publish this rank's buffers / events of one set (under the lock)
  void publish(int seq, int rank, int set, void* stg, void* lnd, cudaEvent_t rdy, cudaEvent_t dn) {
    std::lock_guard<std::mutex> lk(mu);
    events.push_back(rdy);
    events.push_back(dn);
    if ((int)slots.size() <= seq) slots.resize(seq + 1);
    Slot& s = slots[seq];
    if ((int)s.staging[set].size() != p) {
      s.staging[set].assign(p, nullptr);
      s.landing[set].assign(p, nullptr);
      s.ready[set].assign(p, nullptr);
      s.done[set].assign(p, nullptr);
    }
    s.staging[set][rank] = stg;
    s.landing[set][rank] = lnd;
    s.ready[set][rank] = rdy;
    s.done[set][rank] = dn;
  }
  // copy every rank's entries of one set out (under the lock; call after a barrier)
  void collect(int seq, int set, std::vector<void*>& stg, std::vector<void*>& lnd, std::vector<cudaEvent_t>& rdy,
               std::vector<cudaEvent_t>& dn) {
    std::lock_guard<std::mutex> lk(mu);
    const Slot& s = slots[seq];
    stg = s.staging[set];
    lnd = s.landing[set];
    rdy = s.ready[set];
    dn = s.done[set];
  }
};

// transports of a communicator
enum CommKind { COMM_LOCAL = 0, COMM_NCCL = 1, COMM_IPC = 2 };

struct tffft_comm_s {
  int p = 1, rank = 0, device = 0;
  int kind = COMM_LOCAL;
  bool is_nccl = false;  // kind == COMM_NCCL
  ncclComm_t nccl = nullptr;
  std::shared_ptr<LocalFabric> fabric;  // COMM_LOCAL
  tffft_barrier_fn barrier_fn = nullptr;  // COMM_IPC: the caller's host barrier
  void* barrier_ctx = nullptr;
  bool aborted = false;
  int plan_seq = 0;
  int barrier() {  // host barrier of the fabric kinds (local, IPC)
    if (kind == COMM_LOCAL) return fabric->barrier();
    if (aborted) return fail(TFFFT_ERR_TRANSPORT, "communicator aborted");
    if (!barrier_fn) return fail(TFFFT_ERR_TRANSPORT, "IPC communicator without a barrier");
    if (barrier_fn(barrier_ctx) != 0) {
      aborted = true;
      return fail(TFFFT_ERR_TRANSPORT, "IPC communicator: the host barrier failed");
    }
    return TFFFT_OK;
  }
};

// ---------------------------------------------------------------------------
// plans
// ---------------------------------------------------------------------------
struct StageEvents {
  cudaEvent_t e[4] = {nullptr, nullptr, nullptr, nullptr};
  bool forward = true;
  bool pending = false;  // recorded, not yet folded into the plan's stage totals
};
// events are created once (set_timing) and reused round robin, so no event is
// created inside a timed region
constexpr int kEventRing = 128;

// One set of exchange buffers (p > 1).  Band q of every buffer is the
// (n0/p, n1/p, n2c) block [q][i][j][k]; a batched plan pipelines two sets
// (component c uses set c % 2) so component c's exchange overlaps component
// c+1's stage 1.
struct BufSet {
  void* staging = nullptr;    // outgoing bands, staging[q] for rank q (pull / send-recv transports)
  void* landing = nullptr;    // incoming bands, landing[s] from rank s; landing[rank] = the self band
  void** band_dst = nullptr;  // device: destination block of each outgoing band (p pointers)
  std::vector<void*> band_dst_h;  // host copy (the TMA column kernel's store table)
  void** pull_ptrs = nullptr; // fabric pull: device list of (src, dst) per peer
  // fabric transports (local, IPC): every rank's buffers and events of this set
  std::vector<void*> peer_staging, peer_landing;
  std::vector<cudaEvent_t> ready, done;  // [q]: rank q's "staging written" / "landing consumed"
  bool own_events = false;
};

struct tffft_plan_s {
  tffft_comm_t comm = nullptr;
  int n0 = 0, n1 = 0, n2 = 0, p = 1, rank = 0, dtype = TFFFT_F64, pattern = TFFFT_PAIRWISE;
  int L0 = 0, L1 = 0, L2h = 0;
  int n0p = 0, n1p = 0, n2c = 0;
  size_t esz = 16;  // complex element bytes
  int batch = 1;    // fields per forward / inverse call, back to back in memory
  int seq = 0;
  BufSet bs[2];
  int nsets = 1;
  int cur = 0;               // the set the stage launchers address
  int xchunks = 1;           // plane chunks of the chunked exchange, both directions (1 = one exchange per call)
  bool peer_stores = false;  // epilogues store peer bands straight into the peers' landing buffers
  bool peer_stores_wanted = false;  // NCCL communicator: peer stores once the peers' landing buffers are attached
  std::vector<void*> ipc_opened;    // peer mappings opened through CUDA IPC (closed at destroy)
  std::vector<cudaEvent_t> ipc_events;  // peer events opened through CUDA IPC
  int* barrier_word = nullptr;      // NCCL + peer stores: one-int all-reduce used as a stream-ordered barrier
  bool ipc_attached = false;        // IPC communicator: peers' buffers mapped
  // batched p > 1: exchange stream and the pipeline's hand-off events per set
  cudaStream_t xstream = nullptr;
  cudaEvent_t ev_s1[2] = {nullptr, nullptr}, ev_x[2] = {nullptr, nullptr}, ev_s3[2] = {nullptr, nullptr};
  void* tw0 = nullptr;
  void* tw1 = nullptr;
  void* tw2 = nullptr;   // row pass tables (c2r, fused stage 1)
  void* tw2r = nullptr;  // row pass tables in the r2c kernel's schedule
  void* tw2c = nullptr;  // row pass tables in the c2r kernel's schedule
  void* tw2post = nullptr;
  void* tw10 = nullptr;    // 2 x 1024 column kernel (col_wpc2.cuh): the 1024-point pass tables ...
  void* twh11 = nullptr;   // ... and exp(-2 pi i k / 2048), k < 1024
  unsigned long long* stats = nullptr;  // per plane [m2, edge, residue] (ordered doubles), batch * n0p planes
  double* row_stats = nullptr;          // per row records of the c2r kernel
  // stage-3 four-step (fourstep.cuh): L2-resident scratch ring, counters, tables
  int fs_la = 0, fs_G = 0, fs_groups = 0;
  void* fs_scratch = nullptr;
  unsigned* fs_counters = nullptr;
  void* fs_twA = nullptr;
  void* fs_twB = nullptr;
  void* fs_twN = nullptr;
  // exchange strategy (exchange.py:48-50): 0 STRIDED (transpose-free), 1 TRANSPOSE
  int strategy = 0;
  // fused stage 1 (stage1_fused.cuh)
  bool s1_fused = false;
  unsigned* s1_counters = nullptr;
  unsigned long long* col_ticket = nullptr;  // dynamic tile counter of the column kernel (TFFFT_COL_TICKET)
  int tma_cols = 0;      // TMA-fed column passes: 0 off, 1 every supported pass, 2 the measured winners
  size_t workspace = 0;
  bool timing = false;
  std::vector<StageEvents> events;  // kEventRing slots while timing is enabled
  int event_next = 0;
  double stage_ms[3] = {0.0, 0.0, 0.0};
  uint64_t counters[3] = {0, 0, 0};
  uint64_t launches = 0;
  cudaStream_t last_inverse_stream = nullptr;
  bool inverse_ran = false;
  bool deferred_check = false;          // fold every inverse's Hermitian check on the device
  unsigned long long* check_acc = nullptr;  // consistency_fold_kernel accumulator (4 words)
  uint64_t deferred_calls = 0;
};

static bool pow2(long long n) { return n >= 1 && (n & (n - 1)) == 0; }
static int ilog2(long long n) { int l = 0; while ((1LL << l) < n) ++l; return l; }

// pass twiddle tables for length 2^L (see fft_engine.cuh): block for pass p>=1
// holds exp(-2 pi i k / (Ns R)) at [k], k < Ns
static std::vector<double> pass_table(int L, int mb = 0) {
  std::vector<double> t;
  const int P = num_passes(L, mb);
  t.assign(2 * (size_t)std::max(tw_total(L, mb), 1), 0.0);
  for (int p = 1; p < P; ++p) {
    const long long R = 1LL << pass_bits(L, p, mb), NS = 1LL << ns_bits(L, p, mb), M = NS * R;
    const size_t off = tw_offset(L, p, mb);
    for (long long k = 0; k < NS; ++k) {
      const long double a = -2.0L * 3.141592653589793238462643383279502884L * (long double)k / (long double)M;
      t[2 * (off + k)] = (double)cosl(a);
      t[2 * (off + k) + 1] = (double)sinl(a);
    }
  }
  return t;
}

// exp(-2 pi i t / n) for t < n (four-step twiddles)
static std::vector<double> full_table(int n) {
  std::vector<double> t(2 * (size_t)n, 0.0);
  for (int k = 0; k < n; ++k) {
    const long double a = -2.0L * 3.141592653589793238462643383279502884L * k / (long double)n;
    t[2 * k] = (double)cosl(a);
    t[2 * k + 1] = (double)sinl(a);
  }
  return t;
}

// exp(-2 pi i k / n) for k < n/2 (reference twiddle convention, kernels.py:76-81)
static std::vector<double> post_table(int n) {
  std::vector<double> t(2 * (size_t)std::max(n / 2, 1), 0.0);
  for (int k = 0; k < n / 2; ++k) {
    const long double a = -2.0L * 3.141592653589793238462643383279502884L * k / (long double)n;
    t[2 * k] = (double)cosl(a);
    t[2 * k + 1] = (double)sinl(a);
  }
  return t;
}

static int upload_table(const std::vector<double>& t, int dtype, void** dev, size_t* bytes) {
  const size_t n = t.size();
  if (dtype == TFFFT_F64) {
    CUDA_TRY(cudaMalloc(dev, n * sizeof(double)));
    CUDA_TRY(cudaMemcpy(*dev, t.data(), n * sizeof(double), cudaMemcpyHostToDevice));
    *bytes += n * sizeof(double);
  } else {
    std::vector<float> f(n);
    for (size_t i = 0; i < n; ++i) f[i] = (float)t[i];
    CUDA_TRY(cudaMalloc(dev, n * sizeof(float)));
    CUDA_TRY(cudaMemcpy(*dev, f.data(), n * sizeof(float), cudaMemcpyHostToDevice));
    *bytes += n * sizeof(float);
  }
  return TFFFT_OK;
}

// ---------------------------------------------------------------------------
// kernel launch helpers
// ---------------------------------------------------------------------------
// shortest column (log2) that takes the ticket tile order: measured gains for
// the cp.async column kernel from 1024 points (512: 5% slower), for the TMA
// column kernel from 512 points (profiles/r01s11/tma_512.txt)
static int ticket_min_log(bool tma) {
  static const int v = [] {
    const char* e = getenv("TFFFT_TICKET_MINL");
    return e ? atoi(e) : 0;
  }();
  return v > 0 ? v : (tma ? 9 : 10);
}

static cudaError_t col_launch(tffft_plan_t pl, int L, bool inv, bool two, int rd, bool wide, const ColParams& prm0,
                              cudaStream_t s) {
  pl->launches++;
  ColParams prm = prm0;
  // dynamic tile order (1024^3 f64 stage 3 3.69 -> 3.25 ms)
  if (TFFFT_COL_TICKET && L >= ticket_min_log(false)) {
    prm.ticket = pl->col_ticket;
    (void)cudaMemsetAsync(pl->col_ticket, 0, sizeof(unsigned long long), s);
  }
#if TFFFT_PROBES
  {
    static const char* probe = getenv("TFFFT_PROBE_COL");
    prm.probe = probe ? atoi(probe) : 0;
  }
#endif
  return pl->dtype == TFFFT_F64 ? launch_col_fft<double>(L, inv, two, rd, wide, prm, s)
                                : launch_col_fft<float>(L, inv, two, rd, wide, prm, s);
}
static cudaError_t r2c_launch(tffft_plan_t pl, const RowParams& prm, cudaStream_t s) {
  pl->launches++;
  RowParams q = prm;
  q.tw = pl->tw2r;  // the r2c kernel's own radix schedule (r2c_radix_bits)
  return pl->dtype == TFFFT_F64 ? launch_r2c_rows<double>(pl->L2h, q, s)
                                : launch_r2c_rows<float>(pl->L2h, q, s);
}
static cudaError_t c2r_launch(tffft_plan_t pl, const RowParams& prm, cudaStream_t s) {
  pl->launches++;
  RowParams q = prm;
  q.tw = pl->tw2c;  // the c2r kernel's own radix schedule (c2r_radix_bits)
  return pl->dtype == TFFFT_F64 ? launch_c2r_rows<double>(pl->L2h, q, s)
                                : launch_c2r_rows<float>(pl->L2h, q, s);
}

// local-fabric pull: chunk c copies `words` W-sized words from ptrs[2c] to ptrs[2c+1]
template <typename W>
__global__ void pull_chunks_kernel(void* const* __restrict__ ptrs, long long off, long long words, int nchunks) {
  const int c = blockIdx.y;
  if (c >= nchunks) return;
  const W* __restrict__ src = reinterpret_cast<const W*>(ptrs[2 * c]) + off;
  W* __restrict__ dst = reinterpret_cast<W*>(ptrs[2 * c + 1]) + off;
  for (long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x; w < words;
       w += (long long)gridDim.x * blockDim.x)
    dst[w] = src[w];
}

// TRANSPOSE strategy pack / unpack (exchange.py:145-192): a permutation of whole
// k-rows (n2c contiguous complex values).  Row (a, b, c) of an A x B x C
// iteration moves from src + a*sa + b*sb + c*sc to dst + a*da + b*db + c*dc
// (element units); with `self` >= 0, block a == self is read from src_self
// instead (the rank's own block never crosses the exchange).  One warp per row.
struct PermuteParams {
  const void* src;
  const void* src_self;
  void* dst;
  int A, B, C, self;
  long long sa, sb, sc, da, db, dc;
  long long row_words;  // words of W per row
};

template <typename W>
__global__ void permute_rows_kernel(const PermuteParams p, int esz) {
  const long long warps = (long long)gridDim.x * (blockDim.x / 32);
  const long long total = (long long)p.A * p.B * p.C;
  for (long long r = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; r < total; r += warps) {
    const int c = (int)(r % p.C), b = (int)((r / p.C) % p.B), a = (int)(r / ((long long)p.C * p.B));
    const char* sbase = static_cast<const char*>(a == p.self ? p.src_self : p.src);
    const W* s = reinterpret_cast<const W*>(sbase + (a * p.sa + b * p.sb + c * p.sc) * esz);
    W* d = reinterpret_cast<W*>(static_cast<char*>(p.dst) + (a * p.da + b * p.db + c * p.dc) * esz);
    for (long long w = threadIdx.x % 32; w < p.row_words; w += 32) d[w] = s[w];
  }
}

// ---------------------------------------------------------------------------
// stage launchers
// ---------------------------------------------------------------------------
static int columns_tma(tffft_plan_t pl, int L, bool inv, bool wide, void* base, long long cols, long long ngrp,
                       long long rstride, long long gstride, const void* tw, cudaStream_t s, bool* done);

struct TwoLevelJob {
  bool wide;  // stage 3 / 3' (128-byte row segments) or stage 1b / 1b' (narrow CTA shape)
  const void* ld_base;
  long long cols, ngrp;
  long long ld_in_rows, ld_blocks, ld_in, ld_out, ld_g;
  void* st_base;
  std::vector<void*> st_tab;
  long long st_rows, st_in, st_g;
};
static int columns_tma_two(tffft_plan_t pl, int L, bool inv, const TwoLevelJob& j, const void* tw, cudaStream_t s,
                           bool* done);

// stage 1b / 1b': c2c along n1 of every (plane i, bin k) column of `nplanes`
// planes starting at `spec` (a batched p = 1 plan passes all batch * n0p planes)
// (plane0: the first plane's index within the field, for the band redirects)
static int stage1_columns(tffft_plan_t pl, void* spec, bool inv, cudaStream_t s, int nplanes, int plane0 = 0) {
  ColParams c{};
  c.data = spec;
  c.tw = pl->tw1;
  c.ncols = (long long)nplanes * pl->n2c;
  c.cpb = pl->n2c;
  c.grp_stride = (long long)pl->n1 * pl->n2c;
  c.ic_shift = 30;
  c.inner_stride = pl->n2c;
  c.block_stride = 0;
  c.band_shift = ilog2(pl->n1p);
  c.self_band = pl->rank;
  c.staging = nullptr;
  int rd = 0;
  if (pl->p > 1 && pl->strategy == 0) {
    // forward epilogue: band q -> band_dst[q] for EVERY q (the self band goes to
    // landing[rank], peers to staging[q] or straight to rank q's landing);
    // inverse: every band is read from landing[q][i][j][k] (the exchange output)
    const BufSet& B = pl->bs[pl->cur];
    c.staging = B.landing;
    c.band_dst = B.band_dst;
    c.self_band = -1;
    rd = inv ? 2 : 1;
    c.stg_band = (long long)pl->n0p * pl->n1p * pl->n2c;
    c.stg_within = pl->n2c;
    c.stg_grp = (long long)pl->n1p * pl->n2c;
    c.stg_base = (long long)plane0 * c.stg_grp;
  }
#if TFFFT_PROBES
  {  // profiling probe: every plane aliases plane 0 (same work, L2-resident footprint)
    static const char* probe = getenv("TFFFT_PROBE_ALIAS");
    if (probe && atoi(probe)) c.grp_stride = 0;
  }
#endif
  if (rd == 0 && c.grp_stride != 0) {
    bool done = false;
    // stage 1b: rows n2c elements apart, the narrow CTA shape (two per SM)
    TRY(columns_tma(pl, pl->L1, inv, false, c.data, pl->n2c, nplanes, pl->n2c, (long long)pl->n1 * pl->n2c,
                    pl->tw1, s, &done));
    if (done) return TFFFT_OK;
  } else if (rd != 0) {
    // p > 1 through the TMA column kernel: forward = plane loads + band
    // write-redirect; inverse = landing[q][i][j][k] loads + in-place stores
    const BufSet& B = pl->bs[pl->cur];
    const long long n1p = pl->n1p, n2c = pl->n2c, band = (long long)pl->n0p * n1p * n2c;
    TwoLevelJob j{};
    j.wide = false;
    j.cols = n2c;
    j.ngrp = nplanes;
    if (!inv) {
      j.ld_base = spec; j.ld_in_rows = pl->n1; j.ld_blocks = 1; j.ld_in = n2c; j.ld_g = (long long)pl->n1 * n2c;
      for (void* d : B.band_dst_h) j.st_tab.push_back(static_cast<char*>(d) + (size_t)plane0 * n1p * n2c * pl->esz);
      j.st_rows = n1p; j.st_in = n2c; j.st_g = n1p * n2c;
    } else {
      j.ld_base = static_cast<char*>(B.landing) + (size_t)plane0 * n1p * n2c * pl->esz;
      j.ld_in_rows = n1p; j.ld_blocks = pl->p; j.ld_in = n2c; j.ld_out = band;
      j.ld_g = n1p * n2c;
      j.st_base = spec; j.st_rows = pl->n1; j.st_in = n2c; j.st_g = (long long)pl->n1 * n2c;
    }
    bool done = false;
    TRY(columns_tma_two(pl, pl->L1, inv, j, pl->tw1, s, &done));
    if (done) return TFFFT_OK;
  }
  CUDA_TRY(col_launch(pl, pl->L1, inv, false, rd, false, c, s));
  return TFFFT_OK;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (EncodeTiledFn) nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// rank-r map over `base` in real elements of the plan's precision; dims/strides innermost first
static int make_map(tffft_plan_t pl, CUtensorMap* m, void* base, int rank, const cuuint64_t* dims,
                    const cuuint64_t* strides_bytes, const cuuint32_t* box,
                    CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_NONE) {
  EncodeTiledFn fn = encode_tiled();
  if (!fn) return fail(TFFFT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  const CUresult r = fn(m, pl->dtype == TFFFT_F64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                        (cuuint32_t)rank, base, dims, strides_bytes, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swz, promo,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(TFFFT_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return TFFFT_OK;
}

// Column pass through the TMA-fed column kernel (col_tma.cuh): `ngrp` groups
// of `cols` contiguous columns, column elements `rstride` apart, groups
// `gstride` apart (elements).  Sets *done = false when the shape has no TMA
// path (the caller falls back to col_fft_kernel).
// auto mode (tma_cols == 2): every supported column pass -- measured faster
// than the cp.async kernel for both precisions at 512 and 1024 points
// (profiles/r01s10/tma_f64_ticket.txt, r01s11/tma_512.txt)
static bool tma_cols_enabled(tffft_plan_t pl, int L) {
  (void)L;
  return pl->tma_cols != 0;
}

// Warp-per-column kernel (col_wpc.cuh) for the 1024-point column passes at p = 1.
// TFFFT_WPC: 0 never, 1 every pass, 2 (default) the stage-1b / 1b' passes, and
// for float32 the stage-3 / 3' passes too (3.41 -> 3.28 ms per pair live).  The
// float32 stage-1b rows of an odd n2c (8 bytes off 16-byte alignment on odd rows)
// stay on col_tma_kernel: a swizzled box must start on a 16-byte boundary (a box
// started one complex in raised "illegal instruction" on the B200).
// Measured on one box (profiles/r02s4/wpc_ab.txt): stage 1b 2.87 -> 2.57 ms per
// float64 1024^3 launch; stage 3 (rows 8.4 MB apart) ties at 2.99-3.00 ms in
// isolation and is slightly slower live, so it keeps col_tma_kernel.
static int wpc_cols_mode() {
  const char* e = getenv("TFFFT_WPC");
  return e ? atoi(e) : 2;
}

// L2 promotion of the column-pass load maps (TFFFT_TMA_PROMO: 0 none (default), 1 = 64, 2 = 128, 3 = 256 bytes;
// applied to the wide passes only, whose 128-byte row visits sit in 256-byte-aligned pairs)
static CUtensorMapL2promotion col_promo(bool wide) {
  static const int v = [] {
    const char* e = getenv("TFFFT_TMA_PROMO");
    return e ? atoi(e) : 0;
  }();
  if (!wide) return CU_TENSOR_MAP_L2_PROMOTION_NONE;
  return v == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                : v == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                         : v == 3 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE;
}

// Column pass through the warp-per-column kernel: loads as columns_tma_two
// describes them (3D map, or 4D over the landing bands), stores uniform
// (st_tab empty: row r of the column at st_base + r * st_in) or one map per
// destination block (st_tab[r / st_rows], row r mod st_rows).  *done = false
// when the mode, the shape or an alignment rules it out.
static int columns_wpc(tffft_plan_t pl, int L, bool inv, const TwoLevelJob& j, const void* tw, cudaStream_t s,
                       bool* done) {
  *done = false;
  const int mode = wpc_cols_mode();
  const bool x2 = L == 11;  // 2048 points as 2 x 1024 (col_wpc2.cuh): every pass, col_fft_kernel is far slower there
  if (!(mode == 1 || (mode == 2 && (!j.wide || pl->dtype == TFFFT_F32 || x2 || L == 9))) || !col_wpc_supported(L))
    return TFFFT_OK;
  if (x2 && (!pl->tw10 || !pl->twh11 || j.ld_in_rows % 2)) return TFFFT_OK;
  const long long esz = (long long)pl->esz, n = 1LL << L;
  const long long B = pl->dtype == TFFFT_F64 ? col_wpc_width<double>(L) : col_wpc_width<float>(L);
  const bool two = !j.st_tab.empty();
  if (B <= 0 || j.ld_in_rows * j.ld_blocks != n || (int)j.st_tab.size() > kWpcMaps) return TFFFT_OK;
  // a TMA store writes whole 16-byte chunks: an odd number of float32 columns would spill 8 bytes past the
  // last column of every row (DESIGN finding 34)
  if ((j.cols * esz) % 16) return TFFFT_OK;
  if ((j.ld_in * esz) % 16 || (j.ld_blocks > 1 && (j.ld_out * esz) % 16) || (j.ngrp > 1 && (j.ld_g * esz) % 16) ||
      reinterpret_cast<uintptr_t>(j.ld_base) % 16 || (j.st_in * esz) % 16 || (j.ngrp > 1 && (j.st_g * esz) % 16))
    return TFFFT_OK;
  // 2 x 1024: loads by row parity, sub-boxes of half rows within a block
  const long long lbrows = std::min<long long>(256, x2 ? j.ld_in_rows / 2 : j.ld_in_rows);
  const long long srows_blk = two ? j.st_rows : n;
  // rows per output round: a quarter of the column (2 x 1024: 128-row rounds)
  const long long sbrows = std::min<long long>(x2 ? 128 : n / 4, srows_blk);
  const cuuint32_t boxw = (cuuint32_t)(256 / esz);  // reals in a 128-byte sub-box row
  // sub-boxes start on 1024-byte (8-row) boundaries of the swizzled landing boxes
  if (lbrows < 8 || sbrows < 8 || (two && srows_blk * (long long)j.st_tab.size() != n)) return TFFFT_OK;
  for (void* d : j.st_tab)
    if (reinterpret_cast<uintptr_t>(d) % 16) return TFFFT_OK;
  if (!two && reinterpret_cast<uintptr_t>(j.st_base) % 16) return TFFFT_OK;
  WpcMaps maps;
  if (x2 && j.ld_blocks == 1) {  // (cols, parity, half rows, groups)
    cuuint64_t d[4] = {(cuuint64_t)(2 * j.cols), 2, (cuuint64_t)(n / 2), (cuuint64_t)j.ngrp};
    cuuint64_t st[3] = {(cuuint64_t)(j.ld_in * esz), (cuuint64_t)(2 * j.ld_in * esz),
                        (cuuint64_t)(j.ngrp > 1 ? j.ld_g * esz : n * j.ld_in * esz)};
    cuuint32_t box[4] = {boxw, 1, 256, 1};
    TRY(make_map(pl, &maps.ld, const_cast<void*>(j.ld_base), 4, d, st, box, col_promo(j.wide),
                 CU_TENSOR_MAP_SWIZZLE_128B));
  } else if (x2) {  // (cols, parity, half rows within a block, blocks, groups)
    cuuint64_t d[5] = {(cuuint64_t)(2 * j.cols), 2, (cuuint64_t)(j.ld_in_rows / 2), (cuuint64_t)j.ld_blocks,
                       (cuuint64_t)j.ngrp};
    cuuint64_t st[4] = {(cuuint64_t)(j.ld_in * esz), (cuuint64_t)(2 * j.ld_in * esz), (cuuint64_t)(j.ld_out * esz),
                        (cuuint64_t)(j.ngrp > 1 ? j.ld_g * esz : j.ld_blocks * j.ld_out * esz)};
    cuuint32_t box[5] = {boxw, 1, (cuuint32_t)lbrows, 1, 1};
    TRY(make_map(pl, &maps.ld, const_cast<void*>(j.ld_base), 5, d, st, box, col_promo(j.wide),
                 CU_TENSOR_MAP_SWIZZLE_128B));
  } else if (j.ld_blocks == 1) {
    cuuint64_t d[3] = {(cuuint64_t)(2 * j.cols), (cuuint64_t)n, (cuuint64_t)j.ngrp};
    cuuint64_t st[2] = {(cuuint64_t)(j.ld_in * esz), (cuuint64_t)(j.ngrp > 1 ? j.ld_g * esz : n * j.ld_in * esz)};
    cuuint32_t box[3] = {boxw, 256, 1};
    TRY(make_map(pl, &maps.ld, const_cast<void*>(j.ld_base), 3, d, st, box, col_promo(j.wide),
                 CU_TENSOR_MAP_SWIZZLE_128B));
  } else {
    cuuint64_t d[4] = {(cuuint64_t)(2 * j.cols), (cuuint64_t)j.ld_in_rows, (cuuint64_t)j.ld_blocks,
                       (cuuint64_t)j.ngrp};
    cuuint64_t st[3] = {(cuuint64_t)(j.ld_in * esz), (cuuint64_t)(j.ld_out * esz),
                        (cuuint64_t)(j.ngrp > 1 ? j.ld_g * esz : j.ld_blocks * j.ld_out * esz)};
    cuuint32_t box[4] = {boxw, (cuuint32_t)lbrows, 1, 1};
    TRY(make_map(pl, &maps.ld, const_cast<void*>(j.ld_base), 4, d, st, box, col_promo(j.wide),
                 CU_TENSOR_MAP_SWIZZLE_128B));
  }
  const int nst = two ? (int)j.st_tab.size() : 1;
  for (int q = 0; q < nst; ++q) {
    cuuint64_t d[3] = {(cuuint64_t)(2 * j.cols), (cuuint64_t)srows_blk, (cuuint64_t)j.ngrp};
    cuuint64_t st[2] = {(cuuint64_t)(j.st_in * esz),
                        (cuuint64_t)(j.ngrp > 1 ? j.st_g * esz : srows_blk * j.st_in * esz)};
    cuuint32_t box[3] = {boxw, (cuuint32_t)sbrows, 1};
    TRY(make_map(pl, &maps.st[q], two ? j.st_tab[q] : j.st_base, 3, d, st, box, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                 CU_TENSOR_MAP_SWIZZLE_128B));
  }
  for (int q = nst; q < kWpcMaps; ++q) maps.st[q] = maps.st[0];
  WpcParams w{};
  w.tw = x2 ? pl->tw10 : tw;
  w.tw2 = pl->twh11;
  w.tpg = (int)((j.cols + B - 1) / B);
  w.ntiles = (long long)w.tpg * j.ngrp;
  {
    static const char* ef = getenv("TFFFT_TMA_EF");
    w.evict_first = ef ? atoi(ef) : ((j.ld_in * esz) % 128 == 0);
  }
  w.load4 = j.ld_blocks > 1;
  w.lin_shift = ilog2(j.ld_in_rows);
  w.lbrows = (int)lbrows;
  w.nst = nst;
  w.sst_shift = ilog2(srows_blk);
  w.sbrows = (int)sbrows;
  if (TFFFT_COL_TICKET && L >= ticket_min_log(true)) {
    w.ticket = pl->col_ticket;
    CUDA_TRY(cudaMemsetAsync(pl->col_ticket, 0, sizeof(unsigned long long), s));
  }
  pl->launches++;
  CUDA_TRY(pl->dtype == TFFFT_F64 ? launch_col_wpc<double>(L, inv, maps, w, s)
                                  : launch_col_wpc<float>(L, inv, maps, w, s));
  *done = true;
  return TFFFT_OK;
}

static int columns_tma(tffft_plan_t pl, int L, bool inv, bool wide, void* base, long long cols, long long ngrp,
                       long long rstride, long long gstride, const void* tw, cudaStream_t s, bool* done) {
  *done = false;
  const long long esz = (long long)pl->esz;
  const long long rbytes = rstride * esz;
  // rows 16-byte aligned (one map), or 8 bytes off on odd rows only (float32
  // stage 1b, n2c odd: 4104-byte rows): even and odd rows through two maps
  const bool parity = rbytes % 16 != 0;
  if (!tma_cols_enabled(pl, L)) return TFFFT_OK;
  const long long n = 1LL << L;
  if (!parity) {  // warp-per-column kernel (col_wpc.cuh, col_wpc2.cuh) where it applies
    TwoLevelJob j{};
    j.wide = wide;
    j.ld_base = base; j.cols = cols; j.ngrp = ngrp;
    j.ld_in_rows = n; j.ld_blocks = 1; j.ld_in = rstride; j.ld_out = 0; j.ld_g = gstride;
    j.st_base = base; j.st_rows = n; j.st_in = rstride; j.st_g = gstride;
    TRY(columns_wpc(pl, L, inv, j, tw, s, done));
    if (*done) return TFFFT_OK;
  }
  if (!col_tma_supported(L) || (parity && (2 * rbytes) % 16) || (ngrp > 1 && (gstride * esz) % 16) ||
      reinterpret_cast<uintptr_t>(base) % 16)
    return TFFFT_OK;
  const long long B = pl->dtype == TFFFT_F64 ? col_tma_width<double>(L, wide) : col_tma_width<float>(L, wide);
  if (B <= 0) return TFFFT_OK;
  CUtensorMap map, map_odd;
  const long long gbytes = ngrp > 1 ? gstride * esz : n * rbytes;
  if (!parity) {
    cuuint64_t d[3] = {(cuuint64_t)(2 * cols), (cuuint64_t)n, (cuuint64_t)ngrp};
    cuuint64_t st[2] = {(cuuint64_t)rbytes, (cuuint64_t)gbytes};
    cuuint32_t box[3] = {(cuuint32_t)(2 * B), (cuuint32_t)std::min<long long>(n, 256), 1};
    TRY(make_map(pl, &map, base, 3, d, st, box, col_promo(wide)));
    map_odd = map;
  } else {
    // odd rows miss 16-byte alignment by `mis` = one complex: their boxes start
    // one complex early (aligned) and are two complex wider (pitch B + 2)
    const long long mis = rbytes % 16;
    if (mis != esz) return TFFFT_OK;
    cuuint64_t de[3] = {(cuuint64_t)(2 * cols), (cuuint64_t)(n / 2), (cuuint64_t)ngrp};
    cuuint64_t dodd[3] = {(cuuint64_t)(2 * cols + 2), (cuuint64_t)(n / 2), (cuuint64_t)ngrp};
    cuuint64_t st[2] = {(cuuint64_t)(2 * rbytes), (cuuint64_t)gbytes};
    cuuint32_t box[3] = {(cuuint32_t)(2 * B), (cuuint32_t)std::min<long long>(n / 2, 256), 1};
    cuuint32_t boxo[3] = {(cuuint32_t)(2 * B + 4), (cuuint32_t)std::min<long long>(n / 2, 256), 1};
    TRY(make_map(pl, &map, base, 3, de, st, box, CU_TENSOR_MAP_L2_PROMOTION_NONE));
    TRY(make_map(pl, &map_odd, static_cast<char*>(base) + rbytes - mis, 3, dodd, st, boxo,
                 CU_TENSOR_MAP_L2_PROMOTION_NONE));
  }
  TmaColParams w{};
  w.data = base;
  w.tw = tw;
  w.tpg = (int)((cols + B - 1) / B);
  w.ntiles = (long long)w.tpg * ngrp;
  w.cols = (int)cols;
  w.rstride = rstride;
  w.gstride = gstride;
  w.parity = parity;
  if (TFFFT_COL_TICKET && L >= ticket_min_log(true)) {
    w.ticket = pl->col_ticket;
    CUDA_TRY(cudaMemsetAsync(pl->col_ticket, 0, sizeof(unsigned long long), s));
  }
  {
    static const char* ef = getenv("TFFFT_TMA_EF");
    w.evict_first = ef ? atoi(ef) : (rbytes % 128 == 0);
    // half of each output tile through TMA stores (in place, single map)
    static const char* ts = getenv("TFFFT_TMA_STORE");
    w.tma_store = (!parity && ts && atoi(ts) != 0) ? 1 : 0;
  }
  pl->launches++;
  const cudaError_t e = pl->dtype == TFFFT_F64 ? launch_col_tma<double>(L, inv, wide, false, map, map_odd, w, s)
                                               : launch_col_tma<float>(L, inv, wide, false, map, map_odd, w, s);
  CUDA_TRY(e);
  *done = true;
  return TFFFT_OK;
}

// Two-level column pass at p > 1 through the TMA column kernel (col_tma.cuh,
// TWO / 4D load mode).  Loads: a 3D map (2*cols, n, groups) with rows
// `ld_in` apart and groups `ld_g` apart (ld_blocks == 1), or a 4D map (2*cols,
// ld_in_rows, ld_blocks, groups) with rows `ld_in` apart, blocks `ld_out`
// apart and groups `ld_g` apart.  Stores: uniform (st_tab empty: element r of
// column c of group g at st_base + g * st_g + c + r * st_in) or through the
// block table st_tab (element r at st_tab[r >> log2(st_rows)] + g * st_g + c +
// (r mod st_rows) * st_in).  All in complex elements.  *done = false when the
// shape or the alignment has no TMA path.


static int columns_tma_two(tffft_plan_t pl, int L, bool inv, const TwoLevelJob& j, const void* tw, cudaStream_t s,
                           bool* done) {
  *done = false;
  const long long esz = (long long)pl->esz, n = 1LL << L;
  const bool two = !j.st_tab.empty();
  if (!tma_cols_enabled(pl, L)) return TFFFT_OK;
  TRY(columns_wpc(pl, L, inv, j, tw, s, done));
  if (*done) return TFFFT_OK;
  if (!col_tma_supported(L) || (int)j.st_tab.size() > kTmaTab) return TFFFT_OK;
  if ((j.ld_in * esz) % 16 || (j.ld_blocks > 1 && (j.ld_out * esz) % 16) || (j.ngrp > 1 && (j.ld_g * esz) % 16) ||
      reinterpret_cast<uintptr_t>(j.ld_base) % 16)
    return TFFFT_OK;
  const long long B = pl->dtype == TFFFT_F64 ? col_tma_width<double>(L, j.wide) : col_tma_width<float>(L, j.wide);
  if (B <= 0 || j.ld_in_rows * j.ld_blocks != n) return TFFFT_OK;
  const long long brows = std::min<long long>(std::min<long long>(n, 256), j.ld_in_rows);
  CUtensorMap map;
  if (j.ld_blocks == 1) {
    cuuint64_t d[3] = {(cuuint64_t)(2 * j.cols), (cuuint64_t)n, (cuuint64_t)j.ngrp};
    cuuint64_t st[2] = {(cuuint64_t)(j.ld_in * esz), (cuuint64_t)(j.ngrp > 1 ? j.ld_g * esz : n * j.ld_in * esz)};
    cuuint32_t box[3] = {(cuuint32_t)(2 * B), (cuuint32_t)std::min<long long>(n, 256), 1};
    TRY(make_map(pl, &map, const_cast<void*>(j.ld_base), 3, d, st, box, CU_TENSOR_MAP_L2_PROMOTION_NONE));
  } else {
    cuuint64_t d[4] = {(cuuint64_t)(2 * j.cols), (cuuint64_t)j.ld_in_rows, (cuuint64_t)j.ld_blocks,
                       (cuuint64_t)j.ngrp};
    cuuint64_t st[3] = {(cuuint64_t)(j.ld_in * esz), (cuuint64_t)(j.ld_out * esz),
                        (cuuint64_t)(j.ngrp > 1 ? j.ld_g * esz : j.ld_blocks * j.ld_out * esz)};
    cuuint32_t box[4] = {(cuuint32_t)(2 * B), (cuuint32_t)brows, 1, 1};
    TRY(make_map(pl, &map, const_cast<void*>(j.ld_base), 4, d, st, box, CU_TENSOR_MAP_L2_PROMOTION_NONE));
  }
  TmaColParams w{};
  w.data = j.st_base;
  w.tw = tw;
  w.tpg = (int)((j.cols + B - 1) / B);
  w.ntiles = (long long)w.tpg * j.ngrp;
  w.cols = (int)j.cols;
  w.rstride = j.st_in;
  w.gstride = j.st_g;
  w.parity = 0;
  w.load4 = j.ld_blocks > 1;
  w.lin_shift = ilog2(j.ld_in_rows);
  w.brows = (int)brows;
  if (two) {
    w.sin_shift = ilog2(j.st_rows);
    w.sin_stride = j.st_in;
    w.sgstride = j.st_g;
    for (size_t q = 0; q < j.st_tab.size(); ++q) w.tab[q] = j.st_tab[q];
  }
  if (TFFFT_COL_TICKET && L >= ticket_min_log(true)) {
    w.ticket = pl->col_ticket;
    CUDA_TRY(cudaMemsetAsync(pl->col_ticket, 0, sizeof(unsigned long long), s));
  }
  w.evict_first = (j.ld_in * esz) % 128 == 0;
  pl->launches++;
  const cudaError_t e = pl->dtype == TFFFT_F64 ? launch_col_tma<double>(L, inv, j.wide, two, map, map, w, s)
                                               : launch_col_tma<float>(L, inv, j.wide, two, map, map, w, s);
  CUDA_TRY(e);
  *done = true;
  return TFFFT_OK;
}

// stage 3 at p = 1 through the TMA-fed four-step (fourstep_tma.cuh)
static int stage3_tma(tffft_plan_t pl, void* spec, bool inv, cudaStream_t s) {
  const int la = pl->fs_la, lb = pl->L0 - la;
  const long long NA = 1LL << la, NB = 1LL << lb, N = (long long)pl->n0;
  const long long W = 256 / (NA / 8);  // columns per task: 256 threads, NA / 8 threads per column
  const long long ncols = (long long)pl->n1 * pl->n2c;
  const long long esz = (long long)pl->esz, S1 = ncols * esz, G = pl->fs_G;
  CUtensorMap maps[4];
  {
    cuuint64_t d[3] = {(cuuint64_t)(2 * ncols), (cuuint64_t)NA, (cuuint64_t)NB};
    cuuint64_t st[2] = {(cuuint64_t)(NB * S1), (cuuint64_t)S1};
    cuuint32_t box[3] = {(cuuint32_t)(2 * W), (cuuint32_t)NA, 1};
    TRY(make_map(pl, &maps[0], spec, 3, d, st, box));
  }
  {
    cuuint64_t d[3] = {(cuuint64_t)(2 * ncols), (cuuint64_t)NB, (cuuint64_t)NA};
    cuuint64_t st[2] = {(cuuint64_t)(NA * S1), (cuuint64_t)S1};
    cuuint32_t box[3] = {(cuuint32_t)(2 * W), (cuuint32_t)NB, 1};
    TRY(make_map(pl, &maps[1], spec, 3, d, st, box));
  }
  {
    cuuint64_t d[4] = {(cuuint64_t)(2 * G), (cuuint64_t)NA, (cuuint64_t)NB, (cuuint64_t)kFsSlots};
    cuuint64_t st[3] = {(cuuint64_t)(NB * G * esz), (cuuint64_t)(G * esz), (cuuint64_t)(N * G * esz)};
    cuuint32_t boxa[4] = {(cuuint32_t)(2 * W), (cuuint32_t)NA, 1, 1};
    cuuint32_t boxb[4] = {(cuuint32_t)(2 * W), 1, (cuuint32_t)NB, 1};
    TRY(make_map(pl, &maps[2], pl->fs_scratch, 4, d, st, boxa));
    TRY(make_map(pl, &maps[3], pl->fs_scratch, 4, d, st, boxb));
  }
  FsTmaParams f{};
  f.twA = pl->fs_twA;
  f.twB = pl->fs_twB;
  f.twN = pl->fs_twN;
  f.counters = pl->fs_counters;
  f.scratch = pl->fs_scratch;
  f.ngroups = pl->fs_groups;
  f.G = pl->fs_G;
  CUDA_TRY(cudaMemsetAsync(pl->fs_counters, 0, sizeof(unsigned) * (1 + 2 * (size_t)pl->fs_groups), s));
  pl->launches++;
  const cudaError_t e = pl->dtype == TFFFT_F64 ? launch_fourstep_tma<double>(pl->L0, inv, maps, f, s)
                                               : launch_fourstep_tma<float>(pl->L0, inv, maps, f, s);
  CUDA_TRY(e);
  return TFFFT_OK;
}

static cudaError_t fs_launch(tffft_plan_t pl, bool inv, int variant, const FourStepParams& prm, cudaStream_t s) {
  pl->launches++;
  return pl->dtype == TFFFT_F64 ? launch_fourstep<double>(pl->L0, inv, variant, prm, s)
                                : launch_fourstep<float>(pl->L0, inv, variant, prm, s);
}

// stage 3 / 3': c2c along n0 of every STRIDED_INPLACE column c = j*n2c + k
static int stage3_columns(tffft_plan_t pl, void* spec, bool inv, cudaStream_t s) {
  if (pl->fs_la > 0 && pl->p == 1 && fourstep_tma_supported(pl->L0) && !getenv("TFFFT_NO_TMA"))
    return stage3_tma(pl, spec, inv, s);
  if (pl->fs_la > 0) {
    FourStepParams f{};
    f.data = spec;
    f.staging = (inv && pl->p > 1) ? pl->bs[pl->cur].staging : nullptr;
    f.scratch = pl->fs_scratch;
    f.twA = pl->fs_twA;
    f.twB = pl->fs_twB;
    f.twN = pl->fs_twN;
    f.counters = pl->fs_counters;
    f.ncols = (long long)pl->n1p * pl->n2c;
    f.G = pl->fs_G;
    f.ngroups = pl->fs_groups;
    f.ic_shift = ilog2(pl->n0p);
    f.inner_stride = (long long)pl->n1 * pl->n2c;
    f.block_stride = (long long)pl->n1p * pl->n2c;
    f.band_shift = ilog2(pl->n0p);
    f.self_band = pl->rank;
    f.stg_band = (long long)pl->n0p * pl->n1p * pl->n2c;
    f.stg_within = (long long)pl->n1p * pl->n2c;
    CUDA_TRY(cudaMemsetAsync(pl->fs_counters, 0, sizeof(unsigned) * (1 + 2 * (size_t)pl->fs_groups), s));
    CUDA_TRY(fs_launch(pl, inv, pl->p == 1 ? 0 : (f.staging ? 3 : 2), f, s));
    return TFFFT_OK;
  }
  const long long slab = (long long)pl->n0p * pl->n1 * pl->n2c;  // complex elements per field
  const int nb = pl->p == 1 ? pl->batch : 1;  // p = 1: every field of the batch in one launch
  if (pl->p == 1) {
    bool done = false;
    TRY(columns_tma(pl, pl->L0, inv, true, spec, (long long)pl->n1 * pl->n2c, nb, (long long)pl->n1 * pl->n2c,
                    slab, pl->tw0, s, &done));
    if (done) return TFFFT_OK;
  }
  ColParams c{};
  c.data = spec;
  c.tw = pl->tw0;
  c.ncols = (long long)pl->n1p * pl->n2c * nb;
  c.cpb = (int)std::min<long long>((long long)pl->n1p * pl->n2c, 1LL << 30);
  c.grp_stride = slab;
  c.ic_shift = ilog2(pl->n0p);
  c.inner_stride = (long long)pl->n1 * pl->n2c;
  c.block_stride = (long long)pl->n1p * pl->n2c;
  c.band_shift = ilog2(pl->n0p);
  c.self_band = pl->rank;
  c.staging = nullptr;
  // stage 3 walks rows n1*n2c elements apart: widen the DRAM row visits with
  // L2 prefetches one resident wave ahead (tools/micro/stride_bw2.cu)
  {
    static const char* env = getenv("TFFFT_L2PF");
    const long long ahead = env ? atoll(env) : 0;
    const int pfb = 256;
    const bool aligned = ((long long)pl->n1p * pl->n2c * (long long)pl->esz) % pfb == 0 &&
                         ((long long)pl->n1 * pl->n2c * (long long)pl->esz) % pfb == 0;
    c.pf_ahead = aligned ? ahead : 0;
    c.pf_bytes = pfb;
  }
  if (pl->p > 1) {
    // p > 1 through the TMA column kernel: forward = landing[s][i][c] loads +
    // in-place two-level stores; inverse = two-level loads + block redirect
    const BufSet& B = pl->bs[pl->cur];
    const long long n1p = pl->n1p, n2c = pl->n2c, band = (long long)pl->n0p * n1p * n2c;
    TwoLevelJob j{};
    j.wide = true;
    j.cols = n1p * n2c;
    j.ngrp = 1;
    j.ld_in_rows = pl->n0p;
    j.ld_blocks = pl->p;
    j.st_rows = pl->n0p;
    if (!inv) {
      j.ld_base = B.landing; j.ld_in = n1p * n2c; j.ld_out = band;
      for (int q = 0; q < pl->p; ++q) j.st_tab.push_back(static_cast<char*>(spec) + (size_t)q * n1p * n2c * pl->esz);
      j.st_in = (long long)pl->n1 * n2c;
    } else {
      j.ld_base = spec; j.ld_in = (long long)pl->n1 * n2c; j.ld_out = n1p * n2c;
      j.st_tab = B.band_dst_h; j.st_in = n1p * n2c;
    }
    bool done = false;
    TRY(columns_tma_two(pl, pl->L0, inv, j, pl->tw0, s, &done));
    if (done) return TFFFT_OK;
  }
  int rd = 0;
  if (pl->p > 1) {
    // forward: block s is read from landing[s][i][c] (the exchange output; the
    // self block from landing[rank]); inverse epilogue: block s -> band_dst[s]
    // (landing[rank] for the self block, staging[s] or rank s's landing[rank])
    const BufSet& B = pl->bs[pl->cur];
    c.staging = B.landing;
    c.band_dst = B.band_dst;
    c.self_band = -1;
    rd = inv ? 1 : 2;
    c.stg_band = (long long)pl->n0p * pl->n1p * pl->n2c;
    c.stg_within = (long long)pl->n1p * pl->n2c;
    c.stg_grp = 0;
  }
  CUDA_TRY(col_launch(pl, pl->L0, inv, pl->p > 1, rd, true, c, s));
  return TFFFT_OK;
}

// row pass over `nplanes` planes at (real, spec); the c2r statistics of those
// rows go to the records of planes [stat_plane0, stat_plane0 + nplanes) (a
// batch's planes are numbered field after field)
static RowParams row_params(tffft_plan_t pl, void* real, void* spec, int nplanes, long long stat_plane0) {
  RowParams r{};
  r.real = real;
  r.spec = spec;
  r.tw = pl->tw2;
  r.tw_post = pl->tw2post;
  r.nrows = (long long)nplanes * pl->n1;
  r.n2c = pl->n2c;
  r.rows_per_plane = pl->n1;
  r.scale = 1.0 / ((double)pl->n0 * (double)pl->n1 * (double)pl->n2);
  r.row_stats = pl->row_stats + 3 * stat_plane0 * pl->n1;
  return r;
}

// fused stage 1 / 1': one persistent kernel per direction, planes stay in L2
static int stage1_fused(tffft_plan_t pl, void* real, void* spec, bool fwd, cudaStream_t s) {
  Stage1Params f{};
  f.real = real;
  f.spec = spec;
  f.staging = (fwd && pl->p > 1) ? pl->bs[pl->cur].staging : nullptr;
  f.tw_row = pl->tw2;
  f.tw_post = pl->tw2post;
  f.tw_col = pl->tw1;
  f.stats = pl->stats;
  f.counters = pl->s1_counters;
  f.n0p = pl->n0p;
  f.n1 = pl->n1;
  f.n2c = pl->n2c;
  f.scale = 1.0 / ((double)pl->n0 * (double)pl->n1 * (double)pl->n2);
  f.band_shift = ilog2(pl->n1p);
  f.self_band = pl->rank;
  f.stg_band = (long long)pl->n0p * pl->n1p * pl->n2c;
  f.stg_grp = (long long)pl->n1p * pl->n2c;
  {
    static const char* env = getenv("TFFFT_S1_LOOKAHEAD");
    f.lookahead = env ? std::max(1, atoi(env)) : 3;
  }
  CUDA_TRY(cudaMemsetAsync(pl->s1_counters, 0, sizeof(unsigned) * (1 + 2 * (size_t)pl->n0p), s));
  pl->launches++;
  const cudaError_t e = pl->dtype == TFFFT_F64
      ? launch_stage1_fused<double>(pl->L2h, pl->L1, fwd, f.staging != nullptr, f, s)
      : launch_stage1_fused<float>(pl->L2h, pl->L1, fwd, f.staging != nullptr, f, s);
  CUDA_TRY(e);
  return TFFFT_OK;
}

static size_t band_bytes(tffft_plan_t pl) { return (size_t)pl->n0p * pl->n1p * pl->n2c * pl->esz; }

// Stream-ordered barrier over an NCCL communicator: a one-int all-reduce.  It
// completes on this rank only after every rank's preceding kernels have
// completed, so their peer stores into our landing buffer are visible (or,
// before a producing stage, every peer has finished reading its landing
// buffer).
static int nccl_barrier(tffft_plan_t pl, cudaStream_t s) {
  NcclApi& api = nccl();
  NCCL_TRY(api.AllReduce(pl->barrier_word, pl->barrier_word, 1, ncclInt32, ncclSum, pl->comm->nccl, s));
  return TFFFT_OK;
}

static bool fabric_kind(tffft_plan_t pl) { return pl->comm->kind != COMM_NCCL; }

// Before a stage writes the outgoing bands of the current set.  Fabric pull
// (local / IPC): every peer has finished pulling from our staging (its "done"
// event of this set, recorded before the barrier that ended that exchange).
// Peer stores: every peer has consumed its landing buffer -- the host barrier
// makes sure each peer recorded that event for the previous exchange.  NCCL
// send/recv needs nothing: the sends are stream-ordered before this stage.
static int guard_outgoing(tffft_plan_t pl, cudaStream_t s) {
  if (pl->p == 1) return TFFFT_OK;
  BufSet& B = pl->bs[pl->cur];
  if (!fabric_kind(pl)) return pl->peer_stores ? nccl_barrier(pl, s) : TFFFT_OK;
  if (pl->peer_stores) TRY(pl->comm->barrier());
  for (int q = 0; q < pl->p; ++q)
    if (q != pl->rank) CUDA_TRY(cudaStreamWaitEvent(s, B.done[q], 0));
  return TFFFT_OK;
}

// peer stores: this rank has consumed its landing buffer of the current set
static int landing_consumed(tffft_plan_t pl, cudaStream_t s) {
  if (pl->p == 1 || !pl->peer_stores || !fabric_kind(pl)) return TFFFT_OK;  // NCCL: the next guard barrier covers it
  CUDA_TRY(cudaEventRecord(pl->bs[pl->cur].done[pl->rank], s));
  return TFFFT_OK;
}

// destination block of each outgoing band for the write-redirect epilogues of
// one set.  The self band goes to landing[rank] (the next stage reads every
// band from the landing buffer), except on NCCL COLLECTIVE without peer stores,
// where it travels through the all-to-all's self slot (staging[rank] ->
// landing[rank]).
static int build_band_dst(tffft_plan_t pl, int set) {
  BufSet& B = pl->bs[set];
  const size_t band = band_bytes(pl);
  std::vector<void*> h(pl->p, nullptr);
  const bool nccl_a2a = !fabric_kind(pl) && pl->pattern == TFFFT_COLLECTIVE && !pl->peer_stores && nccl().AlltoAll;
  for (int q = 0; q < pl->p; ++q) {
    if (q == pl->rank)
      h[q] = static_cast<char*>(nccl_a2a ? B.staging : B.landing) + (size_t)q * band;
    else if (pl->peer_stores)
      h[q] = static_cast<char*>(B.peer_landing[q]) + (size_t)pl->rank * band;  // rank q's landing block for us
    else
      h[q] = static_cast<char*>(B.staging) + (size_t)q * band;
  }
  if (!B.band_dst) CUDA_TRY(cudaMalloc(&B.band_dst, sizeof(void*) * pl->p));
  CUDA_TRY(cudaMemcpy(B.band_dst, h.data(), sizeof(void*) * pl->p, cudaMemcpyHostToDevice));
  B.band_dst_h = h;
  return TFFFT_OK;
}

// fabric pull list of one set, in the PAIRWISE ring order (d = 1 .. p-1: the
// band of rank (rank - d) mod p): (peer's staging band for us, our landing band)
static int build_pull_list(tffft_plan_t pl, int set) {
  BufSet& B = pl->bs[set];
  const size_t band = band_bytes(pl);
  std::vector<void*> h;
  for (int d = 1; d < pl->p; ++d) {
    const int q = (pl->rank - d + pl->p) % pl->p;
    h.push_back(static_cast<char*>(B.peer_staging[q]) + (size_t)pl->rank * band);
    h.push_back(static_cast<char*>(B.landing) + (size_t)q * band);
  }
  if (!B.pull_ptrs) CUDA_TRY(cudaMalloc(&B.pull_ptrs, sizeof(void*) * 2 * (size_t)(pl->p - 1)));
  CUDA_TRY(cudaMemcpy(B.pull_ptrs, h.data(), h.size() * sizeof(void*), cudaMemcpyHostToDevice));
  return TFFFT_OK;
}

// The exchange proper (exchange.py:263-290) of the current set: my band q
// (n0p chunks of (n1/p)*n2c, contiguous in staging[q]) goes to rank q, whose
// landing[rank] receives it; the next FFT stage reads the landing buffer
// through the STRIDED_INPLACE addressing, so no rearrangement pass follows.
// Failure detection: an asynchronous NCCL error (a peer died,
// a network fault) surfaces as TFFFT_ERR_TRANSPORT on the next exchange, like
// the reference fabric's abort propagation (transport.py:209-219, 446-467).
static int nccl_async_check(tffft_comm_t c) {
  if (!c->is_nccl || c->p == 1 || !c->nccl) return TFFFT_OK;
  NcclApi& api = nccl();
  ncclResult_t st = ncclSuccess;
  NCCL_TRY(api.CommGetAsyncError(c->nccl, &st));
  if (st != ncclSuccess && st != ncclInProgress)
    return fail(TFFFT_ERR_TRANSPORT, "NCCL communicator failed asynchronously: %s", api.GetErrorString(st));
  return TFFFT_OK;
}

// pull rows [i0, i0 + ni) of each listed band (the whole band: i0 = 0, ni = n0p)
static int launch_pull(tffft_plan_t pl, void* const* ptrs, int nchunks, cudaStream_t s, long long i0 = 0,
                       long long ni = -1) {
  if (ni < 0) ni = pl->n0p;
  const long long row = (long long)pl->n1p * pl->n2c * (long long)pl->esz;  // bytes of one plane's chunk
  const bool wide = row % 16 == 0;
  const long long wb = wide ? 16 : 8;
  const long long words = ni * row / wb, off = i0 * row / wb;
  dim3 grid((unsigned)std::min<long long>((words + 255) / 256, 2048), (unsigned)nchunks);
  if (wide)
    pull_chunks_kernel<int4><<<grid, 256, 0, s>>>(ptrs, off, words, nchunks);
  else
    pull_chunks_kernel<int2><<<grid, 256, 0, s>>>(ptrs, off, words, nchunks);
  pl->launches++;
  CUDA_TRY(cudaGetLastError());
  return TFFFT_OK;
}

// i0 / ni: the planes of every band this exchange moves (default: all; the
// chunked forward moves plane chunks as stage 1 produces them)
static int exchange(tffft_plan_t pl, cudaStream_t s, long long i0 = 0, long long ni = -1) {
  if (pl->p == 1) return TFFFT_OK;
  TRY(nccl_async_check(pl->comm));
  BufSet& B = pl->bs[pl->cur];
  if (ni < 0) ni = pl->n0p;
  const long long band = (long long)pl->n0p * pl->n1p * pl->n2c;  // complex elements per peer
  const long long chunk = (long long)pl->n1p * pl->n2c;            // complex elements per plane of a band
  const uint64_t wire = (uint64_t)(pl->p - 1) * ni * chunk * pl->esz;
  if (pl->peer_stores && !fabric_kind(pl)) {
    // the epilogue already stored every band into its peer's landing buffer
    // over NVLink (CUDA IPC mapping): the exchange is the barrier
    TRY(nccl_barrier(pl, s));
    pl->counters[1] += wire;
    return TFFFT_OK;
  }
  if (pl->peer_stores) {
    // the epilogue already stored every band into its peer's landing buffer:
    // the exchange is the barrier after which every rank's stores are visible
    CUDA_TRY(cudaEventRecord(B.ready[pl->rank], s));
    TRY(pl->comm->barrier());
    for (int q = 0; q < pl->p; ++q)
      if (q != pl->rank) CUDA_TRY(cudaStreamWaitEvent(s, B.ready[q], 0));
    pl->counters[1] += wire;
    return TFFFT_OK;
  }
  if (!fabric_kind(pl)) {
    NcclApi& api = nccl();
    const ncclDataType_t dt = pl->dtype == TFFFT_F64 ? ncclFloat64 : ncclFloat32;
    char* stg = static_cast<char*>(B.staging);
    char* lnd = static_cast<char*>(B.landing);
    if (pl->pattern == TFFFT_COLLECTIVE && api.AlltoAll && ni == pl->n0p) {
      // COLLECTIVE (transport.py:395-419): every rank deposits all of its
      // outgoing bands in one all-to-all; the self slot carries the self band
      // from staging[rank] to landing[rank] (build_band_dst)
      NCCL_TRY(api.AlltoAll(stg, lnd, 2 * band, dt, pl->comm->nccl, s));
      pl->counters[1] += wire;
      return TFFFT_OK;
    }
    // one send and one receive per peer (the plane range of each band is contiguous)
    const long long off = i0 * chunk * pl->esz, count = 2 * ni * chunk;
    if (pl->pattern == TFFFT_COLLECTIVE && api.AlltoAll) {
      // COLLECTIVE plans keep the self band in the all-to-all's self slot (build_band_dst); a plane
      // chunk goes through send / recv instead, so the self band's chunk moves with a device copy
      const long long so = (long long)pl->rank * band * pl->esz + off;
      CUDA_TRY(cudaMemcpyAsync(lnd + so, stg + so, (size_t)(ni * chunk * pl->esz), cudaMemcpyDeviceToDevice, s));
    }
    NCCL_TRY(api.GroupStart());
    for (int d = 1; d < pl->p; ++d) {
      const int to = (pl->rank + d) % pl->p, from = (pl->rank - d + pl->p) % pl->p;
      NCCL_TRY(api.Send(stg + (long long)to * band * pl->esz + off, count, dt, to, pl->comm->nccl, s));
      NCCL_TRY(api.Recv(lnd + (long long)from * band * pl->esz + off, count, dt, from, pl->comm->nccl, s));
    }
    NCCL_TRY(api.GroupEnd());
  } else {
    // fabric pull (local fabric or CUDA IPC across processes): every rank
    // records that its staging is written, meets the others at the host
    // barrier, then pulls its p-1 incoming bands from the peers' staging.
    // PAIRWISE: one pull per peer in ring order (the reference posts one
    // strided send/recv pair per peer); COLLECTIVE: all bands in one launch.
    CUDA_TRY(cudaEventRecord(B.ready[pl->rank], s));
    TRY(pl->comm->barrier());
    for (int q = 0; q < pl->p; ++q)
      if (q != pl->rank) CUDA_TRY(cudaStreamWaitEvent(s, B.ready[q], 0));
    if (pl->pattern == TFFFT_COLLECTIVE) {
      TRY(launch_pull(pl, B.pull_ptrs, pl->p - 1, s, i0, ni));
    } else {
      for (int d = 1; d < pl->p; ++d) TRY(launch_pull(pl, B.pull_ptrs + 2 * (d - 1), 1, s, i0, ni));
    }
    CUDA_TRY(cudaEventRecord(B.done[pl->rank], s));
    TRY(pl->comm->barrier());
  }
  pl->counters[1] += wire;
  return TFFFT_OK;
}

// Local fabric: create this rank's events of every set, publish them with the
// buffers, meet the other ranks and copy theirs (no reference into the shared
// fabric is kept past the call).
static int fabric_setup_local(tffft_plan_t pl) {
  LocalFabric& fab = *pl->comm->fabric;
  for (int st = 0; st < pl->nsets; ++st) {
    BufSet& B = pl->bs[st];
    cudaEvent_t rdy, dn;
    CUDA_TRY(cudaEventCreateWithFlags(&rdy, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&dn, cudaEventDisableTiming));
    fab.publish(pl->seq, pl->rank, st, B.staging, B.landing, rdy, dn);
  }
  TRY(fab.barrier());
  for (int st = 0; st < pl->nsets; ++st) {
    BufSet& B = pl->bs[st];
    fab.collect(pl->seq, st, B.peer_staging, B.peer_landing, B.ready, B.done);
  }
  TRY(fab.barrier());  // every rank has copied the table: the slot is never read again
  return TFFFT_OK;
}

// ---------------------------------------------------------------------------
// TRANSPOSE strategy (exchange.py:195-260): local transpose into per-peer
// blocks, contiguous exchange, rearrangement into CONTIGUOUS_FLIPPED
// (element (j, r, k) at j*n0*n2c + r*n2c + k, layout.py:42-44)
// ---------------------------------------------------------------------------
static int permute(tffft_plan_t pl, const PermuteParams& prm, cudaStream_t s) {
  const long long rows = (long long)prm.A * prm.B * prm.C;
  const unsigned blocks = (unsigned)std::min<long long>((rows + 7) / 8, 148LL * 64);
  pl->launches++;
  if (pl->esz == 16)
    permute_rows_kernel<int4><<<blocks, 256, 0, s>>>(prm, 16);
  else
    permute_rows_kernel<int2><<<blocks, 256, 0, s>>>(prm, 8);
  CUDA_TRY(cudaGetLastError());
  return TFFFT_OK;
}

static uint64_t offrank_block_bytes(tffft_plan_t pl) {
  return (uint64_t)(pl->p - 1) * pl->n0p * pl->n1p * pl->n2c * pl->esz;
}

// forward: (n0p, n1, n2c) stage-1 output in `spec` -> staging[q][j][i][k]
static int pack_forward(tffft_plan_t pl, void* spec, cudaStream_t s) {
  const long long n2c = pl->n2c, n1p = pl->n1p, n0p = pl->n0p, band = n0p * n1p * n2c;
  PermuteParams p{};
  p.src = spec; p.src_self = spec; p.dst = pl->bs[pl->cur].staging; p.self = -1;
  p.A = pl->p; p.B = (int)n1p; p.C = (int)n0p;
  p.sa = n1p * n2c; p.sb = n2c; p.sc = (long long)pl->n1 * n2c;
  p.da = band; p.db = n0p * n2c; p.dc = n2c;
  p.row_words = n2c;
  TRY(permute(pl, p, s));
  pl->counters[0] += offrank_block_bytes(pl);
  return TFFFT_OK;
}
// forward: blocks [src][j][i][k] (own block from staging) -> flipped (j, src*n0p + i, k) in `spec`
static int unpack_forward(tffft_plan_t pl, void* spec, cudaStream_t s) {
  const long long n2c = pl->n2c, n1p = pl->n1p, n0p = pl->n0p, band = n0p * n1p * n2c;
  PermuteParams p{};
  p.src = pl->p > 1 ? pl->bs[pl->cur].landing : pl->bs[pl->cur].staging;
  p.dst = spec; p.self = pl->rank;
  p.A = pl->p; p.B = (int)n1p; p.C = (int)n0p;
  p.sa = band; p.sb = n0p * n2c; p.sc = n2c;
  p.da = n0p * n2c; p.db = (long long)pl->n0 * n2c; p.dc = n2c;
  p.row_words = n2c;
  p.src_self = pl->bs[pl->cur].staging;  // indexed like the landing buffer: block `rank` of staging
  TRY(permute(pl, p, s));
  pl->counters[2] += offrank_block_bytes(pl);
  return TFFFT_OK;
}
// inverse: flipped (j, dest*n0p + i, k) in `spec` -> staging[dest][j][i][k]
static int pack_inverse(tffft_plan_t pl, void* spec, cudaStream_t s) {
  const long long n2c = pl->n2c, n1p = pl->n1p, n0p = pl->n0p, band = n0p * n1p * n2c;
  PermuteParams p{};
  p.src = spec; p.src_self = spec; p.dst = pl->bs[pl->cur].staging; p.self = -1;
  p.A = pl->p; p.B = (int)n1p; p.C = (int)n0p;
  p.sa = n0p * n2c; p.sb = (long long)pl->n0 * n2c; p.sc = n2c;
  p.da = band; p.db = n0p * n2c; p.dc = n2c;
  p.row_words = n2c;
  TRY(permute(pl, p, s));
  pl->counters[0] += offrank_block_bytes(pl);
  return TFFFT_OK;
}
// inverse: blocks [src][j][i][k] -> (i, src*n1p + j, k) of the (n0p, n1, n2c) buffer `spec`
static int unpack_inverse(tffft_plan_t pl, void* spec, cudaStream_t s) {
  const long long n2c = pl->n2c, n1p = pl->n1p, n0p = pl->n0p, band = n0p * n1p * n2c;
  PermuteParams p{};
  p.src = pl->p > 1 ? pl->bs[pl->cur].landing : pl->bs[pl->cur].staging;
  p.src_self = pl->bs[pl->cur].staging;
  p.dst = spec; p.self = pl->rank;
  p.A = pl->p; p.B = (int)n1p; p.C = (int)n0p;
  p.sa = band; p.sb = n0p * n2c; p.sc = n2c;
  p.da = n1p * n2c; p.db = n2c; p.dc = (long long)pl->n1 * n2c;
  p.row_words = n2c;
  TRY(permute(pl, p, s));
  pl->counters[2] += offrank_block_bytes(pl);
  return TFFFT_OK;
}

// stage 3 / 3' over the CONTIGUOUS_FLIPPED layout: column (j, k) at stride n2c
static int stage3_flipped(tffft_plan_t pl, void* spec, bool inv, cudaStream_t s) {
  if (pl->p == 1) {
    bool done = false;
    TRY(columns_tma(pl, pl->L0, inv, true, spec, (long long)pl->n1 * pl->n2c, 1, (long long)pl->n1 * pl->n2c, 0,
                    pl->tw0, s, &done));
    if (done) return TFFFT_OK;
  }
  ColParams c{};
  c.data = spec;
  c.tw = pl->tw0;
  c.ncols = (long long)pl->n1p * pl->n2c;
  c.cpb = pl->n2c;
  c.grp_stride = (long long)pl->n0 * pl->n2c;
  c.ic_shift = 30;
  c.inner_stride = pl->n2c;
  c.block_stride = 0;
  c.band_shift = 30;
  c.self_band = 0;
  CUDA_TRY(col_launch(pl, pl->L0, inv, false, 0, false, c, s));
  return TFFFT_OK;
}

struct PlanDeleter {
  void operator()(tffft_plan_s* p) const { tffft_plan_destroy(p); }
};

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {
#pragma GCC visibility push(default)

const char* tffft_last_error(void) { return g_last_error.c_str(); }
int tffft_version(void) { return 100; }

int tffft_get_unique_id(uint8_t out[128]) {
  if (!out) return fail(TFFFT_ERR_CONFIGURATION, "null output");
  NcclApi& api = nccl();
  if (!api.loaded) return fail(TFFFT_ERR_TRANSPORT, "NCCL unavailable: %s", api.err.c_str());
  ncclUniqueId id;
  NCCL_TRY(api.GetUniqueId(&id));
  memcpy(out, id.internal, 128);
  return TFFFT_OK;
}

int tffft_comm_init_rank(int p, int rank, const uint8_t id[128], int device, tffft_comm_t* comm) {
  if (!comm || !id) return fail(TFFFT_ERR_CONFIGURATION, "null argument");
  if (p < 1 || rank < 0 || rank >= p) return fail(TFFFT_ERR_CONFIGURATION, "rank %d outside [0, %d)", rank, p);
  auto c = std::make_unique<tffft_comm_s>();
  c->p = p;
  c->rank = rank;
  c->device = device;
  c->is_nccl = true;
  c->kind = COMM_NCCL;
  CUDA_TRY(cudaSetDevice(device));
  if (p > 1) {
    NcclApi& api = nccl();
    if (!api.loaded) return fail(TFFFT_ERR_TRANSPORT, "NCCL unavailable: %s", api.err.c_str());
    ncclUniqueId uid;
    memcpy(uid.internal, id, 128);
    NCCL_TRY(api.CommInitRank(&c->nccl, p, uid, rank));
  }
  *comm = c.release();
  return TFFFT_OK;
}

// single process, one communicator per listed device (ncclCommInitAll): the
// run_spmd analogue across GPUs, one host thread driving each communicator
int tffft_comm_init_all(int p, const int* devices, tffft_comm_t* comms) {
  if (!comms || !devices) return fail(TFFFT_ERR_CONFIGURATION, "null argument");
  if (p < 1) return fail(TFFFT_ERR_CONFIGURATION, "communicator group needs p >= 1, got %d", p);
  for (int a = 0; a < p; ++a)
    for (int b = a + 1; b < p; ++b)
      if (devices[a] == devices[b])
        return fail(TFFFT_ERR_CONFIGURATION, "comm_init_all: device %d listed twice (NCCL needs one GPU per rank; "
                    "use comm_init_local for ranks sharing a device)", devices[a]);
  std::vector<ncclComm_t> nc(p, nullptr);
  if (p > 1) {
    NcclApi& api = nccl();
    if (!api.loaded) return fail(TFFFT_ERR_TRANSPORT, "NCCL unavailable: %s", api.err.c_str());
    if (!api.CommInitAll) return fail(TFFFT_ERR_TRANSPORT, "ncclCommInitAll missing from the loaded NCCL");
    NCCL_TRY(api.CommInitAll(nc.data(), p, devices));
  }
  for (int r = 0; r < p; ++r) {
    auto* c = new tffft_comm_s();
    c->p = p;
    c->rank = r;
    c->device = devices[r];
    c->is_nccl = true;
    c->kind = COMM_NCCL;
    c->nccl = nc[r];
    comms[r] = c;
  }
  return TFFFT_OK;
}

// one process per rank, exchange through CUDA IPC mappings of the peers'
// buffers ordered by IPC events, with the caller's host barrier (MPI, a
// torch.distributed gloo group, ...) as the only host-side collective
int tffft_comm_init_ipc(int p, int rank, int device, tffft_barrier_fn barrier, void* ctx, tffft_comm_t* comm) {
  if (!comm || !barrier) return fail(TFFFT_ERR_CONFIGURATION, "null argument");
  if (p < 1 || rank < 0 || rank >= p) return fail(TFFFT_ERR_CONFIGURATION, "rank %d outside [0, %d)", rank, p);
  auto* c = new tffft_comm_s();
  c->p = p;
  c->rank = rank;
  c->device = device;
  c->kind = COMM_IPC;
  c->barrier_fn = barrier;
  c->barrier_ctx = ctx;
  *comm = c;
  return TFFFT_OK;
}

int tffft_comm_init_local(int p, int device, tffft_comm_t* comms) {
  if (!comms) return fail(TFFFT_ERR_CONFIGURATION, "null argument");
  if (p < 1) return fail(TFFFT_ERR_CONFIGURATION, "communicator group needs p >= 1, got %d", p);
  auto fab = std::make_shared<LocalFabric>(p, device);
  const char* to = getenv("TFFFT_FABRIC_TIMEOUT");
  if (to) fab->timeout_s = atof(to);
  for (int r = 0; r < p; ++r) {
    auto* c = new tffft_comm_s();
    c->p = p;
    c->rank = r;
    c->device = device;
    c->fabric = fab;
    comms[r] = c;
  }
  return TFFFT_OK;
}

// host barrier of a local-fabric or IPC communicator (Endpoint.barrier's
// rank-meeting half, cli.py:102, 106); NCCL communicators have no host barrier
int tffft_comm_barrier(tffft_comm_t c) {
  if (!c) return fail(TFFFT_ERR_CONFIGURATION, "null communicator");
  if (c->kind == COMM_NCCL) return fail(TFFFT_ERR_CONFIGURATION, "NCCL communicators have no host barrier");
  return c->barrier();
}

int tffft_comm_check(tffft_comm_t c) {
  if (!c) return fail(TFFFT_ERR_CONFIGURATION, "null communicator");
  return nccl_async_check(c);
}

int tffft_comm_rank(tffft_comm_t c, int* r) {
  if (!c || !r) return fail(TFFFT_ERR_CONFIGURATION, "null argument");
  *r = c->rank;
  return TFFFT_OK;
}
int tffft_comm_size(tffft_comm_t c, int* p) {
  if (!c || !p) return fail(TFFFT_ERR_CONFIGURATION, "null argument");
  *p = c->p;
  return TFFFT_OK;
}
int tffft_comm_device(tffft_comm_t c, int* d) {
  if (!c || !d) return fail(TFFFT_ERR_CONFIGURATION, "null argument");
  *d = c->device;
  return TFFFT_OK;
}

int tffft_comm_abort(tffft_comm_t c) {
  if (!c) return fail(TFFFT_ERR_CONFIGURATION, "null comm");
  if (c->fabric) c->fabric->abort();
  c->aborted = true;
  if (c->nccl) {
    NCCL_TRY(nccl().CommAbort(c->nccl));
    c->nccl = nullptr;
  }
  return TFFFT_OK;
}

int tffft_comm_destroy(tffft_comm_t c) {
  if (!c) return TFFFT_OK;
  if (c->nccl) nccl().CommDestroy(c->nccl);
  delete c;
  return TFFFT_OK;
}

static int env_flags() {
  int f = 0;
  const char* tc = getenv("TFFFT_TMA_COLS");
  if (tc && atoi(tc) != 0) f |= TFFFT_FLAG_TMA_COLUMNS;
  const char* fuse = getenv("TFFFT_FUSE");
  const char* fs = getenv("TFFFT_FOURSTEP");
  if (fuse && atoi(fuse) != 0) f |= TFFFT_FLAG_FUSED_STAGE1;
  if (fs && atoi(fs) != 0) f |= TFFFT_FLAG_FOURSTEP_STAGE3;
  return f;
}

int tffft_plan_create(int n0, int n1, int n2, int dtype, int pattern, tffft_comm_t comm, tffft_plan_t* out) {
  return tffft_plan_create_ex(n0, n1, n2, dtype, pattern, -1, comm, out);
}

int tffft_plan_flags(tffft_plan_t pl, int* flags) {
  if (!pl || !flags) return fail(TFFFT_ERR_CONFIGURATION, "null argument");
  *flags = (pl->s1_fused ? TFFFT_FLAG_FUSED_STAGE1 : 0) | (pl->fs_la > 0 ? TFFFT_FLAG_FOURSTEP_STAGE3 : 0) |
           (pl->strategy == 1 ? TFFFT_FLAG_TRANSPOSE : 0) | (pl->peer_stores ? TFFFT_FLAG_PEER_STORES : 0) |
           (pl->tma_cols == 1 ? TFFFT_FLAG_TMA_COLUMNS : 0) | (pl->xchunks > 1 ? TFFFT_FLAG_CHUNKED_EXCHANGE : 0);
  return TFFFT_OK;
}

// ---- CUDA IPC: export this rank's exchange buffers, attach the peers' -----
// Blob of one plan: per buffer set, four 64-byte handles: staging memory,
// landing memory, "ready" event, "done" event (events: IPC communicators only).
static constexpr size_t kIpcSetBytes = 4 * 64;

int tffft_plan_ipc_blob_bytes(tffft_plan_t pl, size_t* bytes) {
  if (!pl || !bytes) return fail(TFFFT_ERR_CONFIGURATION, "null argument");
  *bytes = (size_t)pl->nsets * kIpcSetBytes;
  return TFFFT_OK;
}

int tffft_plan_ipc_export(tffft_plan_t pl, uint8_t* blob) {
  if (!pl || !blob) return fail(TFFFT_ERR_CONFIGURATION, "null argument");
  if (pl->p == 1 || pl->comm->kind == COMM_LOCAL)
    return fail(TFFFT_ERR_CONFIGURATION, "IPC handles exist for NCCL / IPC plans with p > 1 only");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64 && sizeof(cudaIpcEventHandle_t) == 64, "64-byte IPC handles");
  CUDA_TRY(cudaSetDevice(pl->comm->device));
  memset(blob, 0, (size_t)pl->nsets * kIpcSetBytes);
  for (int st = 0; st < pl->nsets; ++st) {
    BufSet& B = pl->bs[st];
    uint8_t* o = blob + st * kIpcSetBytes;
    cudaIpcMemHandle_t m;
    CUDA_TRY(cudaIpcGetMemHandle(&m, B.staging));
    memcpy(o, &m, 64);
    CUDA_TRY(cudaIpcGetMemHandle(&m, B.landing));
    memcpy(o + 64, &m, 64);
    if (pl->comm->kind == COMM_IPC) {
      cudaIpcEventHandle_t e;
      CUDA_TRY(cudaIpcGetEventHandle(&e, B.ready[pl->rank]));
      memcpy(o + 128, &e, 64);
      CUDA_TRY(cudaIpcGetEventHandle(&e, B.done[pl->rank]));
      memcpy(o + 192, &e, 64);
    }
  }
  return TFFFT_OK;
}

// blobs: p blobs of tffft_plan_ipc_blob_bytes each, in rank order (all-gathered
// by the caller).  Collective: every rank of the communicator must attach.
// NCCL plans map the peers' landing buffers (peer stores, TFFFT_FLAG_PEER_STORES);
// IPC plans map the peers' staging and landing buffers and open their events.
int tffft_plan_ipc_attach(tffft_plan_t pl, const uint8_t* blobs) {
  if (!pl || !blobs) return fail(TFFFT_ERR_CONFIGURATION, "null argument");
  if (pl->p == 1 || pl->comm->kind == COMM_LOCAL)
    return fail(TFFFT_ERR_CONFIGURATION, "ipc_attach needs an NCCL or IPC plan with p > 1");
  if (pl->comm->kind == COMM_NCCL && !pl->peer_stores_wanted)
    return fail(TFFFT_ERR_CONFIGURATION, "ipc_attach on an NCCL plan needs TFFFT_FLAG_PEER_STORES");
  if (pl->ipc_attached) return fail(TFFFT_ERR_PROTOCOL, "peers already attached");
  CUDA_TRY(cudaSetDevice(pl->comm->device));
  const size_t blob = (size_t)pl->nsets * kIpcSetBytes;
  const bool ipc = pl->comm->kind == COMM_IPC;
  for (int st = 0; st < pl->nsets; ++st) {
    BufSet& B = pl->bs[st];
    for (int q = 0; q < pl->p; ++q) {
      if (q == pl->rank) continue;
      const uint8_t* o = blobs + (size_t)q * blob + st * kIpcSetBytes;
      cudaIpcMemHandle_t m;
      if (ipc) {
        memcpy(&m, o, 64);
        CUDA_TRY(cudaIpcOpenMemHandle(&B.peer_staging[q], m, cudaIpcMemLazyEnablePeerAccess));
        pl->ipc_opened.push_back(B.peer_staging[q]);
      }
      memcpy(&m, o + 64, 64);
      CUDA_TRY(cudaIpcOpenMemHandle(&B.peer_landing[q], m, cudaIpcMemLazyEnablePeerAccess));
      pl->ipc_opened.push_back(B.peer_landing[q]);
      if (ipc) {
        cudaIpcEventHandle_t e;
        memcpy(&e, o + 128, 64);
        CUDA_TRY(cudaIpcOpenEventHandle(&B.ready[q], e));
        pl->ipc_events.push_back(B.ready[q]);
        memcpy(&e, o + 192, 64);
        CUDA_TRY(cudaIpcOpenEventHandle(&B.done[q], e));
        pl->ipc_events.push_back(B.done[q]);
      }
    }
  }
  if (!ipc) {
    CUDA_TRY(cudaMalloc(&pl->barrier_word, sizeof(int)));
    CUDA_TRY(cudaMemset(pl->barrier_word, 0, sizeof(int)));
  }
  pl->peer_stores = pl->peer_stores_wanted;
  pl->ipc_attached = true;
  for (int st = 0; st < pl->nsets; ++st) {
    if (ipc) TRY(build_pull_list(pl, st));
    TRY(build_band_dst(pl, st));
  }
  return TFFFT_OK;
}

// round-1 names of the NCCL peer-store attach (one buffer set): the landing
// handle alone, and p landing handles in rank order
int tffft_plan_landing_handle(tffft_plan_t pl, uint8_t handle[64]) {
  if (!pl || !handle) return fail(TFFFT_ERR_CONFIGURATION, "null argument");
  if (pl->comm->kind != COMM_NCCL || pl->p == 1 || pl->nsets != 1)
    return fail(TFFFT_ERR_CONFIGURATION, "landing handles exist for unbatched NCCL plans with p > 1 only");
  uint8_t blob[kIpcSetBytes];
  TRY(tffft_plan_ipc_export(pl, blob));
  memcpy(handle, blob + 64, 64);
  return TFFFT_OK;
}

int tffft_plan_attach_peers(tffft_plan_t pl, const uint8_t* handles) {
  if (!pl || !handles) return fail(TFFFT_ERR_CONFIGURATION, "null argument");
  if (pl->comm->kind != COMM_NCCL || pl->p == 1 || pl->nsets != 1 || !pl->peer_stores_wanted)
    return fail(TFFFT_ERR_CONFIGURATION,
                "attach_peers needs an unbatched NCCL plan with p > 1 created with TFFFT_FLAG_PEER_STORES");
  std::vector<uint8_t> blobs((size_t)pl->p * kIpcSetBytes, 0);
  for (int q = 0; q < pl->p; ++q) memcpy(blobs.data() + (size_t)q * kIpcSetBytes + 64, handles + 64 * (size_t)q, 64);
  return tffft_plan_ipc_attach(pl, blobs.data());
}

int tffft_plan_create_ex(int n0, int n1, int n2, int dtype, int pattern, int flags, tffft_comm_t comm,
                         tffft_plan_t* out) {
  return tffft_plan_create_batched(n0, n1, n2, dtype, pattern, flags, 1, comm, out);
}

int tffft_plan_create_batched(int n0, int n1, int n2, int dtype, int pattern, int flags, int batch,
                              tffft_comm_t comm, tffft_plan_t* out) {
  // TMA column passes: explicit flag = every supported pass; environment
  // defaults = the measured winner (float32 column passes, profiles/r01s2/tma_cols.txt, r01s6/f32_stage1b_tma.txt)
  // unless TFFFT_TMA_COLS says otherwise
  int tma_cols = 0;
  if (flags < 0) {
    flags = env_flags();
    const char* tc = getenv("TFFFT_TMA_COLS");
    tma_cols = (flags & TFFFT_FLAG_TMA_COLUMNS) ? 1 : (tc ? 0 : 2);
  } else {
    tma_cols = (flags & TFFFT_FLAG_TMA_COLUMNS) ? 1 : 0;
  }
  if (!comm || !out) return fail(TFFFT_ERR_CONFIGURATION, "null argument");
  const int p = comm->p;
  // layout.py:63-66 (powers of two), layout.py:83-93 (validate)
  const int ns[3] = {n0, n1, n2};
  const char* nm[3] = {"n0", "n1", "n2"};
  for (int a = 0; a < 3; ++a) {
    if (!pow2(ns[a])) return fail(TFFFT_ERR_CONFIGURATION, "%s must be a positive power of two, got %d", nm[a], ns[a]);
    if (ns[a] < 2) return fail(TFFFT_ERR_CONFIGURATION, "%s must be a power of two >= 2, got %d", nm[a], ns[a]);
    if (ns[a] > (1 << kMaxLog)) return fail(TFFFT_ERR_SIZE, "%s=%d exceeds the supported maximum %d", nm[a], ns[a], 1 << kMaxLog);
  }
  if (n0 % p) return fail(TFFFT_ERR_CONFIGURATION, "p does not divide n0 (%d does not divide %d)", p, n0);
  if (n1 % p) return fail(TFFFT_ERR_CONFIGURATION, "p does not divide n1 (%d does not divide %d)", p, n1);
  if (dtype != TFFFT_F64 && dtype != TFFFT_F32) return fail(TFFFT_ERR_CONFIGURATION, "unknown dtype %d", dtype);
  const int strategy = (flags & TFFFT_FLAG_TRANSPOSE) ? 1 : 0;
  // kernels address the local spectral slab with 32-bit element offsets
  if ((long long)(n0 / p) * n1 * (n2 / 2 + 1) >= (1LL << 32))
    return fail(TFFFT_ERR_SIZE, "local slab of %lld complex elements exceeds 2^32; use more ranks",
                (long long)(n0 / p) * n1 * (n2 / 2 + 1));
  if (pattern != TFFFT_PAIRWISE && pattern != TFFFT_COLLECTIVE)
    return fail(TFFFT_ERR_CONFIGURATION, "unknown comm pattern %d", pattern);
  if (batch < 1) return fail(TFFFT_ERR_CONFIGURATION, "batch must be >= 1, got %d", batch);
  if (p == 1 && (long long)batch * (n0 / p) * n1 * (n2 / 2 + 1) >= (1LL << 32))
    return fail(TFFFT_ERR_SIZE, "a p = 1 batch of %d fields exceeds 2^32 complex elements per launch", batch);

  // a failed create releases what it allocated (PlanDeleter -> tffft_plan_destroy)
  std::unique_ptr<tffft_plan_s, PlanDeleter> pl(new tffft_plan_s());
  pl->comm = comm;
  pl->n0 = n0; pl->n1 = n1; pl->n2 = n2;
  pl->p = p; pl->rank = comm->rank; pl->dtype = dtype; pl->pattern = pattern;
  pl->L0 = ilog2(n0); pl->L1 = ilog2(n1); pl->L2h = ilog2(n2) - 1;
  pl->n0p = n0 / p; pl->n1p = n1 / p; pl->n2c = n2 / 2 + 1;
  pl->esz = dtype == TFFFT_F64 ? 16 : 8;
  pl->batch = batch;
  pl->strategy = strategy;
  pl->tma_cols = strategy == 0 ? tma_cols : 0;
  CUDA_TRY(cudaSetDevice(comm->device));

  size_t ws = 0;
  TRY(upload_table(pass_table(pl->L0), dtype, &pl->tw0, &ws));
  TRY(upload_table(pass_table(pl->L1), dtype, &pl->tw1, &ws));
  TRY(upload_table(pass_table(pl->L2h), dtype, &pl->tw2, &ws));
  TRY(upload_table(pass_table(pl->L2h, r2c_radix_bits(pl->L2h, pl->esz / 2)), dtype, &pl->tw2r, &ws));
  TRY(upload_table(pass_table(pl->L2h, c2r_radix_bits(pl->L2h, pl->esz / 2)), dtype, &pl->tw2c, &ws));
  TRY(upload_table(post_table(n2), dtype, &pl->tw2post, &ws));
  if (pl->L0 == 11 || pl->L1 == 11) {
    TRY(upload_table(pass_table(10), dtype, &pl->tw10, &ws));
    TRY(upload_table(post_table(2048), dtype, &pl->twh11, &ws));
  }
  CUDA_TRY(cudaMalloc(&pl->col_ticket, sizeof(unsigned long long)));
  const size_t planes = (size_t)batch * pl->n0p;  // statistics records: every plane of the batch
  CUDA_TRY(cudaMalloc(&pl->stats, sizeof(unsigned long long) * 3 * planes));
  CUDA_TRY(cudaMemset(pl->stats, 0, sizeof(unsigned long long) * 3 * planes));
  ws += sizeof(unsigned long long) * 3 * planes;
  CUDA_TRY(cudaMalloc(&pl->row_stats, sizeof(double) * 3 * planes * pl->n1));
  ws += sizeof(double) * 3 * planes * pl->n1;
  if (p == 1 && strategy == 1) {  // TRANSPOSE packs even on one rank (exchange.py:195-219)
    const size_t sb = (size_t)pl->n0p * pl->n1p * pl->n2c * pl->esz;
    CUDA_TRY(cudaMalloc(&pl->bs[0].staging, sb));
    ws += sb;
  }
  if (p > 1) {
    // a batched plan pipelines two buffer sets (component c's exchange runs on
    // the exchange stream while component c+1's stage 1 fills the other set)
    pl->nsets = (batch > 1 && strategy == 0) ? 2 : 1;
    const size_t sb = (size_t)p * pl->n0p * pl->n1p * pl->n2c * pl->esz;
    const unsigned evflags = cudaEventDisableTiming | (comm->kind == COMM_IPC ? cudaEventInterprocess : 0);
    for (int st = 0; st < pl->nsets; ++st) {
      BufSet& B = pl->bs[st];
      CUDA_TRY(cudaMalloc(&B.staging, sb));
      CUDA_TRY(cudaMalloc(&B.landing, sb));
      ws += 2 * sb;
      B.peer_staging.assign(p, nullptr);
      B.peer_landing.assign(p, nullptr);
      B.peer_staging[pl->rank] = B.staging;
      B.peer_landing[pl->rank] = B.landing;
      if (comm->kind == COMM_IPC) {  // events other processes open through cudaIpcOpenEventHandle
        B.ready.assign(p, nullptr);
        B.done.assign(p, nullptr);
        CUDA_TRY(cudaEventCreateWithFlags(&B.ready[pl->rank], evflags));
        CUDA_TRY(cudaEventCreateWithFlags(&B.done[pl->rank], evflags));
        B.own_events = true;
      }
    }
    {  // exchange stream + hand-off events: batched pipeline, chunked forward
      CUDA_TRY(cudaStreamCreateWithFlags(&pl->xstream, cudaStreamNonBlocking));
      for (int st = 0; st < 2; ++st) {
        CUDA_TRY(cudaEventCreateWithFlags(&pl->ev_s1[st], cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&pl->ev_x[st], cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&pl->ev_s3[st], cudaEventDisableTiming));
      }
    }
    const bool ps = (flags & TFFFT_FLAG_PEER_STORES) && strategy == 0;
    // chunked forward exchange: on NCCL by default (the NVLink transfer of
    // plane chunk c overlaps stage 1 of chunk c+1), opt-in on the fabrics
    if (strategy == 0 && !ps && pl->nsets == 1 && pl->n0p >= 2 &&
        ((flags & TFFFT_FLAG_CHUNKED_EXCHANGE) || comm->kind == COMM_NCCL)) {
      static const int env = [] {
        const char* e = getenv("TFFFT_XCHUNKS");
        return e ? atoi(e) : 0;
      }();
      pl->xchunks = std::max(1, std::min(env > 0 ? env : 4, pl->n0p));
    }
    if (comm->kind == COMM_LOCAL) {
      pl->seq = comm->plan_seq++;
      pl->peer_stores = ps;
      TRY(fabric_setup_local(pl.get()));
      for (int st = 0; st < pl->nsets; ++st) {
        TRY(build_pull_list(pl.get(), st));
        TRY(build_band_dst(pl.get(), st));
      }
    } else {
      // NCCL: peer stores once tffft_plan_ipc_attach mapped the peers' landing
      // buffers; IPC: the exchange needs the attach (peers' staging, landing, events)
      pl->peer_stores_wanted = ps;
      for (int st = 0; st < pl->nsets; ++st) TRY(build_band_dst(pl.get(), st));
    }
  }
  // stage 3 as an L2-resident four-step when the n0 columns are long (fourstep.cuh)
  {
    // measured at 1024^3 (profiles/r01_*): the four-step moves exactly the
    // algorithmic bytes with 1 KB row visits but issues ~60% more instructions per
    // element than the direct 8-column kernel, which is faster today; opt-in
    // with TFFFT_FOURSTEP=1.
    // optional schedules are single-rank kernels (no staging / landing addressing)
    const int la = ((flags & TFFFT_FLAG_FOURSTEP_STAGE3) && p == 1 && strategy == 0 && batch == 1) ? fourstep_la(pl->L0) : 0;
    if (la > 0) {
      static const char* env_g = getenv("TFFFT_FS_G");
      const long long ncols = (long long)pl->n1p * pl->n2c;
      long long G = env_g ? atoll(env_g) : 1024;
      G = std::max<long long>(kFsMaxW, (G / kFsMaxW) * kFsMaxW);
      G = std::min<long long>(G, ((ncols + kFsMaxW - 1) / kFsMaxW) * kFsMaxW);
      pl->fs_la = la;
      pl->fs_G = (int)G;
      pl->fs_groups = (int)((ncols + G - 1) / G);
      const size_t sb = (size_t)kFsSlots * n0 * G * pl->esz;
      CUDA_TRY(cudaMalloc(&pl->fs_scratch, sb));
      CUDA_TRY(cudaMalloc(&pl->fs_counters, sizeof(unsigned) * (1 + 2 * (size_t)pl->fs_groups)));
      ws += sb + sizeof(unsigned) * (1 + 2 * (size_t)pl->fs_groups);
      TRY(upload_table(pass_table(la), dtype, &pl->fs_twA, &ws));
      TRY(upload_table(pass_table(pl->L0 - la), dtype, &pl->fs_twB, &ws));
      TRY(upload_table(full_table(n0), dtype, &pl->fs_twN, &ws));
    }
  }
  {
    // measured at 1024^3 (profiles/r01_*): the fused persistent stage 1 keeps the
    // planes in L2 but its mixed row/column tasks run at lower occupancy; the two
    // streaming kernels are faster today, so fusion is opt-in (TFFFT_FUSE=1)
    if ((flags & TFFFT_FLAG_FUSED_STAGE1) && p == 1 && strategy == 0 && batch == 1 &&
        stage1_fused_supported(pl->L2h, pl->L1)) {
      pl->s1_fused = true;
      CUDA_TRY(cudaMalloc(&pl->s1_counters, sizeof(unsigned) * (1 + 2 * (size_t)pl->n0p)));
      ws += sizeof(unsigned) * (1 + 2 * (size_t)pl->n0p);
    }
  }
  pl->workspace = ws;
  *out = pl.release();
  return TFFFT_OK;
}

int tffft_plan_workspace_bytes(tffft_plan_t pl, size_t* b) {
  if (!pl || !b) return fail(TFFFT_ERR_CONFIGURATION, "null argument");
  *b = pl->workspace;
  return TFFFT_OK;
}

int tffft_plan_sizes(tffft_plan_t pl, int64_t* re, int64_t* sp) {
  if (!pl || !re || !sp) return fail(TFFFT_ERR_CONFIGURATION, "null argument");
  *re = (int64_t)pl->n0p * pl->n1 * pl->n2;
  *sp = (int64_t)pl->n1p * pl->n0 * pl->n2c;
  return TFFFT_OK;
}

static void free_events(tffft_plan_t pl) {
  for (auto& ev : pl->events)
    for (auto& e : ev.e)
      if (e) cudaEventDestroy(e);
  pl->events.clear();
  pl->event_next = 0;
}

// fold one recorded call into the stage totals
// (forward: stage1, exchange, stage3; inverse: stage3', exchange, stage1')
static int harvest(tffft_plan_t pl, StageEvents& ev) {
  if (!ev.pending) return TFFFT_OK;
  CUDA_TRY(cudaEventSynchronize(ev.e[3]));
  float a, b, c;
  CUDA_TRY(cudaEventElapsedTime(&a, ev.e[0], ev.e[1]));
  CUDA_TRY(cudaEventElapsedTime(&b, ev.e[1], ev.e[2]));
  CUDA_TRY(cudaEventElapsedTime(&c, ev.e[2], ev.e[3]));
  pl->stage_ms[ev.forward ? 0 : 2] += a;
  pl->stage_ms[1] += b;
  pl->stage_ms[ev.forward ? 2 : 0] += c;
  ev.pending = false;
  return TFFFT_OK;
}

int tffft_plan_destroy(tffft_plan_t pl) {
  if (!pl) return TFFFT_OK;
  cudaSetDevice(pl->comm->device);
  if (pl->xstream) cudaStreamSynchronize(pl->xstream);
  free_events(pl);
  cudaFree(pl->tw0); cudaFree(pl->tw1); cudaFree(pl->tw2); cudaFree(pl->tw2r); cudaFree(pl->tw2c); cudaFree(pl->tw2post); cudaFree(pl->tw10); cudaFree(pl->twh11);
  cudaFree(pl->stats); cudaFree(pl->row_stats);
  for (void* m : pl->ipc_opened) cudaIpcCloseMemHandle(m);
  for (cudaEvent_t e : pl->ipc_events) cudaEventDestroy(e);
  for (auto& B : pl->bs) {
    cudaFree(B.staging); cudaFree(B.landing); cudaFree(B.pull_ptrs); cudaFree(B.band_dst);
    if (B.own_events && !B.ready.empty()) {
      // own events (the local fabric's peers' entries belong to the peers' plans)
      if (B.ready[pl->rank]) cudaEventDestroy(B.ready[pl->rank]);
      if (B.done[pl->rank]) cudaEventDestroy(B.done[pl->rank]);
    }
  }
  for (int st = 0; st < 2; ++st) {
    if (pl->ev_s1[st]) cudaEventDestroy(pl->ev_s1[st]);
    if (pl->ev_x[st]) cudaEventDestroy(pl->ev_x[st]);
    if (pl->ev_s3[st]) cudaEventDestroy(pl->ev_s3[st]);
  }
  if (pl->xstream) cudaStreamDestroy(pl->xstream);
  cudaFree(pl->fs_scratch); cudaFree(pl->fs_counters); cudaFree(pl->fs_twA); cudaFree(pl->fs_twB);
  cudaFree(pl->fs_twN);
  cudaFree(pl->s1_counters);
  cudaFree(pl->col_ticket);
  cudaFree(pl->barrier_word);
  cudaFree(pl->check_acc);
  delete pl;
  return TFFFT_OK;
}

static int check_ptr(const void* ptr, const char* what, size_t align) {
  if (!ptr) return fail(TFFFT_ERR_CONTRACT, "%s is null", what);
  if (reinterpret_cast<uintptr_t>(ptr) % align)
    return fail(TFFFT_ERR_CONTRACT, "%s must be %zu-byte aligned", what, align);
  return TFFFT_OK;
}

static int begin_events(tffft_plan_t pl, bool fwd, cudaStream_t s, StageEvents** ev) {
  *ev = nullptr;
  if (!pl->timing) return TFFFT_OK;
  if (pl->events.empty()) {  // timing enabled without set_timing (defensive)
    pl->events.resize(kEventRing);
    for (auto& x : pl->events)
      for (auto& e : x.e) CUDA_TRY(cudaEventCreate(&e));
  }
  StageEvents& e = pl->events[pl->event_next];
  pl->event_next = (pl->event_next + 1) % kEventRing;
  TRY(harvest(pl, e));  // a slot still pending from kEventRing calls ago
  e.forward = fwd;
  e.pending = true;
  *ev = &e;
  CUDA_TRY(cudaEventRecord(e.e[0], s));
  return TFFFT_OK;
}

#define MARK(ev, i, s) \
  if (ev) CUDA_TRY(cudaEventRecord((ev)->e[i], s));

// NVTX ranges around each call and stage (SURVEY.md §5 tracing): header-only
// NVTX3, a no-op unless a tool (ncu --nvtx, nsys) injects itself.
// e.g. ncu --nvtx --nvtx-include "tffft.forward/stage3/" ...
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// ---- orchestration ---------------------------------------------------------
static size_t real_bytes(tffft_plan_t pl) { return (size_t)pl->n0p * pl->n1 * pl->n2 * (pl->esz / 2); }
static size_t spec_bytes(tffft_plan_t pl) { return (size_t)pl->n0p * pl->n1 * pl->n2c * pl->esz; }

static int check_ready(tffft_plan_t pl) {
  if (pl->p > 1 && pl->comm->kind == COMM_IPC && !pl->ipc_attached)
    return fail(TFFFT_ERR_PROTOCOL, "IPC plan used before tffft_plan_ipc_attach");
  if (pl->comm->aborted) return fail(TFFFT_ERR_TRANSPORT, "communicator aborted");
  return TFFFT_OK;
}

// stage 1 (dfft.py:161-163) of `nf` fields at (real, spec): r2c rows + n1 columns
// planes per chunk of the plane-interleaved stage 1 (TFFFT_S1_CHUNK, 0 = off):
// the n1 columns of a chunk run right after its rows, while the chunk is
// still L2-resident, so the column pass reads and overwrites it in L2
static int s1_chunk(tffft_plan_t pl) {
  static const int v = [] {
    const char* e = getenv("TFFFT_S1_CHUNK");
    return e ? atoi(e) : 0;
  }();
  return (v > 0 && pl->p == 1) ? v : 0;
}

static int fwd_stage1(tffft_plan_t pl, const void* real, void* spec, int nf, cudaStream_t s) {
  NvtxRange r("stage1");
  if (pl->s1_fused) return stage1_fused(pl, const_cast<void*>(real), spec, true, s);
  const int planes = nf * pl->n0p, K = s1_chunk(pl);
  if (K > 0 && K < planes) {
    const size_t rb = (size_t)pl->n1 * pl->n2 * (pl->esz / 2), sb = (size_t)pl->n1 * pl->n2c * pl->esz;
    for (int a = 0; a < planes; a += K) {
      const int k = std::min(K, planes - a);
      const char* rr = static_cast<const char*>(real) + (size_t)a * rb;
      char* ss = static_cast<char*>(spec) + (size_t)a * sb;
      CUDA_TRY(r2c_launch(pl, row_params(pl, const_cast<char*>(rr), ss, k, a), s));
      TRY(stage1_columns(pl, ss, false, s, k));
    }
    return TFFFT_OK;
  }
  CUDA_TRY(r2c_launch(pl, row_params(pl, const_cast<void*>(real), spec, planes, 0), s));
  return stage1_columns(pl, spec, false, s, planes);
}
// stage 1' (dfft.py:206-209) of one field (component c of the batch) or, at
// p = 1, of `nf` fields: n1 columns + c2r rows with 1/(n0 n1 n2)
static int inv_stage1(tffft_plan_t pl, void* spec, void* real, int nf, int c, cudaStream_t s) {
  NvtxRange r("stage1");
  if (pl->s1_fused) return stage1_fused(pl, real, spec, false, s);
  const int planes = nf * pl->n0p, K = s1_chunk(pl);
  if (K > 0 && K < planes) {
    const size_t rb = (size_t)pl->n1 * pl->n2 * (pl->esz / 2), sb = (size_t)pl->n1 * pl->n2c * pl->esz;
    for (int a = 0; a < planes; a += K) {
      const int k = std::min(K, planes - a);
      char* ss = static_cast<char*>(spec) + (size_t)a * sb;
      TRY(stage1_columns(pl, ss, true, s, k));
      CUDA_TRY(c2r_launch(pl, row_params(pl, static_cast<char*>(real) + (size_t)a * rb, ss, k,
                                         (long long)c * pl->n0p + a), s));
    }
    return TFFFT_OK;
  }
  TRY(stage1_columns(pl, spec, true, s, nf * pl->n0p));
  TRY(landing_consumed(pl, s));
  CUDA_TRY(c2r_launch(pl, row_params(pl, real, spec, nf * pl->n0p, (long long)c * pl->n0p), s));
  return TFFFT_OK;
}

static int forward_field(tffft_plan_t pl, const void* real, void* spec, int nf, cudaStream_t s, StageEvents* ev) {
  TRY(guard_outgoing(pl, s));
  TRY(fwd_stage1(pl, real, spec, nf, s));
  MARK(ev, 1, s);
  if (pl->strategy == 1) {
    // TRANSPOSE (exchange.py:195-219): pack -> contiguous exchange -> unpack
    TRY(pack_forward(pl, spec, s));
    TRY(exchange(pl, s));
    TRY(unpack_forward(pl, spec, s));
    MARK(ev, 2, s);
    TRY(stage3_flipped(pl, spec, false, s));
    MARK(ev, 3, s);
    return TFFFT_OK;
  }
  {  // exchange (exchange.py:263-276)
    NvtxRange r("exchange");
    TRY(exchange(pl, s));
  }
  MARK(ev, 2, s);
  {  // stage 3: strided columns (dfft.py:170-171)
    NvtxRange r("stage3");
    TRY(stage3_columns(pl, spec, false, s));
    TRY(landing_consumed(pl, s));
  }
  MARK(ev, 3, s);
  return TFFFT_OK;
}

static int inverse_field(tffft_plan_t pl, void* spec, void* real, int nf, int c, cudaStream_t s, StageEvents* ev) {
  if (pl->s1_fused)  // the fused kernel max-reduces into the per-plane statistics
    CUDA_TRY(cudaMemsetAsync(pl->stats, 0, sizeof(unsigned long long) * 3 * pl->n0p, s));
  TRY(guard_outgoing(pl, s));
  if (pl->strategy == 1) {
    TRY(stage3_flipped(pl, spec, true, s));
    MARK(ev, 1, s);
    // TRANSPOSE (exchange.py:222-260): pack -> contiguous exchange -> un-transpose
    TRY(pack_inverse(pl, spec, s));
    TRY(exchange(pl, s));
    TRY(unpack_inverse(pl, spec, s));
    MARK(ev, 2, s);
  } else {
    {  // stage 3' (dfft.py:196-197)
      NvtxRange r("stage3");
      TRY(stage3_columns(pl, spec, true, s));
    }
    MARK(ev, 1, s);
    {  // exchange (exchange.py:279-290)
      NvtxRange r("exchange");
      TRY(exchange(pl, s));
    }
    MARK(ev, 2, s);
  }
  TRY(inv_stage1(pl, spec, real, nf, c, s));
  MARK(ev, 3, s);
  return TFFFT_OK;
}

// Chunked forward at p > 1 (one field): stage 1 runs plane chunk after plane
// chunk on the caller's stream s; each chunk's part of every band is exchanged
// on the exchange stream x as soon as the chunk is produced, so the transfer
// of chunk c overlaps stage 1 of chunk c+1 (a band's plane range is contiguous
// in staging and landing).  Stage 3 waits for the last chunk.
static int forward_chunked(tffft_plan_t pl, const void* real, void* spec, cudaStream_t s, StageEvents* ev) {
  cudaStream_t x = pl->xstream;
  pl->cur = 0;
  TRY(guard_outgoing(pl, s));
  const int C = pl->xchunks, m = (pl->n0p + C - 1) / C;
  const size_t rb = (size_t)pl->n1 * pl->n2 * (pl->esz / 2), sb = (size_t)pl->n1 * pl->n2c * pl->esz;
  {
    NvtxRange r("stage1+exchange");
    for (int a = 0, k = 0; a < pl->n0p; a += m, ++k) {
      const int cnt = std::min(m, pl->n0p - a);
      char* sp = static_cast<char*>(spec) + (size_t)a * sb;
      CUDA_TRY(r2c_launch(pl, row_params(pl, const_cast<char*>(static_cast<const char*>(real) + (size_t)a * rb), sp,
                                         cnt, a), s));
      TRY(stage1_columns(pl, sp, false, s, cnt, a));
      CUDA_TRY(cudaEventRecord(pl->ev_s1[k & 1], s));
      CUDA_TRY(cudaStreamWaitEvent(x, pl->ev_s1[k & 1], 0));
      TRY(exchange(pl, x, a, cnt));
    }
    CUDA_TRY(cudaEventRecord(pl->ev_x[0], x));
    CUDA_TRY(cudaStreamWaitEvent(s, pl->ev_x[0], 0));
  }
  MARK(ev, 1, s);
  MARK(ev, 2, s);
  {
    NvtxRange r("stage3");
    TRY(stage3_columns(pl, spec, false, s));
  }
  MARK(ev, 3, s);
  return TFFFT_OK;
}

// Batched p > 1 (STRIDED): a two-deep software pipeline over the fields.  The
// stages run on the caller's stream s, the exchanges on the plan's exchange
// stream x; field c uses buffer set c % 2, so field c's exchange overlaps
// field c+1's producing stage.  Enqueue order on s:
//   produce(0), produce(1), consume(0), produce(2), consume(1), ...
// Hand-offs: x waits produce(c) (ev_s1); consume(c) waits exchange(c) (ev_x);
// produce(c+2) reuses the set after exchange(c) read its staging (ev_x).
// Every rank enqueues in the same order, so the fabric's host barriers and
// NCCL's per-communicator ordering see the same sequence on every rank.
extern "C++" {
template <class Produce, class Consume>
static int pipeline(tffft_plan_t pl, cudaStream_t s, Produce produce, Consume consume) {
  cudaStream_t x = pl->xstream;
  const int B = pl->batch;
  for (int c = 0; c <= B; ++c) {
    if (c < B) {
      const int st = c & 1;
      pl->cur = st;
      if (c >= 2) CUDA_TRY(cudaStreamWaitEvent(s, pl->ev_x[st], 0));
      if (!fabric_kind(pl) && pl->peer_stores) {
        // NCCL: the guard barrier goes on the exchange stream too, so every NCCL
        // operation of the communicator is issued on one stream in one order
        CUDA_TRY(cudaEventRecord(pl->ev_s3[st], s));
        CUDA_TRY(cudaStreamWaitEvent(x, pl->ev_s3[st], 0));
        TRY(guard_outgoing(pl, x));
        CUDA_TRY(cudaEventRecord(pl->ev_x[st], x));
        CUDA_TRY(cudaStreamWaitEvent(s, pl->ev_x[st], 0));
      } else {
        TRY(guard_outgoing(pl, s));
      }
      TRY(produce(c));
      CUDA_TRY(cudaEventRecord(pl->ev_s1[st], s));
      CUDA_TRY(cudaStreamWaitEvent(x, pl->ev_s1[st], 0));
      {
        NvtxRange r("exchange");
        TRY(exchange(pl, x));
      }
      CUDA_TRY(cudaEventRecord(pl->ev_x[st], x));
    }
    if (c >= 1) {
      const int st = (c - 1) & 1;
      pl->cur = st;
      CUDA_TRY(cudaStreamWaitEvent(s, pl->ev_x[st], 0));
      TRY(consume(c - 1));
      CUDA_TRY(cudaEventRecord(pl->ev_s3[st], s));
    }
  }
  pl->cur = 0;
  return TFFFT_OK;
}

}  // extern "C++"

// Chunked inverse at p > 1 (one field, component c of the batch): stage 3'
// writes every band, then the bands are exchanged plane chunk after plane
// chunk on the exchange stream x, and stage 1' (n1 columns + c2r rows) of
// chunk k runs on the caller's stream s as soon as that chunk has landed, so
// it overlaps the transfer of chunk k+1 -- the mirror of forward_chunked (the
// consuming stage, not the producing one, hides the exchange here: a column
// of stage 3' feeds every plane, while a plane of stage 1' needs one chunk).
static int inverse_chunked(tffft_plan_t pl, void* spec, void* real, int c, cudaStream_t s, StageEvents* ev) {
  cudaStream_t x = pl->xstream;
  pl->cur = 0;
  TRY(guard_outgoing(pl, s));
  {
    NvtxRange r("stage3");
    TRY(stage3_columns(pl, spec, true, s));
  }
  MARK(ev, 1, s);
  CUDA_TRY(cudaEventRecord(pl->ev_s1[0], s));
  CUDA_TRY(cudaStreamWaitEvent(x, pl->ev_s1[0], 0));
  const int C = pl->xchunks, m = (pl->n0p + C - 1) / C;
  const size_t rb = (size_t)pl->n1 * pl->n2 * (pl->esz / 2), sb = (size_t)pl->n1 * pl->n2c * pl->esz;
  {
    NvtxRange r("exchange+stage1");
    for (int a = 0, k = 0; a < pl->n0p; a += m, ++k) {
      const int cnt = std::min(m, pl->n0p - a);
      TRY(exchange(pl, x, a, cnt));
      CUDA_TRY(cudaEventRecord(pl->ev_x[k & 1], x));
      CUDA_TRY(cudaStreamWaitEvent(s, pl->ev_x[k & 1], 0));
      char* sp = static_cast<char*>(spec) + (size_t)a * sb;
      TRY(stage1_columns(pl, sp, true, s, cnt, a));
      CUDA_TRY(c2r_launch(pl, row_params(pl, static_cast<char*>(real) + (size_t)a * rb, sp, cnt,
                                         (long long)c * pl->n0p + a), s));
    }
  }
  MARK(ev, 2, s);
  MARK(ev, 3, s);
  return TFFFT_OK;
}

int tffft_forward(tffft_plan_t pl, const void* real_in, void* spec_out, void* stream) {
  if (!pl) return fail(TFFFT_ERR_CONFIGURATION, "null plan");
  TRY(check_ptr(real_in, "real_in", pl->esz));
  TRY(check_ptr(spec_out, "spec_out", pl->esz));
  TRY(check_ready(pl));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CUDA_TRY(cudaSetDevice(pl->comm->device));
  NvtxRange call("tffft.forward");
  const char* real = static_cast<const char*>(real_in);
  char* spec = static_cast<char*>(spec_out);
  if (pl->p == 1 && pl->strategy == 0) {  // every field of the batch in the same launches
    StageEvents* ev;
    TRY(begin_events(pl, true, s, &ev));
    return forward_field(pl, real, spec, pl->batch, s, ev);
  }
  if (pl->nsets == 1) {  // one field at a time
    for (int c = 0; c < pl->batch; ++c) {
      StageEvents* ev;
      TRY(begin_events(pl, true, s, &ev));
      pl->cur = 0;
      if (pl->xchunks > 1)
        TRY(forward_chunked(pl, real + c * real_bytes(pl), spec + c * spec_bytes(pl), s, ev));
      else
        TRY(forward_field(pl, real + c * real_bytes(pl), spec + c * spec_bytes(pl), 1, s, ev));
    }
    return TFFFT_OK;
  }
  StageEvents* ev;  // pipelined: the whole call is timed as stage 1 + stage 3
  TRY(begin_events(pl, true, s, &ev));
  MARK(ev, 1, s);
  MARK(ev, 2, s);
  TRY(pipeline(
      pl, s, [&](int c) { return fwd_stage1(pl, real + c * real_bytes(pl), spec + c * spec_bytes(pl), 1, s); },
      [&](int c) {
        NvtxRange r("stage3");
        TRY(stage3_columns(pl, spec + c * spec_bytes(pl), false, s));
        return landing_consumed(pl, s);
      }));
  MARK(ev, 3, s);
  return TFFFT_OK;
}

int tffft_inverse(tffft_plan_t pl, void* spec_inout, void* real_out, void* stream) {
  if (!pl) return fail(TFFFT_ERR_CONFIGURATION, "null plan");
  TRY(check_ptr(spec_inout, "spec_inout", pl->esz));
  TRY(check_ptr(real_out, "real_out", pl->esz));
  TRY(check_ready(pl));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CUDA_TRY(cudaSetDevice(pl->comm->device));
  NvtxRange call("tffft.inverse");
  char* spec = static_cast<char*>(spec_inout);
  char* real = static_cast<char*>(real_out);
  if (pl->p == 1 && pl->strategy == 0) {
    StageEvents* ev;
    TRY(begin_events(pl, false, s, &ev));
    TRY(inverse_field(pl, spec, real, pl->batch, 0, s, ev));
  } else if (pl->nsets == 1) {
    for (int c = 0; c < pl->batch; ++c) {
      StageEvents* ev;
      TRY(begin_events(pl, false, s, &ev));
      pl->cur = 0;
      if (pl->xchunks > 1 && !pl->peer_stores && pl->strategy == 0 && !pl->s1_fused)
        TRY(inverse_chunked(pl, spec + c * spec_bytes(pl), real + c * real_bytes(pl), c, s, ev));
      else
        TRY(inverse_field(pl, spec + c * spec_bytes(pl), real + c * real_bytes(pl), 1, c, s, ev));
    }
  } else {
    StageEvents* ev;
    TRY(begin_events(pl, false, s, &ev));
    MARK(ev, 1, s);
    MARK(ev, 2, s);
    TRY(pipeline(
        pl, s,
        [&](int c) {
          NvtxRange r("stage3");
          return stage3_columns(pl, spec + c * spec_bytes(pl), true, s);
        },
        [&](int c) { return inv_stage1(pl, spec + c * spec_bytes(pl), real + c * real_bytes(pl), 1, c, s); }));
    MARK(ev, 3, s);
  }
  if (pl->deferred_check) {  // the Hermitian check of this call, folded on the device
    if (!pl->s1_fused) {
      reduce_row_stats_kernel<<<pl->n0p * pl->batch, 256, 0, s>>>(pl->row_stats, pl->n1, pl->stats);
      pl->launches++;
    }
    consistency_fold_kernel<<<1, 256, 0, s>>>(pl->stats, pl->n0p * pl->batch, (double)pl->n2,
                                              pl->dtype == TFFFT_F64 ? 1e-9 : 1e-4, pl->check_acc);
    pl->launches++;
    CUDA_TRY(cudaGetLastError());
    pl->deferred_calls++;
  }
  pl->last_inverse_stream = s;
  pl->inverse_ran = true;
  return TFFFT_OK;
}

static int reset_check_acc(tffft_plan_t pl, cudaStream_t s) {
  const unsigned long long init[4] = {0ull, 0ull, ~0ull, 0ull};
  CUDA_TRY(cudaMemcpyAsync(pl->check_acc, init, sizeof(init), cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return TFFFT_OK;
}

// Deferred consistency (mode 1): every inverse folds its Hermitian check into
// a device accumulator instead of waiting for tffft_consistency; the verdict
// of all inverses since the last collect is read by tffft_consistency_collect.
int tffft_set_consistency_mode(tffft_plan_t pl, int deferred) {
  if (!pl) return fail(TFFFT_ERR_CONFIGURATION, "null plan");
  CUDA_TRY(cudaSetDevice(pl->comm->device));
  if (deferred && !pl->check_acc) CUDA_TRY(cudaMalloc(&pl->check_acc, 4 * sizeof(unsigned long long)));
  if (deferred) TRY(reset_check_acc(pl, nullptr));
  pl->deferred_check = deferred != 0;
  pl->deferred_calls = 0;
  return TFFFT_OK;
}

int tffft_consistency_collect(tffft_plan_t pl, double* residue, uint64_t* calls) {
  if (!pl || !residue) return fail(TFFFT_ERR_CONFIGURATION, "null argument");
  *residue = 0.0;
  if (calls) *calls = pl->deferred_calls;
  if (!pl->deferred_check) return fail(TFFFT_ERR_CONFIGURATION, "the plan is not in the deferred consistency mode");
  CUDA_TRY(cudaSetDevice(pl->comm->device));
  if (pl->last_inverse_stream || pl->inverse_ran) CUDA_TRY(cudaStreamSynchronize(pl->last_inverse_stream));
  unsigned long long h[4];
  CUDA_TRY(cudaMemcpy(h, pl->check_acc, sizeof(h), cudaMemcpyDeviceToHost));
  const uint64_t n = pl->deferred_calls;
  pl->deferred_calls = 0;
  TRY(reset_check_acc(pl, pl->last_inverse_stream));
  double r, ratio;
  memcpy(&r, &h[0], 8);
  memcpy(&ratio, &h[3], 8);
  *residue = r;
  if (h[1] > 0)
    return fail(TFFFT_ERR_CONSISTENCY,
                "bins 0 and n/2 must be real for a half spectrum: %llu plane(s) over the tolerance in %llu "
                "inverse call(s), first at field %llu plane %llu, worst %.3g x the tolerance",
                (unsigned long long)h[1], (unsigned long long)n, (unsigned long long)(h[2] / pl->n0p),
                (unsigned long long)(h[2] % pl->n0p), ratio);
  return TFFFT_OK;
}

// Debug aid (compute-sanitizer is closed on this pool): fill every
// plan-internal buffer that a stage reads after another stage or rank wrote
// it -- exchange staging and landing of every set, the c2r row records -- with
// 0xFF bytes (a NaN in either precision).  A kernel that reads an element
// nobody wrote, or reads it before it was written, then turns the output into
// NaN (tests/test_gpu_races.py).  Synchronous.
int tffft_plan_poison(tffft_plan_t pl) {
  if (!pl) return fail(TFFFT_ERR_CONFIGURATION, "null plan");
  CUDA_TRY(cudaSetDevice(pl->comm->device));
  CUDA_TRY(cudaDeviceSynchronize());
  const size_t band = band_bytes(pl);
  for (int st = 0; st < 2; ++st) {
    BufSet& B = pl->bs[st];
    const size_t sb = pl->p > 1 ? (size_t)pl->p * band : band;
    if (B.staging) CUDA_TRY(cudaMemset(B.staging, 0xFF, sb));
    if (B.landing) CUDA_TRY(cudaMemset(B.landing, 0xFF, sb));
  }
  if (!pl->s1_fused)
    CUDA_TRY(cudaMemset(pl->row_stats, 0xFF, sizeof(double) * 3 * (size_t)pl->batch * pl->n0p * pl->n1));
  CUDA_TRY(cudaDeviceSynchronize());
  return TFFFT_OK;
}

// Diagnostic: the exchange's NCCL calls as a one-rank loopback on `device` --
// a communicator of size 1 (ncclCommInitRank), one grouped ncclSend / ncclRecv
// pair to itself of `count` real elements of `dtype` (the PAIRWISE exchange
// above), one ncclAlltoAll (the COLLECTIVE exchange; skipped when the loaded
// NCCL lacks it), the one-int ncclAllReduce of the peer-store barrier and the
// async-error poll, all through the dlopen'ed function table.  Received data
// must equal what was sent.  NCCL refuses two ranks on one GPU, so on a
// one-GPU box this is as much of the NCCL path as can execute.
int tffft_nccl_loopback(int device, long long count, int dtype, int* ran_alltoall) {
  if (count < 1 || (dtype != TFFFT_F64 && dtype != TFFFT_F32))
    return fail(TFFFT_ERR_CONFIGURATION, "nccl_loopback: count %lld, dtype %d", count, dtype);
  NcclApi& api = nccl();
  if (!api.loaded) return fail(TFFFT_ERR_TRANSPORT, "NCCL unavailable: %s", api.err.c_str());
  CUDA_TRY(cudaSetDevice(device));
  const size_t rb = dtype == TFFFT_F64 ? 8 : 4, bytes = (size_t)count * rb;
  const ncclDataType_t dt = dtype == TFFFT_F64 ? ncclFloat64 : ncclFloat32;
  ncclUniqueId uid;
  NCCL_TRY(api.GetUniqueId(&uid));
  ncclComm_t comm = nullptr;
  NCCL_TRY(api.CommInitRank(&comm, 1, uid, 0));
  std::vector<unsigned char> h(bytes), back(bytes);
  for (size_t i = 0; i < bytes; ++i) h[i] = (unsigned char)((i * 2654435761u) >> 13);
  if (dtype == TFFFT_F64) {  // finite values: clear the exponent's top bits
    for (size_t i = 7; i < bytes; i += 8) h[i] &= 0x3f;
  } else {
    for (size_t i = 3; i < bytes; i += 4) h[i] &= 0x3f;
  }
  void *src = nullptr, *dst = nullptr, *dst2 = nullptr;
  int* flag = nullptr;
  cudaStream_t s = nullptr;
  int rc = TFFFT_OK;
  auto cleanup = [&] {
    if (s) cudaStreamDestroy(s);
    cudaFree(src); cudaFree(dst); cudaFree(dst2); cudaFree(flag);
    if (comm) api.CommDestroy(comm);
  };
#define LB_CUDA(expr)                                                                        \
  do {                                                                                       \
    cudaError_t _e = (expr);                                                                 \
    if (_e != cudaSuccess) {                                                                 \
      rc = fail(TFFFT_ERR_CUDA, "%s failed: %s", #expr, cudaGetErrorString(_e));             \
      cleanup();                                                                             \
      return rc;                                                                             \
    }                                                                                        \
  } while (0)
#define LB_NCCL(expr)                                                                        \
  do {                                                                                       \
    ncclResult_t _r = (expr);                                                                \
    if (_r != ncclSuccess) {                                                                 \
      rc = fail(TFFFT_ERR_TRANSPORT, "%s failed: %s", #expr, api.GetErrorString(_r));        \
      cleanup();                                                                             \
      return rc;                                                                             \
    }                                                                                        \
  } while (0)
  LB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  LB_CUDA(cudaMalloc(&src, bytes));
  LB_CUDA(cudaMalloc(&dst, bytes));
  LB_CUDA(cudaMalloc(&dst2, bytes));
  LB_CUDA(cudaMalloc(&flag, sizeof(int)));
  LB_CUDA(cudaMemcpyAsync(src, h.data(), bytes, cudaMemcpyHostToDevice, s));
  LB_CUDA(cudaMemsetAsync(dst, 0xFF, bytes, s));
  LB_CUDA(cudaMemsetAsync(dst2, 0xFF, bytes, s));
  LB_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), s));
  LB_NCCL(api.GroupStart());
  LB_NCCL(api.Send(src, (size_t)count, dt, 0, comm, s));
  LB_NCCL(api.Recv(dst, (size_t)count, dt, 0, comm, s));
  LB_NCCL(api.GroupEnd());
  if (api.AlltoAll) LB_NCCL(api.AlltoAll(src, dst2, (size_t)count, dt, comm, s));
  LB_NCCL(api.AllReduce(flag, flag, 1, ncclInt32, ncclSum, comm, s));
  LB_CUDA(cudaStreamSynchronize(s));
  ncclResult_t async_err = ncclSuccess;
  LB_NCCL(api.CommGetAsyncError(comm, &async_err));
  LB_NCCL(async_err);
  LB_CUDA(cudaMemcpy(back.data(), dst, bytes, cudaMemcpyDeviceToHost));
  if (memcmp(back.data(), h.data(), bytes) != 0) {
    rc = fail(TFFFT_ERR_TRANSPORT, "nccl_loopback: send/recv payload differs");
    cleanup();
    return rc;
  }
  if (api.AlltoAll) {
    LB_CUDA(cudaMemcpy(back.data(), dst2, bytes, cudaMemcpyDeviceToHost));
    if (memcmp(back.data(), h.data(), bytes) != 0) {
      rc = fail(TFFFT_ERR_TRANSPORT, "nccl_loopback: all-to-all payload differs");
      cleanup();
      return rc;
    }
  }
#undef LB_CUDA
#undef LB_NCCL
  if (ran_alltoall) *ran_alltoall = api.AlltoAll ? 1 : 0;
  cleanup();
  return TFFFT_OK;
}

int tffft_plan_batch(tffft_plan_t pl, int* batch) {
  if (!pl || !batch) return fail(TFFFT_ERR_CONFIGURATION, "null argument");
  *batch = pl->batch;
  return TFFFT_OK;
}

int tffft_set_timing(tffft_plan_t pl, int enable) {
  if (!pl) return fail(TFFFT_ERR_CONFIGURATION, "null plan");
  pl->timing = enable != 0;
  if (pl->timing && pl->events.empty()) {
    CUDA_TRY(cudaSetDevice(pl->comm->device));
    pl->events.resize(kEventRing);
    for (auto& x : pl->events)
      for (auto& e : x.e) CUDA_TRY(cudaEventCreate(&e));
  }
  return TFFFT_OK;
}

int tffft_stage_times(tffft_plan_t pl, double ms[3]) {
  if (!pl || !ms) return fail(TFFFT_ERR_CONFIGURATION, "null argument");
  for (auto& ev : pl->events) TRY(harvest(pl, ev));
  for (int i = 0; i < 3; ++i) ms[i] = pl->stage_ms[i];
  return TFFFT_OK;
}

int tffft_counters(tffft_plan_t pl, uint64_t b[3]) {
  if (!pl || !b) return fail(TFFFT_ERR_CONFIGURATION, "null argument");
  for (int i = 0; i < 3; ++i) b[i] = pl->counters[i];
  return TFFFT_OK;
}

int tffft_reset_instrumentation(tffft_plan_t pl) {
  if (!pl) return fail(TFFFT_ERR_CONFIGURATION, "null plan");
  for (auto& ev : pl->events) ev.pending = false;
  pl->stage_ms[0] = pl->stage_ms[1] = pl->stage_ms[2] = 0.0;
  pl->counters[0] = pl->counters[1] = pl->counters[2] = 0;
  pl->launches = 0;
  return TFFFT_OK;
}

int tffft_launch_count(tffft_plan_t pl, uint64_t* n) {
  if (!pl || !n) return fail(TFFFT_ERR_CONFIGURATION, "null argument");
  *n = pl->launches;
  return TFFFT_OK;
}

int tffft_consistency(tffft_plan_t pl, double* residue) {
  if (!pl || !residue) return fail(TFFFT_ERR_CONFIGURATION, "null argument");
  *residue = 0.0;
  if (!pl->inverse_ran) return TFFFT_OK;
  CUDA_TRY(cudaSetDevice(pl->comm->device));
  if (!pl->s1_fused) {  // fold the c2r row records into per-plane maxima
    reduce_row_stats_kernel<<<pl->n0p * pl->batch, 256, 0, pl->last_inverse_stream>>>(pl->row_stats, pl->n1, pl->stats);
    pl->launches++;
    CUDA_TRY(cudaGetLastError());
  }
  CUDA_TRY(cudaStreamSynchronize(pl->last_inverse_stream));
  const int planes = pl->n0p * pl->batch;  // every plane of the batch, field after field
  std::vector<double> st(3 * (size_t)planes);
  CUDA_TRY(cudaMemcpy(st.data(), pl->stats, st.size() * sizeof(double), cudaMemcpyDeviceToHost));
  double res = 0.0;
  int bad = -1;
  double bad_v = 0.0, bad_tol = 0.0;
  for (int i = 0; i < planes; ++i) {
    // kernels.py:222-223 (C2R_RESIDUE_TOL = 1e-9, calibrated for float64); float32
    // plans use 1e-4, which still flags an O(1) imaginary DC / Nyquist bin
    const double rtol = pl->dtype == TFFFT_F64 ? 1e-9 : 1e-4;
    const double tol = rtol * pl->n2 * std::sqrt(st[3 * i]);
    const double edge = st[3 * i + 1], r = st[3 * i + 2];
    res = std::max(res, r);
    if (bad < 0 && (edge > tol || r > tol)) {
      bad = i;
      bad_v = std::max(edge, r);
      bad_tol = tol;
    }
  }
  *residue = res;
  if (bad >= 0)
    return fail(TFFFT_ERR_CONSISTENCY,
                "bins 0 and n/2 must be real for a half spectrum (field %d, plane %d: imag %.3e > %.3e)",
                bad / pl->n0p, bad % pl->n0p, bad_v, bad_tol);
  return TFFFT_OK;
}

int tffft_exchange_schedule(int n0, int n1, int n2, int p, int rank, int64_t* ops, int64_t max_ops,
                            int64_t* nops) {
  if (!nops) return fail(TFFFT_ERR_CONFIGURATION, "null argument");
  if (p < 1 || rank < 0 || rank >= p || n0 % p || n1 % p)
    return fail(TFFFT_ERR_CONFIGURATION, "invalid geometry");
  const int64_t n0p = n0 / p, n1p = n1 / p, n2c = n2 / 2 + 1, band = n0p * n1p * n2c;
  int64_t cnt = 0;
  for (int d = 1; d < p; ++d) {
    const int q = (rank + d) % p;
    if (ops && cnt < max_ops) {
      ops[4 * cnt + 0] = q;
      ops[4 * cnt + 1] = (int64_t)q * band;  // staging[q]: my planes' band q, [i][j][k]
      ops[4 * cnt + 2] = (int64_t)q * band;  // landing[q]: rank q's planes' band rank, [i][j][k]
      ops[4 * cnt + 3] = band;
    }
    ++cnt;
  }
  *nops = cnt;
  if (ops && cnt > max_ops) return fail(TFFFT_ERR_CONFIGURATION, "ops buffer too small (%lld needed)", (long long)cnt);
  return TFFFT_OK;
}

int tffft_radix_schedule(int log2n, int* radices, int* npasses) {
  if (!npasses || log2n < 0 || log2n > kMaxLog) return fail(TFFFT_ERR_SIZE, "log2n out of range");
  *npasses = num_passes(log2n);
  if (radices)
    for (int p = 0; p < *npasses; ++p) radices[p] = 1 << pass_bits(log2n, p);
  return TFFFT_OK;
}

#pragma GCC visibility pop
}  // extern "C"
