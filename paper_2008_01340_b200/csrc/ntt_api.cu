// ntt_api.cu -- the C ABI of libntt (include/ntt.h): validation, planning,
// workspace management, the MU iteration driver, the nTT sweep, contraction /
// error, and the NCCL layer for the last-mode-partitioned multi-GPU sweep.
#include <dlfcn.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <memory>
#include <string>
#include <vector>

#include <nccl.h>

#include "../../include/ntt.h"
#include "common.cuh"
#include "kernels.h"
#include "mu_fused.h"
#include "mu_tc.h"

using namespace ntt;

// ----------------------------------------------------------------- NCCL (dlopen)
namespace {
struct NcclApi {
  bool loaded = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;

bool load_nccl() {
  if (g_nccl.loaded) return true;
  const char* env = getenv("NTT_NCCL_LIB");
  const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
  void* lib = nullptr;
  for (const char* nm : names) {
    if (!nm) continue;
    lib = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (lib) break;
  }
  if (!lib) return false;
#define SYM(f, n) g_nccl.f = reinterpret_cast<decltype(g_nccl.f)>(dlsym(lib, n)); if (!g_nccl.f) return false;
  SYM(GetUniqueId, "ncclGetUniqueId")
  SYM(CommInitRank, "ncclCommInitRank")
  SYM(CommDestroy, "ncclCommDestroy")
  SYM(AllReduce, "ncclAllReduce")
  SYM(Broadcast, "ncclBroadcast")
  SYM(GroupStart, "ncclGroupStart")
  SYM(GroupEnd, "ncclGroupEnd")
  SYM(CommSplit, "ncclCommSplit")
  SYM(GetErrorString, "ncclGetErrorString")
#undef SYM
  g_nccl.loaded = true;
  return true;
}
}  // namespace

// --------------------------------------------------------------------- handle
struct ntt_handle_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  int64_t l2_bytes = 126 << 20;
  unsigned long long* ptrace = nullptr;  // persistent-kernel phase stamps (NTT_PERSIST_TRACE)
  std::string err;
  int64_t launches = 0;
  int64_t collectives = 0;  // NCCL calls enqueued (ntt_collective_count)
  // internal scratch (grown, never shrunk)
  void* ws = nullptr;
  size_t ws_bytes = 0;
  // staging for host buffers
  void* stage = nullptr;
  size_t stage_bytes = 0;
  void* sweep = nullptr;  // ntt_decompose_bcd's H / W / cores buffers (kept across calls)
  size_t sweep_bytes = 0;
  double* host_part = nullptr;  // pinned host landing zone for small reductions
  size_t host_part_count = 0;
  // distributed
  int nranks = 1, rank = 0;
  // 2-D pr x pc process grid for the plain NMF (SURVEY s.8(e)); rank = ga * pc + gb.
  // comm_row: the pc ranks of grid row ga (same X row block / W block),
  // comm_col: the pr ranks of grid column gb (same X column block / H block).
  int pr = 1, pc = 1, ga = 0, gb = 0;
  ncclComm_t comm_row = nullptr, comm_col = nullptr;
  ncclComm_t comm = nullptr;
  // in-kernel cross-GPU exchange of the persistent MU kernels (PersistArgs::xpeers): own buffer
  // (IPC-exported), the peers' buffers opened through IPC, the device array of all bases
  void* xbuf = nullptr;
  std::vector<void*> xopened;
  double** xpeers = nullptr;
  bool xready = false;  // buffers mapped on every rank
  int xmode = 1;        // ntt_set_dist_exchange: 1 = in-kernel exchange, 0 = per-pass ncclAllReduce
  FusedCtx fused;
  // profiling (ntt_profile_enable)
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  int cur_step = 0;  // TT step of the launches being recorded (0 outside ntt_decompose)
  struct Rec {
    int cls;
    int step;
    int ev0;
    double bytes;
  };
  std::vector<Rec> recs;
  struct Acc {
    int64_t n = 0;
    double ms = 0.0, bytes = 0.0;
  };
  Acc acc[8][66];
  // CUDA graph of the last ntt_decompose (replayed when the arguments repeat)
  // ntt_set_validation: NTT_VALIDATE_NONNEG checks X / A before the run (one extra read)
  int validate = 0;
  unsigned long long* vbad = nullptr;  // device counter of the check
  // test hook (ntt_debug_bcd_force_correct): BCD iterations whose l.17 test is forced true
  uint64_t bcd_force = 0;
  bool capturing = false;
  cudaStream_t gstream = nullptr;
  cudaEvent_t gev_in = nullptr, gev_out = nullptr;
  cudaGraphExec_t gexec = nullptr;
  cudaGraphExec_t bcd_exec = nullptr;  // ntt_nmf_bcd's one-iteration graph, reused while its key matches
  std::string bcd_key;
  int64_t bcd_per_it = 0;
  std::vector<uint64_t> gkey;
  std::vector<cudaEvent_t> gev_pool;
  size_t gev_used = 0;
  std::vector<Rec> grecs;
  int64_t glaunches = 0;
  // a second cached decompose graph (non-profiled calls): inputs prefetched into alternating
  // slots (ntt_prefetch_input) give two input pointers, each with its own instantiated graph
  cudaGraphExec_t gexec_alt = nullptr;
  std::vector<uint64_t> gkey_alt;
  int64_t glaunches_alt = 0;
  // ntt_prefetch_input: two device input slots filled on a copy stream
  cudaStream_t cstream = nullptr;
  cudaEvent_t cev[2] = {nullptr, nullptr};   // copy into slot s done
  cudaEvent_t uev[2] = {nullptr, nullptr};   // last decompose reading slot s done
  void* slot[2] = {nullptr, nullptr};
  size_t slot_cap[2] = {0, 0};
  const void* slot_src[2] = {nullptr, nullptr};
  int64_t slot_n[2] = {0, 0};
  bool slot_ready[2] = {false, false};
  uint64_t slot_seq[2] = {0, 0};  // fill order: a decompose takes the OLDEST matching slot (FIFO)
  uint64_t fills = 0;
  int next_slot = 0;
};

// drop every cached decompose graph (the path, the profiler or the exchange mode changed)
void drop_graphs(ntt_handle h) {
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  if (h->gexec_alt) cudaGraphExecDestroy(h->gexec_alt);
  h->gexec = h->gexec_alt = nullptr;
  h->gkey.clear();
  h->gkey_alt.clear();
}

namespace {

ntt_status fail(ntt_handle h, ntt_status s, const char* fmt, ...) {
  if (h) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    h->err = buf;
  }
  return s;
}

// NTT_VALIDATE_NONNEG (ntt_set_validation): one counting pass over the rows x cols input
// (row stride ld); NTT_ERR_NONNEG when any entry is negative or NaN.  Synchronises.
ntt_status check_nonneg(ntt_handle h, const float* v, int64_t rows, int64_t cols, int64_t ld, const char* what) {
  if (!(h->validate & 1)) return NTT_OK;
  if (!h->vbad) {
    cudaError_t e = cudaMalloc(&h->vbad, sizeof(unsigned long long));
    if (e != cudaSuccess) return fail(h, NTT_ERR_CUDA, "validation buffer: %s", cudaGetErrorString(e));
  }
  cudaError_t e = launch_count_not_nonneg(v, rows, cols, ld, h->vbad, h->num_sms, h->stream);
  unsigned long long bad = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&bad, h->vbad, sizeof(bad), cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return fail(h, NTT_ERR_CUDA, "validation pass: %s", cudaGetErrorString(e));
  if (bad) return fail(h, NTT_ERR_NONNEG, "%s has %llu negative or NaN entries", what, bad);
  return NTT_OK;
}

#define CU(h, call)                                                                          \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      return fail((h), NTT_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_)); \
  } while (0)

#define LAUNCH(h, call) PLAUNCH(h, 4, 0.0, call)

// Launch with optional event bracketing for the roofline profile (class, algorithmic bytes).
#define PLAUNCH(h, cls, bytes, call)          \
  do {                                        \
    int ev0_ = prof_begin(h);                 \
    CU(h, (call));                            \
    (h)->launches++;                          \
    prof_end(h, ev0_, (cls), (bytes));        \
  } while (0)

#define NC(h, call)                                                                             \
  do {                                                                                          \
    ncclResult_t r_ = (call);                                                                   \
    if (r_ != ncclSuccess)                                                                      \
      return fail((h), NTT_ERR_NCCL, "%s:%d %s: %s", __FILE__, __LINE__, #call, g_nccl.GetErrorString(r_)); \
    (h)->collectives++;                                                                         \
  } while (0)

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

ntt_status ensure_ws(ntt_handle h, size_t bytes) {
  if (bytes <= h->ws_bytes) return NTT_OK;
  CU(h, cudaStreamSynchronize(h->stream));
  if (h->ws) CU(h, cudaFree(h->ws));
  h->ws = nullptr;
  h->ws_bytes = 0;
  CU(h, cudaMalloc(&h->ws, bytes));
  h->ws_bytes = bytes;
  return NTT_OK;
}

ntt_status ensure_stage(ntt_handle h, size_t bytes) {
  if (bytes <= h->stage_bytes) return NTT_OK;
  CU(h, cudaStreamSynchronize(h->stream));
  if (h->stage) CU(h, cudaFree(h->stage));
  h->stage = nullptr;
  h->stage_bytes = 0;
  CU(h, cudaMalloc(&h->stage, bytes));
  h->stage_bytes = bytes;
  return NTT_OK;
}

ntt_status ensure_host_part(ntt_handle h, size_t count) {
  if (count <= h->host_part_count) return NTT_OK;
  if (h->host_part) CU(h, cudaFreeHost(h->host_part));
  h->host_part = nullptr;
  h->host_part_count = 0;
  CU(h, cudaMallocHost(&h->host_part, count * sizeof(double)));
  h->host_part_count = count;
  return NTT_OK;
}

// Events live in two pools: eager launches use ev_pool (recycled by
// ntt_profile_enable), launches captured into the decompose graph use gev_pool
// (owned by the graph, re-recorded at every replay).
int prof_begin(ntt_handle h) {
  if (!h->prof) return -1;
  auto& pool = h->capturing ? h->gev_pool : h->ev_pool;
  size_t& used = h->capturing ? h->gev_used : h->ev_used;
  if (used + 2 > pool.size()) {
    for (int i = 0; i < 256; ++i) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return -1;
      pool.push_back(e);
    }
  }
  int i = (int)used;
  used += 2;
  // inside stream capture an event record must be EXTERNAL to become a real
  // record node that re-records (and can be timed) at every graph replay
  cudaEventRecordWithFlags(pool[i], h->stream, h->capturing ? cudaEventRecordExternal : cudaEventRecordDefault);
  return i;
}

void prof_end(ntt_handle h, int ev0, int cls, double bytes) {
  if (ev0 < 0) return;
  auto& pool = h->capturing ? h->gev_pool : h->ev_pool;
  cudaEventRecordWithFlags(pool[ev0 + 1], h->stream, h->capturing ? cudaEventRecordExternal : cudaEventRecordDefault);
  (h->capturing ? h->grecs : h->recs).push_back({cls, h->cur_step, ev0, bytes});
}

// Fold completed event pairs into the accumulators (stream must be synchronised).
void prof_fold(ntt_handle h, std::vector<ntt_handle_s::Rec>& recs, std::vector<cudaEvent_t>& pool) {
  for (const auto& r : recs) {
    float t = 0.0f;
    cudaError_t e = cudaEventElapsedTime(&t, pool[r.ev0], pool[r.ev0 + 1]);
    if (e != cudaSuccess) {
      static bool warned = false;
      if (!warned && getenv("NTT_DEBUG")) fprintf(stderr, "ntt profile: cudaEventElapsedTime: %s\n", cudaGetErrorString(e));
      warned = true;
      cudaGetLastError();
      continue;
    }
    int step = r.step < 0 ? 0 : (r.step > 65 ? 65 : r.step);
    auto& a = h->acc[r.cls][step];
    a.n += 1;
    a.ms += t;
    a.bytes += r.bytes;
  }
}

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

bool mul_ok(int64_t a, int64_t b, int64_t* out) {
  if (a < 0 || b < 0) return false;
  if (a != 0 && b > INT64_MAX / a) return false;
  *out = a * b;
  return true;
}

// ---------------------------------------------------------- MU iteration driver
// Scratch requirement (bytes) of one MU run on an m x n problem with rank r.
struct MuPlan {
  int64_t m, n;
  int r;
  bool fused;     // 1-pass short-wide kernel (mu_fused.cu)
  bool acc;       // generic 1-pass (hpass accumulates P, Q)
  XhtPlan xp;     // X H^T pass
  XhtPlan qp;     // H H^T pass
  int hgrid;      // H-pass CTAs
  int nwup;       // W-update CTAs
  int fgrid;      // fused kernel CTAs
  int fparts;     // fused kernel partial slots
  bool tc;        // tensor-core 2-pass path (mu_tc.cu) for tall / square X
  TcPlan tp;
  bool persist;   // fused path as one persistent cooperative launch per call
  bool tiny;      // whole MU loop in one CTA from shared memory (mu_tiny.cu)
  bool clu;       // whole MU loop in one thread-block cluster, X in distributed smem (mu_cluster.cu)
  int tail;       // k_fused_m dynamic-tail groups (fused_tail_groups)
  int hks;        // generic path: split-K H pass splits (0 = per-tile k_hpass)
  size_t off_hs;  // its S partials
  size_t off_P, off_Q, off_G, off_S, off_tc, off_pp, off_park, off_red, off_ctr, off_x16, bytes;
};

// dist: a handle from ntt_create_dist* (any number of ranks, 1 included) -- its MU runs
// the distributed branches (all-reduce of the pass partials between passes)
MuPlan plan_mu(int64_t m, int64_t n, int r, int num_sms, bool dist, bool xpersist = false) {
  MuPlan p;
  p.m = m;
  p.n = n;
  p.r = r;
  // shape-level eligibility of the fused TMA kernel; pointer alignment is
  // re-checked at run time (scratch below is sized for either path).
  p.fused = fused_supported(m, n, r, n, nullptr, nullptr);
  p.acc = m * r <= kMaxAccMR;
  p.xp = plan_xht(m, n, num_sms);
  p.qp = plan_xht(r, n, num_sms);
  p.hgrid = hpass_ctas(m, n, r, p.acc, num_sms);
  p.nwup = wupdate_ctas(m, r);
  p.fgrid = fused_grid(m, n, r, num_sms);
  p.fparts = fused_partials(m, n, r, num_sms);
  int64_t nP = std::max<int64_t>({(int64_t)p.xp.ncs, p.acc ? p.hgrid : 0, (int64_t)p.fparts, 1});
  int64_t nQ = std::max<int64_t>({(int64_t)p.qp.ncs, p.acc ? p.hgrid : 0, (int64_t)p.fparts, 1});
  int64_t nG = std::max<int64_t>({(int64_t)p.nwup, (int64_t)wupdate2_ctas(m, r), 1});
  size_t o = 0;
  p.off_P = o;
  o = align_up(o + sizeof(double) * (size_t)(nP * m * r));
  p.off_Q = o;
  o = align_up(o + sizeof(double) * (size_t)(nQ * r * r));
  p.off_G = o;
  o = align_up(o + sizeof(double) * (size_t)(nG * r * r));
  p.off_S = o;  // reduced (m r + r r) vector for the distributed all-reduce
  o = align_up(o + sizeof(double) * (size_t)(m * r + r * r));
  p.hks = p.acc ? 0 : hpass_splits(m, n, num_sms);
  p.off_hs = o;
  if (p.hks) {
    const int rpad = r <= 2 ? 2 : r <= 4 ? 4 : r <= 8 ? 8 : r <= 16 ? 16 : r <= 32 ? 32 : 64;
    o = align_up(o + sizeof(double) * (size_t)p.hks * (size_t)n * (size_t)rpad);
  }
  // shape-level eligibility of the tensor-core path (alignment re-checked at run time)
  p.tc = !p.fused && tc_supported(m, n, r, n, nullptr) && !getenv("NTT_NO_TC");
  p.off_tc = o;
  if (p.tc) {
    p.tp = plan_tc(m, n, r, num_sms);
    o = align_up(o + p.tp.bytes);
  }
  p.persist = (!dist || xpersist) && p.fused && !getenv("NTT_NO_PERSIST");
  // cluster mode beats the one-CTA tiny kernel from ~4 K entries on (measured: 30 x 216 5.7 vs
  // 6.1 us per iteration, 64 x 180 5.5 vs 9.6); below, tiny wins (30 x 36 3.5 vs 5.2)
  const bool clu_ok = !dist && !getenv("NTT_NO_CLUSTER") && cluster_supported(m, n, r);
  p.tiny = !dist && tiny_supported(m, n, r) && !getenv("NTT_NO_TINY") && !(clu_ok && m * n >= 4096);
  p.clu = clu_ok && !p.tiny;
  p.off_pp = o;
  p.tail = p.persist ? fused_tail_groups(m, n, r, p.fgrid) : 0;
  if (p.persist) o = align_up(o + sizeof(double) * (size_t)(p.fgrid + 8 * p.tail) * (size_t)(m * r + r * r));
  p.off_park = o;
  if (p.tail) o = align_up(o + sizeof(double) * (size_t)p.fgrid * 8 * 320);
  p.off_red = o;
  if (p.persist) o = align_up(o + sizeof(double) * (size_t)(m * r + r * r));
  p.off_ctr = o;
  if (p.persist) o = align_up(o + 64);
  p.off_x16 = o;  // fp16 hi / lo copy of X for the persistent k_fused_c (m > 40)
  if (p.persist) o = align_up(o + fused_x16_bytes(m, n));
  p.bytes = o;
  return p;
}

// Sum nP partials of (P, Q) into one vector and all-reduce it over the ranks.
ntt_status dist_reduce(ntt_handle h, const MuPlan& p, double* Ppart, int nP, double* Qpart, int nQ, double* red) {
  LAUNCH(h, launch_sum_partials(Ppart, nP, p.m * p.r, red, h->stream));
  LAUNCH(h, launch_sum_partials(Qpart, nQ, (int64_t)p.r * p.r, red + p.m * p.r, h->stream));
  NC(h, g_nccl.AllReduce(red, red, (size_t)(p.m * p.r + p.r * p.r), ncclFloat64, ncclSum, h->comm, h->stream));
  return NTT_OK;
}

ntt_status run_mu(ntt_handle h, const MuPlan& p, const float* X, int64_t ldx, int32_t iters, float eps, float* W,
                  float* H, char* scratch, double* dev_trace /*nullable: iters*nobj*/) {
  const int64_t m = p.m, n = p.n;
  const int r = p.r;
  double* Ppart = reinterpret_cast<double*>(scratch + p.off_P);
  double* Qpart = reinterpret_cast<double*>(scratch + p.off_Q);
  double* Gpart = reinterpret_cast<double*>(scratch + p.off_G);
  double* red = reinterpret_cast<double*>(scratch + p.off_S);
  const bool dist = h->comm != nullptr;  // every ntt_create_dist* handle, 1 rank included
  cudaStream_t st = h->stream;
  int nobj = objective_ctas(n);
  if (iters <= 0) return NTT_OK;

  if (p.tiny && !dist && !dev_trace) {
    // tiny mode: every iteration in one CTA from shared memory (mu_tiny.cu)
    PLAUNCH(h, 0, (double)iters * 4.0 * (double)(m + 2 * r) * (double)n,
            launch_tiny(X, ldx, m, n, r, iters, eps, W, H, st, h->ptrace));
    return NTT_OK;
  }
  if (p.clu && !dist && !dev_trace) {
    // cluster mode: every iteration in one thread-block cluster, X in distributed shared memory
    PLAUNCH(h, 0, (double)iters * 4.0 * (double)(m + 2 * r) * (double)n,
            launch_cluster_mu(X, ldx, m, n, r, iters, eps, W, H, st, h->ptrace));
    return NTT_OK;
  }
  if (p.fused && p.persist && (!dist || (h->xready && h->xmode == 1)) && !dev_trace &&
      fused_supported(m, n, r, ldx, X, H)) {
    // whole MU loop of this call in one cooperative launch (mu_fused.cu persist_step); on a
    // distributed handle the ranks' partials are exchanged inside the kernel (PersistArgs::xpeers)
    PersistArgs pa;
    if (dist) {
      pa.xpeers = h->xpeers;
      pa.nranks = h->nranks;
      pa.rank = h->rank;
    }
    pa.iters = iters;
    pa.part = reinterpret_cast<double*>(scratch + p.off_pp);
    pa.red = reinterpret_cast<double*>(scratch + p.off_red);
    pa.ctr = reinterpret_cast<unsigned*>(scratch + p.off_ctr);
    pa.Wout = W;
    pa.trace = h->ptrace;  // diagnostics (NTT_PERSIST_TRACE), else null
    pa.x16 = fused_x16_bytes(m, n) ? reinterpret_cast<unsigned char*>(scratch + p.off_x16) : nullptr;
    if (p.tail) {  // the k_fused_m shapes only (fused_tail_groups)
      pa.tail_groups = p.tail;
      pa.park = reinterpret_cast<double*>(scratch + p.off_park);
    }
    CU(h, cudaMemsetAsync(pa.ctr, 0, 64, st));
    PLAUNCH(h, 0, (double)iters * 4.0 * (double)(m + 2 * r) * (double)n + 4.0 * (double)(m + r) * (double)n,
            launch_fused(X, ldx, m, n, r, W, nullptr, 0, eps, H, nullptr, nullptr, 0, p.fgrid, st, &pa));
    return NTT_OK;
  }
  if (p.fused && fused_supported(m, n, r, ldx, X, H)) {
    // 1-pass: prologue P0 = X H0^T, Q0 = H0 H0^T; then per iteration
    //   W update (reduces the partials)  ->  fused pass (H update + next P, Q).
    const int fg = p.fgrid, fp = p.fparts;
    const int nG = wupdate2_ctas(m, r);
    PLAUNCH(h, 1, 4.0 * (double)(m + r) * (double)n,
            launch_fused(X, ldx, m, n, r, W, nullptr, 0, eps, H, Ppart, Qpart, kFusedAcc, fg, st));
    for (int it = 0; it < iters; ++it) {
      if (dist) {
        ntt_status s = dist_reduce(h, p, Ppart, fp, Qpart, fp, red);
        if (s) return s;
        PLAUNCH(h, 2, 8.0 * (double)(2 * m * r + r * r), launch_wupdate2(W, m, r, red, 1, red + m * r, 1, eps, Gpart, st));
      } else {
        PLAUNCH(h, 2, 8.0 * ((double)fp * (m * r + r * r) + m * r),
                launch_wupdate2(W, m, r, Ppart, fp, Qpart, fp, eps, Gpart, st));
      }
      const int mode = kFusedUpdate | ((it + 1 < iters) ? kFusedAcc : 0);
      PLAUNCH(h, 0, 4.0 * (double)(m + 2 * r) * (double)n,
              launch_fused(X, ldx, m, n, r, W, Gpart, nG, eps, H, Ppart, Qpart, mode, fg, st));
      if (dev_trace) LAUNCH(h, launch_objective(X, ldx, m, n, W, H, r, dev_trace + (int64_t)it * nobj, st));
    }
    return NTT_OK;
  }

  if (p.tc && tc_supported(m, n, r, ldx, X)) {
    // tensor-core 2-pass iteration (mu_tc.cu): X > L2 streams evict-first.
    // Distributed (2-D grid, DESIGN.md s.7): the local partials are reduced and
    // all-reduced over the grid row (P = X H^T, Q = H H^T) and the grid column
    // (G = W^T W, S = W^T X); the updates then run redundantly per group.
    const TcPlan& tp = p.tp;
    char* tws = scratch + p.off_tc;
    const int ef = (double)m * (double)ldx * 4.0 > 0.6 * (double)h->l2_bytes ? 1 : 0;
    double* red = reinterpret_cast<double*>(tws + tp.off_red);
    double* gred = reinterpret_cast<double*>(tws + tp.off_Gred);
    double* sred = reinterpret_cast<double*>(tws + tp.off_Sred);
    TcMaps maps;
    LAUNCH(h, tc_prepare(tp, X, ldx, H, tws, &maps, st));
    if (tp.f16) {
      LAUNCH(h, tc16_prepare(tp, X, ldx, H, tws, &maps, st));
      LAUNCH(h, tc16_pack_h(tp, H, tws, st, -1));
    }
    for (int it = 0; it < iters; ++it) {
      LAUNCH(h, tc_sum_Q(tp, tws, st));
      PLAUNCH(h, 6, 4.0 * (double)(m + 2 * tp.R) * (double)n,
              tp.f16 ? tc16_pass_w(tp, maps, tws, ef, st) : tc_pass_w(tp, maps, tws, ef, st));
      if (dist) {
        LAUNCH(h, tc_reduce_PQ(tp, tws, st));
        NC(h, g_nccl.AllReduce(red, red, (size_t)(m * r + r * r), ncclFloat64, ncclSum, h->comm_row, st));
        PLAUNCH(h, 2, 8.0 * (double)(2 * m * r + r * r) + 4.0 * 2 * tp.R * m,
                tc_wupdate_ex(tp, W, eps, tws, red, 1, red + m * r, st, it));
        NC(h, g_nccl.AllReduce(gred, gred, (size_t)(r * r), ncclFloat64, ncclSum, h->comm_col, st));
      } else {
        PLAUNCH(h, 2, 8.0 * (double)tp.splitW * m * r + 8.0 * m * r + 4.0 * 2 * tp.R * m,
                tc_wupdate(tp, W, eps, tws, st, it));
      }
      if (tp.f16) LAUNCH(h, tc16_pack_w(tp, W, tws, st, it));
      PLAUNCH(h, 7, 4.0 * (double)(n + 2 * tp.R) * (double)m,
              tp.f16 ? tc16_pass_h(tp, maps, tws, ef, st) : tc_pass_h(tp, maps, tws, ef, st));
      if (dist) {
        LAUNCH(h, tc_reduce_S(tp, tws, st));
        NC(h, g_nccl.AllReduce(sred, sred, (size_t)(n * r), ncclFloat64, ncclSum, h->comm_col, st));
        PLAUNCH(h, 4, 8.0 * (double)n * r + 4.0 * (3 * tp.R + r) * (double)n, tc_hupdate_ex(tp, H, eps, tws, sred, 1, st, it));
      } else {
        PLAUNCH(h, 4, 8.0 * (double)tp.splitH * n * r + 4.0 * (3 * tp.R + r) * (double)n,
                tc_hupdate(tp, H, eps, tws, st, it));
      }
      if (tp.f16) LAUNCH(h, tc16_pack_h(tp, H, tws, st, it));
      if (dev_trace) LAUNCH(h, launch_objective(X, ldx, m, n, W, H, r, dev_trace + (int64_t)it * nobj, st));
    }
    return NTT_OK;
  }
  if (h->pr > 1)
    return fail(h, NTT_ERR_UNSUPPORTED,
                "2-D grid (pr = %d) NMF needs the tensor-core path: r <= 32, local m, n >= 256, 16-byte aligned X "
                "(got m=%lld n=%lld r=%d)", h->pr, (long long)m, (long long)n, r);

  // prologue (1-pass) or first W pass: P = X H^T, Q = H H^T
  int nP = 0, nQ = 0;
  for (int it = 0; it < iters; ++it) {
    if (!p.acc || it == 0) {
      PLAUNCH(h, 1, 4.0 * (double)(m + r) * (double)n, launch_xht_partial(X, ldx, m, n, H, n, r, p.xp, Ppart, st));
      PLAUNCH(h, 4, 4.0 * (double)r * (double)n, launch_xht_partial(H, n, r, n, H, n, r, p.qp, Qpart, st));
      nP = p.xp.ncs;
      nQ = p.qp.ncs;
    }
    if (dist) {
      ntt_status s = dist_reduce(h, p, Ppart, nP, Qpart, nQ, red);
      if (s) return s;
      PLAUNCH(h, 2, 8.0 * (double)(m * r + r * r) + 8.0 * (double)(m * r), launch_wupdate(W, m, r, red, 1, red + m * r, 1, eps, Gpart, st));
    } else {
      PLAUNCH(h, 2, 8.0 * ((double)nP * m * r + (double)nQ * r * r) + 8.0 * (double)(m * r),
              launch_wupdate(W, m, r, Ppart, nP, Qpart, nQ, eps, Gpart, st));
    }
    const bool acc_now = p.acc && (it + 1 < iters);
    if (p.hks && !acc_now)  // few column tiles, many rows: split-K over the rows
      PLAUNCH(h, 5, 4.0 * (double)(m + 2 * r) * (double)n,
              launch_hpass_sk(X, ldx, m, n, W, r, Gpart, p.nwup, eps, H, p.hks,
                              reinterpret_cast<double*>(scratch + p.off_hs), red, st));
    else
      PLAUNCH(h, 5, 4.0 * (double)(m + 2 * r) * (double)n,
              launch_hpass(X, ldx, m, n, W, r, Gpart, p.nwup, eps, H, p.hgrid, acc_now ? Ppart : nullptr,
                           acc_now ? Qpart : nullptr, st));
    if (acc_now) {
      nP = p.hgrid;
      nQ = p.hgrid;
    }
    if (dev_trace) LAUNCH(h, launch_objective(X, ldx, m, n, W, H, r, dev_trace + (int64_t)it * nobj, st));
  }
  return NTT_OK;
}

ntt_status check_mu_args(ntt_handle h, const float* X, int64_t m, int64_t n, int64_t ldx, int32_t r, int32_t iters,
                         float eps, const float* W, const float* H) {
  if (!h) return NTT_ERR_INVALID_ARG;
  if (!X || !W || !H) return fail(h, NTT_ERR_INVALID_ARG, "null X, W or H");
  if (m < 1 || n < 1) return fail(h, NTT_ERR_INVALID_ARG, "m, n must be >= 1 (got %lld, %lld)", (long long)m, (long long)n);
  if (ldx < n) return fail(h, NTT_ERR_INVALID_ARG, "ldx (%lld) < n (%lld)", (long long)ldx, (long long)n);
  if (iters < 0) return fail(h, NTT_ERR_INVALID_ARG, "iters < 0");
  if (!(eps >= 0.0f)) return fail(h, NTT_ERR_INVALID_ARG, "eps must be >= 0");
  if (r < 1 || r > kMaxRank || r > m || r > n)
    return fail(h, NTT_ERR_RANK, "rank %d outside [1, min(m, n, %d)]", r, kMaxRank);
  int64_t t;
  if (!mul_ok(m, ldx, &t)) return fail(h, NTT_ERR_DIMENSION, "m * ldx overflows");
  return NTT_OK;
}

struct TTShape {
  int d;
  int64_t dims[64];
  int64_t r[65];   // r_0..r_d
  int64_t N;       // prod dims
  int64_t cores;   // packed size
  int64_t off[65]; // core offsets o_1..o_d (1-based)
};

ntt_status check_tt(ntt_handle h, int32_t d, const int64_t* dims, const int32_t* ranks, TTShape* s, bool check_ranks) {
  if (d < 2 || d > 64 || !dims || (d > 1 && !ranks)) return fail(h, NTT_ERR_DIMENSION, "need 2 <= d <= 64 and dims/ranks");
  s->d = d;
  s->N = 1;
  for (int l = 0; l < d; ++l) {
    if (dims[l] < 1) return fail(h, NTT_ERR_DIMENSION, "dims[%d] = %lld < 1", l, (long long)dims[l]);
    s->dims[l] = dims[l];
    if (!mul_ok(s->N, dims[l], &s->N)) return fail(h, NTT_ERR_DIMENSION, "prod(dims) overflows");
  }
  s->r[0] = 1;
  s->r[d] = 1;
  for (int l = 1; l < d; ++l) s->r[l] = ranks[l - 1];
  int64_t rest = s->N;
  for (int l = 1; l < d; ++l) {
    rest /= dims[l - 1];  // prod_{i>l} n_i
    int64_t rows = s->r[l - 1] * dims[l - 1];
    if (s->r[l] < 1 || s->r[l] > kMaxRank || (check_ranks && (s->r[l] > rows || s->r[l] > rest)))
      return fail(h, NTT_ERR_RANK, "rank r_%d = %lld outside [1, min(%lld, %lld, %d)]", l, (long long)s->r[l],
                  (long long)rows, (long long)rest, kMaxRank);
  }
  s->cores = 0;
  for (int l = 1; l <= d; ++l) {
    s->off[l] = s->cores;
    s->cores += s->r[l - 1] * dims[l - 1] * s->r[l];
  }
  return NTT_OK;
}

}  // namespace

// -------------------------------------------------------- reconstruct / error
namespace {
struct ContractPlan {
  int k;                 // split bond
  int64_t NL, NR, lmax, rmax;
  int grid;
  size_t off_L, off_R, off_part, off_cores, bytes;
};

ContractPlan plan_contract(const TTShape& s, int num_sms) {
  ContractPlan c;
  const int d = s.d;
  // split bond k minimising |L| + |R| = (N_L + N_R) r_k
  int best = 1;
  double bestc = 1e300;
  for (int k = 1; k < d; ++k) {
    double NL = 1, NR = 1;
    for (int l = 0; l < k; ++l) NL *= (double)s.dims[l];
    for (int l = k; l < d; ++l) NR *= (double)s.dims[l];
    double cst = (NL + NR) * (double)s.r[k];
    if (cst < bestc) {
      bestc = cst;
      best = k;
    }
  }
  c.k = best;
  c.NL = 1;
  c.NR = 1;
  for (int l = 0; l < c.k; ++l) c.NL *= s.dims[l];
  for (int l = c.k; l < d; ++l) c.NR *= s.dims[l];
  c.lmax = 1;
  c.rmax = 1;
  int64_t acc = 1;
  for (int l = 1; l <= c.k; ++l) {
    acc *= s.dims[l - 1];
    c.lmax = std::max(c.lmax, acc * s.r[l]);
  }
  acc = 1;
  for (int l = d; l > c.k; --l) {
    acc *= s.dims[l - 1];
    c.rmax = std::max(c.rmax, s.r[l - 1] * acc);
  }
  c.grid = stream_ctas(c.NL, c.NR, num_sms);
  size_t o = 0;
  c.off_L = o;
  o = align_up(o + sizeof(float) * (size_t)(2 * c.lmax));
  c.off_R = o;
  o = align_up(o + sizeof(float) * (size_t)(2 * c.rmax));
  c.off_part = o;
  o = align_up(o + sizeof(double) * 2 * (size_t)(c.grid + 1));
  c.off_cores = o;
  o = align_up(o + sizeof(float) * (size_t)s.cores);
  c.bytes = o;
  return c;
}

// Contract the train (device cores `dc`) and stream it against ref / into out.
// Leaves the per-CTA (num, den) error partials at scratch + off_part when ref.
ntt_status contract_run(ntt_handle h, const TTShape& s, const ContractPlan& c, const float* dc, float* dout,
                        float noise_amp, uint64_t noise_key, const float* dref, char* scratch) {
  cudaStream_t cs = h->stream;
  const int d = s.d, k = c.k;
  float* Lb[2] = {reinterpret_cast<float*>(scratch + c.off_L), reinterpret_cast<float*>(scratch + c.off_L) + c.lmax};
  float* Rb[2] = {reinterpret_cast<float*>(scratch + c.off_R), reinterpret_cast<float*>(scratch + c.off_R) + c.rmax};
  double* part = reinterpret_cast<double*>(scratch + c.off_part);
  // left chain: L_1 = G_1 (n_1 x r_1); L_l = L_{l-1} G_l
  const float* L = dc + s.off[1];
  int64_t Ncur = s.dims[0];
  for (int l = 2; l <= k; ++l) {
    float* o = Lb[l & 1];
    PLAUNCH(h, 4, 0.0, launch_contract_left(L, Ncur, (int)s.r[l - 1], dc + s.off[l], s.dims[l - 1], (int)s.r[l], o, cs));
    L = o;
    Ncur *= s.dims[l - 1];
  }
  // right chain: R_d = G_d (r_{d-1} x n_d); R_l = G_l R_{l+1}
  const float* R = dc + s.off[d];
  int64_t NRcur = s.dims[d - 1];
  for (int l = d - 1; l > k; --l) {
    float* o = Rb[l & 1];
    PLAUNCH(h, 4, 0.0, launch_contract_right(dc + s.off[l], (int)s.r[l - 1], s.dims[l - 1], (int)s.r[l], R, NRcur, o, cs));
    R = o;
    NRcur *= s.dims[l - 1];
  }
  // algorithmic bytes: ref read + out write (+ L, R once)
  double bytes = 4.0 * (double)s.N * ((dref ? 1 : 0) + (dout ? 1 : 0)) + 4.0 * (double)(c.NL + c.NR) * (double)s.r[k];
  PLAUNCH(h, 3, bytes, launch_tt_stream(L, R, c.NL, c.NR, (int)s.r[k], dout, noise_amp, noise_key, dref,
                                         dref ? part : nullptr, c.grid, cs));
  return NTT_OK;
}

// Sum the error partials (fixed order), optionally all-reduce over ranks, and
// copy (num, den) to the pinned host landing zone (ensure_host_part(h, 2) first).
ntt_status finish_error_device(ntt_handle h, const ContractPlan& c, char* scratch, bool allreduce) {
  cudaStream_t cs = h->stream;
  double* part = reinterpret_cast<double*>(scratch + c.off_part);
  double* tot = part + 2 * c.grid;
  PLAUNCH(h, 4, 0.0, launch_sum_pairs(part, c.grid, tot, cs));
  if (allreduce) NC(h, g_nccl.AllReduce(tot, tot, 2, ncclFloat64, ncclSum, h->comm, cs));
  CU(h, cudaMemcpyAsync(h->host_part, tot, 2 * sizeof(double), cudaMemcpyDeviceToHost, cs));
  return NTT_OK;
}

// Eq. 3 from the landed (num, den); the stream must have been synchronised.
ntt_status finish_error_host(ntt_handle h, double* rel_err) {
  if (h->host_part[1] == 0.0) return fail(h, NTT_ERR_DEGENERATE, "||ref||_F = 0");
  *rel_err = sqrt(h->host_part[0]) / sqrt(h->host_part[1]);
  return NTT_OK;
}

ntt_status finish_error(ntt_handle h, const ContractPlan& c, char* scratch, bool allreduce, double* rel_err) {
  ntt_status st = ensure_host_part(h, 2);
  if (st) return st;
  if ((st = finish_error_device(h, c, scratch, allreduce))) return st;
  CU(h, cudaStreamSynchronize(h->stream));
  return finish_error_host(h, rel_err);
}

ntt_status contract_stream(ntt_handle h, const TTShape& s, const float* cores, float* out, float noise_amp,
                           uint64_t noise_key, const float* ref, double* rel_err) {
  cudaStream_t cs = h->stream;
  ContractPlan c = plan_contract(s, h->num_sms);
  const bool cores_dev = is_device_ptr(cores);
  const bool out_dev = !out || is_device_ptr(out);
  const bool ref_dev = !ref || is_device_ptr(ref);
  ntt_status st = ensure_ws(h, c.bytes);
  if (st) return st;
  char* ws = reinterpret_cast<char*>(h->ws);
  const float* dc = cores;
  if (!cores_dev) {
    float* t = reinterpret_cast<float*>(ws + c.off_cores);
    CU(h, cudaMemcpyAsync(t, cores, sizeof(float) * (size_t)s.cores, cudaMemcpyHostToDevice, cs));
    dc = t;
  }
  size_t sbytes = (out_dev ? 0 : align_up(sizeof(float) * (size_t)s.N)) + (ref_dev ? 0 : align_up(sizeof(float) * (size_t)s.N));
  if (sbytes && (st = ensure_stage(h, sbytes))) return st;
  float* dout = out;
  const float* dref = ref;
  char* sg = reinterpret_cast<char*>(h->stage);
  if (!out_dev) {
    dout = reinterpret_cast<float*>(sg);
    sg += align_up(sizeof(float) * (size_t)s.N);
  }
  if (!ref_dev) {
    float* t = reinterpret_cast<float*>(sg);
    CU(h, cudaMemcpyAsync(t, ref, sizeof(float) * (size_t)s.N, cudaMemcpyHostToDevice, cs));
    dref = t;
  }
  if ((st = contract_run(h, s, c, dc, dout, noise_amp, noise_key, dref, ws))) return st;
  if (!out_dev) CU(h, cudaMemcpyAsync(out, dout, sizeof(float) * (size_t)s.N, cudaMemcpyDeviceToHost, cs));
  if (rel_err) {
    if ((st = finish_error(h, c, ws, false, rel_err))) return st;
  }
  if (!out_dev) CU(h, cudaStreamSynchronize(cs));
  return NTT_OK;
}
}  // namespace

// ============================================================================ ABI
extern "C" {

int ntt_abi_version(void) { return NTT_ABI_VERSION; }

const char* ntt_status_string(ntt_status s) {
  switch (s) {
    case NTT_OK: return "ok";
    case NTT_ERR_INVALID_ARG: return "invalid argument";
    case NTT_ERR_DIMENSION: return "dimension error";
    case NTT_ERR_RANK: return "rank error";
    case NTT_ERR_DEGENERATE: return "degenerate input";
    case NTT_ERR_NONNEG: return "negative input";
    case NTT_ERR_WORKSPACE: return "workspace too small";
    case NTT_ERR_CUDA: return "CUDA error";
    case NTT_ERR_NCCL: return "NCCL error";
    case NTT_ERR_UNSUPPORTED: return "unsupported";
  }
  return "unknown status";
}

const char* ntt_last_error(ntt_handle h) { return h ? h->err.c_str() : "null handle"; }
int64_t ntt_launch_count(ntt_handle h) { return h ? h->launches : -1; }

static ntt_status create_common(ntt_handle* out, int device, void* stream) {
  if (!out) return NTT_ERR_INVALID_ARG;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= device || device < 0) {
    cudaGetLastError();
    return NTT_ERR_CUDA;
  }
  if (cudaSetDevice(device) != cudaSuccess) return NTT_ERR_CUDA;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return NTT_ERR_CUDA;
  if (prop.major != 10) return NTT_ERR_CUDA;  // sm_100a image only
  ntt_handle h = new ntt_handle_s();
  h->device = device;
  h->stream = reinterpret_cast<cudaStream_t>(stream);
  h->num_sms = prop.multiProcessorCount;
  h->l2_bytes = prop.l2CacheSize;
  if (getenv("NTT_PERSIST_TRACE")) cudaMallocManaged(&h->ptrace, sizeof(unsigned long long) * (4 * 4096 + 2048 + 4096));
  *out = h;
  return NTT_OK;
}

ntt_status ntt_create(ntt_handle* out, int device, void* cuda_stream) {
  return create_common(out, device, cuda_stream);
}

ntt_status ntt_set_stream(ntt_handle h, void* cuda_stream) {
  if (!h) return NTT_ERR_INVALID_ARG;
  h->stream = reinterpret_cast<cudaStream_t>(cuda_stream);
  return NTT_OK;
}

ntt_status ntt_destroy(ntt_handle h) {
  if (!h) return NTT_ERR_INVALID_ARG;
  cudaSetDevice(h->device);
  cudaStreamSynchronize(h->stream);
  fused_destroy(h->fused);
  if (h->ws) cudaFree(h->ws);
  if (h->ptrace) cudaFree(h->ptrace);
  if (h->vbad) cudaFree(h->vbad);
  if (h->stage) cudaFree(h->stage);
  if (h->sweep) cudaFree(h->sweep);
  if (h->host_part) cudaFreeHost(h->host_part);
  for (void* pp : h->xopened) cudaIpcCloseMemHandle(pp);
  if (h->xpeers) cudaFree(h->xpeers);
  if (h->xbuf) cudaFree(h->xbuf);
  if (h->comm_row && g_nccl.loaded) g_nccl.CommDestroy(h->comm_row);
  if (h->comm_col && g_nccl.loaded) g_nccl.CommDestroy(h->comm_col);
  if (h->comm && g_nccl.loaded) g_nccl.CommDestroy(h->comm);
  for (auto e : h->ev_pool) cudaEventDestroy(e);
  for (auto e : h->gev_pool) cudaEventDestroy(e);
  drop_graphs(h);
  if (h->bcd_exec) cudaGraphExecDestroy(h->bcd_exec);
  for (int q = 0; q < 2; ++q) {
    if (h->slot[q]) cudaFree(h->slot[q]);
    if (h->cev[q]) cudaEventDestroy(h->cev[q]);
    if (h->uev[q]) cudaEventDestroy(h->uev[q]);
  }
  if (h->cstream) cudaStreamDestroy(h->cstream);
  if (h->gev_in) cudaEventDestroy(h->gev_in);
  if (h->gev_out) cudaEventDestroy(h->gev_out);
  if (h->gstream) cudaStreamDestroy(h->gstream);
  delete h;
  return NTT_OK;
}

ntt_status ntt_fill_uniform(ntt_handle h, float* p, int64_t count, uint64_t seed, uint64_t stream,
                            int64_t index_offset) {
  if (!h) return NTT_ERR_INVALID_ARG;
  if (!p || count < 0 || index_offset < 0) return fail(h, NTT_ERR_INVALID_ARG, "bad fill_uniform arguments");
  CU(h, cudaSetDevice(h->device));
  if (count == 0) return NTT_OK;
  if (is_device_ptr(p)) {
    LAUNCH(h, launch_fill_uniform(p, count, seed, stream, index_offset, h->stream));
    return NTT_OK;
  }
  ntt_status s = ensure_stage(h, sizeof(float) * (size_t)count);
  if (s) return s;
  float* d = reinterpret_cast<float*>(h->stage);
  LAUNCH(h, launch_fill_uniform(d, count, seed, stream, index_offset, h->stream));
  CU(h, cudaMemcpyAsync(p, d, sizeof(float) * (size_t)count, cudaMemcpyDeviceToHost, h->stream));
  CU(h, cudaStreamSynchronize(h->stream));
  return NTT_OK;
}

ntt_status ntt_nmf_mu(ntt_handle h, const float* X, int64_t m, int64_t n, int64_t ldx, int32_t r, int32_t iters,
                      float eps, float* W, float* H, double* objective_trace) {
  ntt_status s = check_mu_args(h, X, m, n, ldx, r, iters, eps, W, H);
  if (s) return s;
  CU(h, cudaSetDevice(h->device));
  MuPlan p = plan_mu(m, n, r, h->num_sms, h->comm != nullptr, h->xready && h->xmode == 1);
  const bool xd = is_device_ptr(X), wd = is_device_ptr(W), hd = is_device_ptr(H);
  // staging layout for host buffers: [X | W | H]
  size_t sx = xd ? 0 : align_up(sizeof(float) * (size_t)(m * ldx));
  size_t sw = wd ? 0 : align_up(sizeof(float) * (size_t)(m * r));
  size_t sh = hd ? 0 : align_up(sizeof(float) * (size_t)(r * n));
  int nobj = objective_ctas(n);
  size_t strace = objective_trace ? align_up(sizeof(double) * (size_t)iters * nobj) : 0;
  if ((s = ensure_ws(h, p.bytes + strace))) return s;
  if (sx + sw + sh) {
    if ((s = ensure_stage(h, sx + sw + sh))) return s;
  }
  char* stg = reinterpret_cast<char*>(h->stage);
  const float* dX = X;
  float* dW = W;
  float* dH = H;
  if (!xd) {
    dX = reinterpret_cast<float*>(stg);
    CU(h, cudaMemcpyAsync((void*)dX, X, sizeof(float) * (size_t)(m * ldx), cudaMemcpyHostToDevice, h->stream));
  }
  if (!wd) {
    dW = reinterpret_cast<float*>(stg + sx);
    CU(h, cudaMemcpyAsync(dW, W, sizeof(float) * (size_t)(m * r), cudaMemcpyHostToDevice, h->stream));
  }
  if (!hd) {
    dH = reinterpret_cast<float*>(stg + sx + sw);
    CU(h, cudaMemcpyAsync(dH, H, sizeof(float) * (size_t)(r * n), cudaMemcpyHostToDevice, h->stream));
  }
  if ((s = check_nonneg(h, dX, m, n, ldx, "X"))) return s;
  char* scratch = reinterpret_cast<char*>(h->ws);
  double* dtrace = objective_trace ? reinterpret_cast<double*>(scratch + p.bytes) : nullptr;
  if (h->comm && h->nranks > 1 && h->xready && h->xmode == 1) {
    // every rank in the persistent kernel or none (the in-kernel exchange; see ntt_decompose):
    // the ranks' local shapes / alignments may differ
    int flag = (p.persist && !dtrace && fused_supported(m, n, r, ldx, dX, dH)) ? 1 : 0;
    int* dfl = nullptr;
    CU(h, cudaMallocAsync(reinterpret_cast<void**>(&dfl), sizeof(int), h->stream));
    CU(h, cudaMemcpyAsync(dfl, &flag, sizeof(int), cudaMemcpyHostToDevice, h->stream));
    NC(h, g_nccl.AllReduce(dfl, dfl, 1, ncclInt32, ncclMin, h->comm, h->stream));
    CU(h, cudaMemcpyAsync(&flag, dfl, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    CU(h, cudaFreeAsync(dfl, h->stream));
    CU(h, cudaStreamSynchronize(h->stream));
    p.persist = flag != 0;
  }
  if ((s = run_mu(h, p, dX, ldx, iters, eps, dW, dH, scratch, dtrace))) return s;
  if (!wd) CU(h, cudaMemcpyAsync(W, dW, sizeof(float) * (size_t)(m * r), cudaMemcpyDeviceToHost, h->stream));
  if (!hd) CU(h, cudaMemcpyAsync(H, dH, sizeof(float) * (size_t)(r * n), cudaMemcpyDeviceToHost, h->stream));
  if (objective_trace) {
    std::vector<double> tmp((size_t)iters * nobj);
    CU(h, cudaMemcpyAsync(tmp.data(), dtrace, sizeof(double) * tmp.size(), cudaMemcpyDeviceToHost, h->stream));
    CU(h, cudaStreamSynchronize(h->stream));
    for (int it = 0; it < iters; ++it) {
      double acc = 0.0;
      for (int b = 0; b < nobj; ++b) acc += tmp[(size_t)it * nobj + b];
      objective_trace[it] = 0.5 * acc;
    }
  }
  if (!wd || !hd) CU(h, cudaStreamSynchronize(h->stream));
  return NTT_OK;
}


// ------------------------------------------------------------------ decompose
namespace {
struct DecompPlan {
  TTShape s;
  int64_t nloc_last;         // local extent of the last mode (distributed)
  int64_t last_off;          // global offset of this rank's block
  int64_t m[65], ncol[65];   // per step l: rows m_l and LOCAL columns n_l
  int64_t hbuf[2];           // ping-pong H buffer sizes (floats)
  int64_t wmax;              // max m_l r_l
  size_t mu_bytes;
  size_t off_h0, off_h1, off_w, off_mu, off_cores, off_err, off_gath, bytes;
  MuPlan mu[65];
  TTShape sl;        // local shape (last mode = local block) for the error pass
  ContractPlan cp;
};

void plan_decompose(const TTShape& s, int num_sms, int nranks, int rank, bool dist, DecompPlan* P, bool xpersist = false) {
  P->s = s;
  int64_t off = 0;
  P->nloc_last = ntt_dist_block(s.dims[s.d - 1], nranks, rank, &off);
  P->last_off = off;
  int64_t Nloc = s.N / s.dims[s.d - 1] * P->nloc_last;
  int64_t rest = Nloc;
  P->hbuf[0] = P->hbuf[1] = 1;
  P->wmax = 1;
  P->mu_bytes = 0;
  for (int l = 1; l < s.d; ++l) {
    P->m[l] = s.r[l - 1] * s.dims[l - 1];
    rest /= s.dims[l - 1];
    P->ncol[l] = rest;
    int64_t hsz = s.r[l] * rest;
    P->hbuf[(l - 1) & 1] = std::max(P->hbuf[(l - 1) & 1], hsz);
    P->wmax = std::max(P->wmax, P->m[l] * s.r[l]);
    P->mu[l] = plan_mu(P->m[l], P->ncol[l], (int)s.r[l], num_sms, dist, xpersist);
    P->mu_bytes = std::max(P->mu_bytes, P->mu[l].bytes);
  }
  size_t o = 0;
  P->off_h0 = o;
  o = align_up(o + sizeof(float) * (size_t)P->hbuf[0]);
  P->off_h1 = o;
  o = align_up(o + sizeof(float) * (size_t)P->hbuf[1]);
  P->off_w = o;
  o = align_up(o + sizeof(float) * (size_t)P->wmax);
  P->off_cores = o;
  o = align_up(o + sizeof(float) * (size_t)s.cores);
  P->off_mu = o;
  o = align_up(o + P->mu_bytes);
  P->sl = s;
  P->sl.dims[s.d - 1] = P->nloc_last;
  P->sl.N = s.N / s.dims[s.d - 1] * P->nloc_last;
  P->sl.cores = s.cores - s.r[s.d - 1] * (s.dims[s.d - 1] - P->nloc_last);
  P->cp = plan_contract(P->sl, num_sms);
  P->off_err = o;
  o = align_up(o + P->cp.bytes);
  P->off_gath = o;  // last-core all-gather staging (distributed)
  o = align_up(o + sizeof(float) * (size_t)(s.r[s.d - 1] * s.dims[s.d - 1]));
  P->bytes = o;
}

// All device work of one ntt_decompose, enqueued on h->stream (graph-capturable:
// no allocation, no synchronisation, no host reads of device data).
ntt_status decompose_device(ntt_handle h, const DecompPlan& P, const TTShape& s, const float* dA, float* dcores,
                            char* ws, int32_t iters, uint64_t seed, float eps, bool want_err) {
  ntt_status st;
  cudaStream_t cs = h->stream;
  const int d = s.d;
  float* hb[2] = {reinterpret_cast<float*>(ws + P.off_h0), reinterpret_cast<float*>(ws + P.off_h1)};
  float* Wd = reinterpret_cast<float*>(ws + P.off_w);
  char* mus = ws + P.off_mu;
  const float* X = dA;
  float* Hl = nullptr;
  for (int l = 1; l < d; ++l) {
    const int64_t m = P.m[l], n = P.ncol[l];
    const int r = (int)s.r[l];
    Hl = hb[(l - 1) & 1];
    h->cur_step = l;
    LAUNCH(h, launch_fill_uniform(Wd, m * r, seed, stream_w(l), 0, cs));
    if (!h->comm) {
      LAUNCH(h, launch_fill_uniform(Hl, (int64_t)r * n, seed, stream_h(l), 0, cs));
    } else {
      // global column index of local column c: (c / b) * n_d + off + c % b  (DESIGN.md s.7)
      const int64_t nglob = n / P.nloc_last * s.dims[d - 1];
      LAUNCH(h, launch_fill_uniform_cols(Hl, r, n, P.nloc_last, s.dims[d - 1], P.last_off, nglob, seed,
                                         stream_h(l), cs));
    }
    if ((st = run_mu(h, P.mu[l], X, n, iters, eps, Wd, Hl, mus, nullptr))) return st;
    CU(h, cudaMemcpyAsync(dcores + s.off[l], Wd, sizeof(float) * (size_t)(m * r), cudaMemcpyDeviceToDevice, cs));
    X = Hl;
  }
  h->cur_step = d;  // last-core gather and the error pass
  // last core G_d[k][i][0] = T_{d-1}[k][i]  (Alg. 2 l.11)
  const int64_t rl = s.r[d - 1], nd = s.dims[d - 1];
  if (!h->comm) {
    CU(h, cudaMemcpyAsync(dcores + s.off[d], Hl, sizeof(float) * (size_t)(rl * nd), cudaMemcpyDeviceToDevice, cs));
  } else {
    // all_gather of the ragged column blocks: one broadcast per rank into a
    // rank-major staging area, then a permute into the core layout.
    float* gath = reinterpret_cast<float*>(ws + P.off_gath);
    NC(h, g_nccl.GroupStart());
    for (int g = 0; g < h->nranks; ++g) {
      int64_t og = 0;
      int64_t bg = ntt_dist_block(nd, h->nranks, g, &og);
      const float* src = (g == h->rank) ? Hl : gath + rl * og;
      NC(h, g_nccl.Broadcast(src, gath + rl * og, (size_t)(rl * bg), ncclFloat32, g, h->comm, cs));
    }
    NC(h, g_nccl.GroupEnd());
    LAUNCH(h, launch_gather_last_core(gath, rl, nd, h->nranks, dcores + s.off[d], cs));
  }
  if (want_err) {
    // Eq. 3 of the result against (this rank's block of) A; the local train is
    // cores 1..d-1 plus this rank's column block of the last core (= H_{d-1}).
    char* es = ws + P.off_err;
    float* lc = reinterpret_cast<float*>(es + P.cp.off_cores);
    CU(h, cudaMemcpyAsync(lc, dcores, sizeof(float) * (size_t)s.off[d], cudaMemcpyDeviceToDevice, cs));
    CU(h, cudaMemcpyAsync(lc + s.off[d], Hl, sizeof(float) * (size_t)(rl * P.nloc_last), cudaMemcpyDeviceToDevice, cs));
    if ((st = contract_run(h, P.sl, P.cp, lc, nullptr, 0.0f, 0, dA, es))) return st;
    if ((st = finish_error_device(h, P.cp, es, h->comm != nullptr))) return st;
  }
  h->cur_step = 0;
  return NTT_OK;
}
}  // namespace

size_t ntt_decompose_workspace_bytes(int32_t d, const int64_t* dims, const int32_t* ranks) {
  TTShape s;
  if (check_tt(nullptr, d, dims, ranks, &s, true) != NTT_OK) return 0;
  DecompPlan* P = new DecompPlan();
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaGetLastError();
  plan_decompose(s, sms, 1, 0, false, P);
  size_t b = P->bytes;
  delete P;
  return b;
}

ntt_status ntt_decompose(ntt_handle h, const float* A, int32_t d, const int64_t* dims, const int32_t* ranks,
                         int32_t iters, uint64_t seed, float eps, float* cores, double* rel_err,
                         void* workspace, size_t workspace_bytes) {
  if (!h) return NTT_ERR_INVALID_ARG;
  if (!A || !cores) return fail(h, NTT_ERR_INVALID_ARG, "null A or cores");
  if (iters < 0) return fail(h, NTT_ERR_INVALID_ARG, "iters < 0");
  if (!(eps >= 0.0f)) return fail(h, NTT_ERR_INVALID_ARG, "eps must be >= 0");
  if (h->pr > 1)
    return fail(h, NTT_ERR_UNSUPPORTED, "ntt_decompose partitions the last tensor mode: use a 1 x p grid (pr = %d)",
                h->pr);
  TTShape s;
  ntt_status st = check_tt(h, d, dims, ranks, &s, true);
  if (st) return st;
  if (h->nranks > 1 && s.dims[d - 1] < h->nranks)
    return fail(h, NTT_ERR_DIMENSION, "last mode (%lld) smaller than the number of ranks (%d)",
                (long long)s.dims[d - 1], h->nranks);
  CU(h, cudaSetDevice(h->device));
  DecompPlan* Pp = new DecompPlan();
  std::unique_ptr<DecompPlan> guard(Pp);
  DecompPlan& P = *Pp;
  plan_decompose(s, h->num_sms, h->nranks, h->rank, h->comm != nullptr, &P, h->xready && h->xmode == 1);
  if (h->comm && h->nranks > 1 && h->xready && h->xmode == 1) {
    // the in-kernel exchange needs every rank in the persistent kernel of a step: ragged last-mode
    // blocks can make a step persistent-eligible on some ranks only (n % 4), so the ranks agree
    // per step (min over the ranks' flags); the per-pass NCCL paths issue one identical
    // all-reduce per pass on any kernel path
    int flags[64] = {0};
    for (int l = 1; l < d; ++l) flags[l] = P.mu[l].persist ? 1 : 0;
    int* dfl = nullptr;
    CU(h, cudaMallocAsync(reinterpret_cast<void**>(&dfl), sizeof flags, h->stream));
    CU(h, cudaMemcpyAsync(dfl, flags, sizeof flags, cudaMemcpyHostToDevice, h->stream));
    NC(h, g_nccl.AllReduce(dfl, dfl, 64, ncclInt32, ncclMin, h->comm, h->stream));
    CU(h, cudaMemcpyAsync(flags, dfl, sizeof flags, cudaMemcpyDeviceToHost, h->stream));
    CU(h, cudaFreeAsync(dfl, h->stream));
    CU(h, cudaStreamSynchronize(h->stream));
    for (int l = 1; l < d; ++l) P.mu[l].persist = flags[l] != 0;
  }
  char* ws;
  if (workspace) {
    if (workspace_bytes < P.bytes)
      return fail(h, NTT_ERR_WORKSPACE, "workspace %zu < required %zu bytes", workspace_bytes, P.bytes);
    if (!is_device_ptr(workspace)) return fail(h, NTT_ERR_INVALID_ARG, "workspace must be device memory");
    ws = reinterpret_cast<char*>(workspace);
  } else {
    if ((st = ensure_ws(h, P.bytes))) return st;
    ws = reinterpret_cast<char*>(h->ws);
  }
  const int64_t Nloc = s.N / s.dims[d - 1] * P.nloc_last;
  const float* dA = A;
  int used_slot = -1;
  if (!is_device_ptr(A)) {
    for (int q = 0; q < 2; ++q)  // staged by ntt_prefetch_input: wait for its copy, do not copy again
      if (h->slot_ready[q] && h->slot_src[q] == (const void*)A && h->slot_n[q] == Nloc &&
          (used_slot < 0 || h->slot_seq[q] < h->slot_seq[used_slot]))
        used_slot = q;
    if (used_slot >= 0) {
      CU(h, cudaStreamWaitEvent(h->stream, h->cev[used_slot], 0));
      dA = reinterpret_cast<const float*>(h->slot[used_slot]);
      h->slot_ready[used_slot] = false;
    } else {
      if ((st = ensure_stage(h, sizeof(float) * (size_t)Nloc))) return st;
      dA = reinterpret_cast<const float*>(h->stage);
      CU(h, cudaMemcpyAsync((void*)dA, A, sizeof(float) * (size_t)Nloc, cudaMemcpyHostToDevice, h->stream));
    }
  }
  if ((st = check_nonneg(h, dA, 1, Nloc, Nloc, "A"))) return st;
  const bool cores_dev = is_device_ptr(cores);
  float* dcores = cores_dev ? cores : reinterpret_cast<float*>(ws + P.off_cores);
  if (rel_err && (st = ensure_host_part(h, 2))) return st;

  // ---- the device part: captured once into a CUDA graph and replayed while
  // the arguments repeat (NTT_GRAPH=0 disables).  The graph runs on an internal
  // stream ordered after / before the caller's stream by events.
  static const bool graphs_on = [] {
    const char* e = getenv("NTT_GRAPH");
    return !(e && e[0] == '0');
  }();
  std::vector<uint64_t> key;
  if (graphs_on) {
    key = {(uint64_t)(uintptr_t)dA, (uint64_t)d, (uint64_t)iters, seed, (uint64_t)[](float f) { uint32_t u; memcpy(&u, &f, 4); return u; }(eps),
           (uint64_t)(uintptr_t)dcores, (uint64_t)(uintptr_t)ws, (uint64_t)(rel_err != nullptr), (uint64_t)h->prof,
           (uint64_t)(uintptr_t)h->host_part};
    for (int l = 0; l < d; ++l) key.push_back((uint64_t)s.dims[l]);
    for (int l = 1; l < d; ++l) key.push_back((uint64_t)s.r[l]);
  }
  cudaStream_t user = h->stream;
  if (graphs_on) {
    if (!h->gstream) {
      CU(h, cudaStreamCreateWithFlags(&h->gstream, cudaStreamNonBlocking));
      CU(h, cudaEventCreateWithFlags(&h->gev_in, cudaEventDisableTiming));
      CU(h, cudaEventCreateWithFlags(&h->gev_out, cudaEventDisableTiming));
    }
    if ((!h->gexec || key != h->gkey) && !h->prof && h->gexec_alt && key == h->gkey_alt) {
      std::swap(h->gexec, h->gexec_alt);  // the other cached graph (alternating prefetch slots)
      std::swap(h->gkey, h->gkey_alt);
      std::swap(h->glaunches, h->glaunches_alt);
    }
    if (!h->gexec || key != h->gkey) {
      if (h->gexec) {
        CU(h, cudaStreamSynchronize(h->gstream));
        if (!h->prof) {  // keep it as the second cached graph
          if (h->gexec_alt) cudaGraphExecDestroy(h->gexec_alt);
          h->gexec_alt = h->gexec;
          h->gkey_alt = h->gkey;
          h->glaunches_alt = h->glaunches;
        } else {
          cudaGraphExecDestroy(h->gexec);
          if (h->gexec_alt) cudaGraphExecDestroy(h->gexec_alt);
          h->gexec_alt = nullptr;
          h->gkey_alt.clear();
        }
        h->gexec = nullptr;
      }
      h->gkey.clear();
      h->grecs.clear();
      h->gev_used = 0;
      const int64_t l0 = h->launches;
      h->stream = h->gstream;
      h->capturing = true;
      cudaError_t e0 = cudaStreamBeginCapture(h->gstream, cudaStreamCaptureModeThreadLocal);
      ntt_status sd = (e0 == cudaSuccess) ? decompose_device(h, P, s, dA, dcores, ws, iters, seed, eps, rel_err != nullptr)
                                          : NTT_ERR_CUDA;
      cudaGraph_t graph = nullptr;
      cudaError_t e1 = cudaStreamEndCapture(h->gstream, &graph);
      h->capturing = false;
      h->stream = user;
      h->glaunches = h->launches - l0;
      h->launches = l0;
      if (e0 != cudaSuccess || sd != NTT_OK || e1 != cudaSuccess) {
        if (graph) cudaGraphDestroy(graph);
        if (sd != NTT_OK) return sd;
        return fail(h, NTT_ERR_CUDA, "graph capture failed: %s", cudaGetErrorString(e0 != cudaSuccess ? e0 : e1));
      }
      cudaError_t e2 = cudaGraphInstantiate(&h->gexec, graph, 0);
      cudaGraphDestroy(graph);
      if (e2 != cudaSuccess) {
        h->gexec = nullptr;
        return fail(h, NTT_ERR_CUDA, "graph instantiate failed: %s", cudaGetErrorString(e2));
      }
      h->gkey = key;
    }
    CU(h, cudaEventRecord(h->gev_in, user));
    CU(h, cudaStreamWaitEvent(h->gstream, h->gev_in, 0));
    CU(h, cudaGraphLaunch(h->gexec, h->gstream));
    CU(h, cudaEventRecord(h->gev_out, h->gstream));
    CU(h, cudaStreamWaitEvent(user, h->gev_out, 0));
    h->launches += h->glaunches;
    if (h->prof) {
      CU(h, cudaStreamSynchronize(h->gstream));
      prof_fold(h, h->grecs, h->gev_pool);
    }
  } else {
    if ((st = decompose_device(h, P, s, dA, dcores, ws, iters, seed, eps, rel_err != nullptr))) return st;
  }
  if (used_slot >= 0) CU(h, cudaEventRecord(h->uev[used_slot], user));  // the slot may be refilled after this
  if (rel_err) {
    CU(h, cudaStreamSynchronize(user));
    if ((st = finish_error_host(h, rel_err))) return st;
  }
  if (!cores_dev) {
    CU(h, cudaMemcpyAsync(cores, dcores, sizeof(float) * (size_t)s.cores, cudaMemcpyDeviceToHost, user));
    CU(h, cudaStreamSynchronize(user));
  }
  return NTT_OK;
}

// BCD NMF (Alg. 3, readings R22-R27).  Every branch of the iteration is decided on the
// device (bcd.cu, state block BcdState), so one iteration is a fixed launch sequence:
// captured once into a CUDA graph and replayed `iters` times (NTT_BCD_GRAPH=0: eager).
// The two passes over X per iteration (S = W^T X for the H step, P = X H^T for the
// objective and the next W step) run on the fp16x2 tensor-core kernels of the MU path
// where those take the shape (mu_tc16.cu), else on FFMA kernels.
ntt_status ntt_nmf_bcd(ntt_handle h, const float* X, int64_t m, int64_t n, int64_t ldx, int32_t r, int32_t iters,
                       double delta, float* W, float* H, double* objective_trace) {
  if (!h) return NTT_ERR_INVALID_ARG;
  if (!X || !W || !H) return fail(h, NTT_ERR_INVALID_ARG, "null X, W or H");
  if (m < 1 || n < 1 || ldx < n) return fail(h, NTT_ERR_INVALID_ARG, "bad shape m=%lld n=%lld ldx=%lld",
                                              (long long)m, (long long)n, (long long)ldx);
  if (iters < 0) return fail(h, NTT_ERR_INVALID_ARG, "iters < 0");
  if (!(delta >= 0.0 && delta < 1.0)) return fail(h, NTT_ERR_INVALID_ARG, "delta must be in [0, 1)");
  if (r < 1 || r > 32 || r > std::min(m, n)) return fail(h, NTT_ERR_RANK, "BCD needs 1 <= r <= min(m, n, 32)");
  if (h->nranks > 1) return fail(h, NTT_ERR_UNSUPPORTED, "ntt_nmf_bcd runs on a single-GPU handle");
  if (!is_device_ptr(X) || !is_device_ptr(W) || !is_device_ptr(H))
    return fail(h, NTT_ERR_INVALID_ARG, "ntt_nmf_bcd takes device buffers");
  CU(h, cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  // one-pass fused kernels in BCD mode where they win (r <= 8): always for m <= 40 (k_fused);
  // for 40 < m <= 256 (k_fused_c, non-persistent) measured on config 3's shapes against the
  // tensor-core 2-pass path: 256 x 2^20 57 vs 88 ms / 100 it, 256 x 2^10 5.7 vs 7.5, but
  // 256 x 2^15 19 vs 9.5 -- most of the 19 ms was k_bcd_post summing 296 partials in one CTA
  static const int f1_max = [] {
    const char* e = getenv("NTT_BCD_1PASS_M");
    return e ? atoi(e) : 256;
  }();
  // (with the GPU-wide partial pre-sum before k_bcd_post the one-pass path also wins at 2^15:
  // 6.3 vs 8.9 ms / 100 it, so it is taken for every n)
  const bool f1_shape = m <= f1_max && fused_supported(m, n, r, ldx, X, H) &&
                        !getenv("NTT_BCD_NO_1PASS") && !getenv("NTT_BCD_NO_FUSED");
  bool tc = !f1_shape && tc_supported(m, n, r, ldx, X) && !getenv("NTT_NO_TC");
  TcPlan tp;
  if (tc) {
    tp = plan_tc(m, n, r, h->num_sms);
    tc = tp.f16;
  }
  const XhtPlan xp = plan_xht(m, n, h->num_sms), qp = plan_xht(r, n, h->num_sms);
  const int nwc = bcd_w_ctas(m);
  const int nS = tc ? tp.splitH16 : bcd_spart_splits(m, n, h->num_sms);
  // short-wide X (r <= 8, m <= 256): P, Q from the 1-pass fused kernel's acc-only mode
  const bool fa = !tc && fused_supported(m, n, r, ldx, X, H) && !getenv("NTT_BCD_NO_FUSED");
  const int fparts = fa ? fused_partials(m, n, r, h->num_sms) : 0;
  const bool f1 = fa && f1_shape;  // the whole H half-iteration in one pass
  size_t o = 0;
  auto take = [&](size_t b) {
    size_t at = o;
    o = align_up(o + b);
    return at;
  };
  const size_t oWm = take(sizeof(float) * m * r), oWp = take(sizeof(float) * m * r);
  const size_t oHm = take(sizeof(float) * r * n), oHp = take(sizeof(float) * r * n);
  const size_t oP0 = take(sizeof(double) * m * r), oP1 = take(sizeof(double) * m * r);
  const size_t oQ0 = take(sizeof(double) * r * r), oQ1 = take(sizeof(double) * r * r);
  const size_t oG = take(sizeof(double) * r * r), oC = take(sizeof(double) * r);
  const size_t oPp = tc ? 0 : take(sizeof(double) * (size_t)std::max(xp.ncs, fparts) * m * r);
  const size_t oSp = (tc || nS == 1) ? 0 : take(sizeof(double) * (size_t)nS * n * r);
  const size_t oQp = take(sizeof(double) * (size_t)std::max(qp.ncs, fparts) * r * r);
  const size_t oSH = take(sizeof(double) * 96);  // row scales of H_m, H_prev, H_prev2 (k_bcd_hscale)
  const size_t oCp = take(sizeof(double) * (size_t)nwc * r), oGp = take(sizeof(double) * (size_t)nwc * r * r);
  const int ndot = bcd_dot_ctas(m * r, h->num_sms);
  const size_t oD = take(sizeof(double) * ndot), oSq = take(sizeof(double) * sumsq_ctas());
  const size_t oBs = take(sizeof(double) * BS_COUNT);
  const size_t oTc = tc ? take(tp.bytes) : 0;
  // the trace goes last: it is the only region whose size depends on iters, so no offset the
  // cached iteration graph bakes in (tensor-core scratch, tensor maps) moves with iters
  const size_t oTr = take(sizeof(double) * std::max(iters, 1));
  ntt_status s = ensure_ws(h, o);
  if (s) return s;
  char* ws = reinterpret_cast<char*>(h->ws);
  float* Wm = reinterpret_cast<float*>(ws + oWm);
  float* Wp = reinterpret_cast<float*>(ws + oWp);
  float* Hm = reinterpret_cast<float*>(ws + oHm);
  float* Hp = reinterpret_cast<float*>(ws + oHp);
  double* Pc = reinterpret_cast<double*>(ws + oP0);  // X H_prev^T, H_prev H_prev^T (accepted H)
  double* Pn = reinterpret_cast<double*>(ws + oP1);  // the same for the candidate H
  double* Qc = reinterpret_cast<double*>(ws + oQ0);
  double* Qn = reinterpret_cast<double*>(ws + oQ1);
  double* G = reinterpret_cast<double*>(ws + oG);
  double* c = reinterpret_cast<double*>(ws + oC);
  double* Qpart = reinterpret_cast<double*>(ws + oQp);
  double* cpart = reinterpret_cast<double*>(ws + oCp);
  double* Gpart = reinterpret_cast<double*>(ws + oGp);
  double* dotpart = reinterpret_cast<double*>(ws + oD);  // per-CTA partials of <W, X H^T>
  double* sq = reinterpret_cast<double*>(ws + oSq);
  double* bs = reinterpret_cast<double*>(ws + oBs);
  double* dtrace = reinterpret_cast<double*>(ws + oTr);
  char* tws = ws + oTc;
  double* Ppart = tc ? reinterpret_cast<double*>(tws + tp.off_P) : reinterpret_cast<double*>(ws + oPp);
  double* Spart = tc ? reinterpret_cast<double*>(tws + tp.off_S) : reinterpret_cast<double*>(ws + oSp);
  const int nP = tc ? tp.splitW16 : fa ? fparts : xp.ncs;
  double* sH = reinterpret_cast<double*>(ws + oSH);
  TcMaps maps;
  unsigned* mxh = tc ? tc16_max_slot(tp, tws, 5) : nullptr;  // max H, then max W (slot 6)
  unsigned* mxw = tc ? tc16_max_slot(tp, tws, 6) : nullptr;
  const double xbytes = 4.0 * (double)m * (double)n;
  const char* fe = getenv("NTT_BCD_FLUSH");
  const int bflush = fe ? std::max(1, atoi(fe)) : 4;
  const int bef = (double)m * (double)ldx * 4.0 > 0.6 * (double)h->l2_bytes ? 1 : 0;  // X > L2: evict-first
  auto spec = [&](const double* M, double* out) -> ntt_status {  // spectral norm of an r x r Gram
    LAUNCH(h, launch_spec_norm(M, r, out, st));
    return NTT_OK;
  };
  // P = X H^T, Q = H H^T; in the iteration also the <W, P> partials of the objective, and
  // the fp16 scale of H from the max k_bcd_hup left in slot 5
  auto pq = [&](const float* Hs, double* P, double* Q, bool in_iter) -> ntt_status {
    if (tc) {
      if (in_iter) LAUNCH(h, tc16_pack_h_slot(tp, Hs, tws, st, 5));
      else LAUNCH(h, tc16_pack_h_fresh(tp, Hs, tws, st));
      PLAUNCH(h, 6, xbytes, tc16_pass_w(tp, maps, tws, bef, st, bflush));
    } else if (fa) {  // one pass: P = X H^T and Q = H H^T partials per CTA
      PLAUNCH(h, 1, xbytes + 4.0 * r * (double)n,
              launch_fused(X, ldx, m, n, r, W, nullptr, 0, 0.0f, const_cast<float*>(Hs), Ppart, Qpart, kFusedAcc,
                           fused_grid(m, n, r, h->num_sms), st));
    } else {
      PLAUNCH(h, 1, xbytes, launch_xht_partial(X, ldx, m, n, Hs, n, r, xp, Ppart, st));
    }
    LAUNCH(h, launch_bcd_psum_dot(Ppart, nP, m * r, in_iter ? W : nullptr, P, in_iter ? dotpart : nullptr,
                                  h->num_sms, st));
    if (!fa) LAUNCH(h, launch_xht_partial(Hs, n, r, n, Hs, n, r, qp, Qpart, st));
    LAUNCH(h, launch_sum_partials(Qpart, fa ? fparts : qp.ncs, (int64_t)r * r, Q, st));
    return NTT_OK;
  };
  if ((s = check_nonneg(h, X, m, n, ldx, "X"))) return s;
  // ---- init (Alg. 3 l.1-4, R22, R23)
  CU(h, cudaMemsetAsync(bs, 0, sizeof(double) * BS_COUNT, st));
  LAUNCH(h, launch_sumsq(X, m, n, ldx, sq, st, bef != 0));
  LAUNCH(h, launch_sum_partials(sq, sumsq_ctas(), 1, bs + BS_XX, st));
  LAUNCH(h, launch_sumsq(W, m, r, r, sq, st));
  LAUNCH(h, launch_sum_partials(sq, sumsq_ctas(), 1, bs + BS_W0, st));
  LAUNCH(h, launch_sumsq(H, r, n, n, sq, st));
  LAUNCH(h, launch_sum_partials(sq, sumsq_ctas(), 1, bs + BS_H0, st));
  double nrm[3] = {0.0, 0.0, 0.0};  // ||X||^2, ||W0||^2, ||H0||^2 (BS_XX, BS_W0, BS_H0)
  CU(h, cudaMemcpyAsync(nrm, bs + BS_XX, sizeof(nrm), cudaMemcpyDeviceToHost, st));
  CU(h, cudaStreamSynchronize(st));
  if (!(nrm[0] > 0.0)) return fail(h, NTT_ERR_DEGENERATE, "||X|| = 0");
  // l.2 divides by ||W0|| and ||H0||: an all-zero initial factor has no normalisation
  if (!(nrm[1] > 0.0) || !(nrm[2] > 0.0)) return fail(h, NTT_ERR_DEGENERATE, "||W0|| = 0 or ||H0|| = 0");
  LAUNCH(h, launch_scale_copy(W, Wm, Wp, m * r, bs + BS_XX, bs + BS_W0, st));
  LAUNCH(h, launch_scale_copy(H, Hm, Hp, (int64_t)r * n, bs + BS_XX, bs + BS_H0, st));
  LAUNCH(h, launch_bcd_hout(Hp, r, n, sH, nullptr, 1, nullptr, st));  // sH = 1
  if (tc) {
    LAUNCH(h, tc_prepare(tp, X, ldx, Hp, tws, &maps, st));
    LAUNCH(h, tc16_prepare(tp, X, ldx, Hp, tws, &maps, st));
  }
  if ((s = pq(Hp, Pc, Qc, false))) return s;
  LAUNCH(h, launch_bcd_wnorm(Wp, Wp, m, r, nullptr, Gpart, nullptr, st));  // W_prev^T W_prev (no normalisation)
  LAUNCH(h, launch_sum_partials(Gpart, nwc, (int64_t)r * r, G, st));
  if ((s = spec(Qc, bs + BS_LW))) return s;
  if ((s = spec(G, bs + BS_LH))) return s;
  // ---- one iteration (l.5-27), a fixed launch sequence
  // small W (non-TC): one-CTA stages for the W side and for everything after the H pass
  const bool cta = !tc && bcd_cta_ok(m, r) && !getenv("NTT_BCD_NO_CTA");
  // one-pass path with k_fused's staged H: the pass forms H_m from the two H buffers itself
  // (BS_FOLD), so the per-iteration H commit (3 H-sized streams) disappears
  const bool fold = cta && f1 && fused_fold_ok(m, n, r, ldx, X, H, Hp) && !getenv("NTT_BCD_NO_FOLD");
  const bool presum = !getenv("NTT_BCD_NO_PRESUM");
  LAUNCH(h, launch_bcd_init(bs, delta, fold, h->bcd_force, st));
  auto iteration_cta = [&]() -> ntt_status {
    LAUNCH(h, launch_bcd_wside(Wm, W, Wp, (int)m, r, Pc, Qc, bs, c, G, sH, st));  // l.5-10
    int nPp = nP, nQp = qp.ncs;
    if (f1) {  // l.11-15 in one pass
      PersistArgs pa;
      pa.iters = 0;
      pa.part = pa.red = nullptr;
      pa.ctr = nullptr;
      pa.Wout = nullptr;
      pa.trace = nullptr;
      pa.bcdL = bs + BS_LH;
      pa.bcdS = sH;
      pa.Hout = H;  // the two H buffers swap roles on acceptance (k_bcd_commit_h_role)
      pa.Hout2 = Hp;
      pa.bcdRole = bs + BS_ROLE;
      pa.bcdFold = fold;
      PLAUNCH(h, 0, xbytes + 8.0 * r * (double)n,
              launch_fused(X, ldx, m, n, r, W, G, 1, 0.0f, Hm, Ppart, Qpart, kFusedUpdate | kFusedAcc,
                           fused_grid(m, n, r, h->num_sms), st, &pa));
      nPp = nQp = fparts;
    } else {
      if (nS == 1) {
        PLAUNCH(h, 5, xbytes + 8.0 * r * (double)n, launch_bcd_shup(X, ldx, m, n, W, r, G, bs + BS_LH, Hm, sH, H, st));
      } else {
        PLAUNCH(h, 5, xbytes, launch_bcd_spart(X, ldx, m, n, W, r, nS, Spart, st));
        LAUNCH(h, launch_bcd_hup(Spart, nS, n, r, G, bs + BS_LH, Hm, sH, H, nullptr, h->num_sms, st));
      }
      if (fa) {
        PLAUNCH(h, 1, xbytes + 4.0 * r * (double)n,
                launch_fused(X, ldx, m, n, r, W, nullptr, 0, 0.0f, H, Ppart, Qpart, kFusedAcc,
                             fused_grid(m, n, r, h->num_sms), st));
        nPp = nQp = fparts;
      } else {
        PLAUNCH(h, 1, xbytes, launch_xht_partial(X, ldx, m, n, H, n, r, xp, Ppart, st));
        LAUNCH(h, launch_xht_partial(H, n, r, n, H, n, r, qp, Qpart, st));
        nPp = xp.ncs;
      }
    }
    // many partials (k_fused_c writes 2 per SM; m = 256): reduce them across the GPU first -- the
    // one-CTA post kernel summing 296 x 2048 doubles itself took 225 us of a 600 us iteration
    const double* Pin = Ppart;
    const double* Qin = Qpart;
    if (presum && (double)nPp * (double)(m * r) > 131072.0) {
      LAUNCH(h, launch_sum_partials(Ppart, nPp, m * r, Pn, st));
      LAUNCH(h, launch_sum_partials(Qpart, nQp, (int64_t)r * r, Qn, st));
      Pin = Pn;
      Qin = Qn;
      nPp = nQp = 1;
    }
    LAUNCH(h, launch_bcd_post(Pin, nPp, Qin, nQp, (int)m, r, W, Wm, Wp, Pc, Qc, c, G, bs, dtrace, st));
    if (f1) {  // l.18-27 (H side); with the fold the next pass forms H_m itself
      if (!fold) LAUNCH(h, launch_bcd_commit_h_role(H, Hp, Hm, r, n, sH, bs, st));
    } else {
      LAUNCH(h, launch_bcd_commit_h(H, Hm, Hp, r, n, sH, bs, st));
    }
    return NTT_OK;
  };
  auto iteration = [&]() -> ntt_status {
    if (cta) return iteration_cta();
    if ((s = spec(Qc, bs + BS_LW))) return s;                                    // l.7
    LAUNCH(h, launch_bcd_w(Wm, m, r, Pc, Qc, bs + BS_LW, W, cpart, st));          // l.6-8
    LAUNCH(h, launch_sum_partials(cpart, nwc, r, c, st));
    LAUNCH(h, launch_bcd_wnorm(W, Wp, m, r, c, Gpart, mxw, st));                  // l.9 (R24)
    LAUNCH(h, launch_bcd_hscale(sH, r, c, st));
    LAUNCH(h, launch_sum_partials(Gpart, nwc, (int64_t)r * r, G, st));             // l.10
    if ((s = spec(G, bs + BS_LH))) return s;
    if (tc) {                                                                     // S = W^T X
      LAUNCH(h, tc16_pack_w_slot(tp, W, tws, st, 6));
      PLAUNCH(h, 7, xbytes, tc16_pass_h(tp, maps, tws, bef, st, bflush));
    }
    if (f1) {  // ONE pass (m <= 40): S, the H step, and P, Q of the new H (l.11-15), k_fused in BCD mode
      PersistArgs pa;
      pa.iters = 0;
      pa.part = pa.red = nullptr;
      pa.ctr = nullptr;
      pa.Wout = nullptr;
      pa.trace = nullptr;
      pa.bcdL = bs + BS_LH;
      pa.bcdS = sH;
      pa.Hout = H;
      PLAUNCH(h, 0, xbytes + 8.0 * r * (double)n,
              launch_fused(X, ldx, m, n, r, W, G, 1, 0.0f, Hm, Ppart, Qpart, kFusedUpdate | kFusedAcc,
                           fused_grid(m, n, r, h->num_sms), st, &pa));
      LAUNCH(h, launch_bcd_psum_dot(Ppart, fparts, m * r, W, Pn, dotpart, h->num_sms, st));
      LAUNCH(h, launch_sum_partials(Qpart, fparts, (int64_t)r * r, Qn, st));
    } else {
      if (!tc && nS == 1) {  // S and the H step in one pass (l.11-14)
        PLAUNCH(h, 5, xbytes + 8.0 * r * (double)n, launch_bcd_shup(X, ldx, m, n, W, r, G, bs + BS_LH, Hm, sH, H, st));
      } else {
        if (!tc) PLAUNCH(h, 5, xbytes, launch_bcd_spart(X, ldx, m, n, W, r, nS, Spart, st));
        LAUNCH(h, launch_bcd_hup(Spart, nS, n, r, G, bs + BS_LH, Hm, sH, H, mxh, h->num_sms, st));  // l.11-14
      }
      if ((s = pq(H, Pn, Qn, true))) return s;                                               // l.15
    }
    LAUNCH(h, launch_bcd_decide(bs, dtrace, dotpart, ndot, G, Qn, r, mxh, st));             // l.16-17 (R25)
    LAUNCH(h, launch_bcd_commit(W, Wm, Wp, m * r, bs, BS_WW, st));                    // l.18-27
    LAUNCH(h, launch_bcd_commit_h(H, Hm, Hp, r, n, sH, bs, st));
    LAUNCH(h, launch_bcd_commit_pq(Pc, Pn, m, r, Qc, Qn, c, bs, sH, st));
    return NTT_OK;
  };
  const char* ge = getenv("NTT_BCD_GRAPH");
  const bool graph = iters >= 2 && !h->prof && !(ge && ge[0] == '0');
  if (graph) {
    if (!h->gstream) {
      CU(h, cudaStreamCreateWithFlags(&h->gstream, cudaStreamNonBlocking));
      CU(h, cudaEventCreateWithFlags(&h->gev_in, cudaEventDisableTiming));
      CU(h, cudaEventCreateWithFlags(&h->gev_out, cudaEventDisableTiming));
    }
    CU(h, cudaEventRecord(h->gev_in, st));
    CU(h, cudaStreamWaitEvent(h->gstream, h->gev_in, 0));
    const int64_t l0 = h->launches;
    st = h->gstream;
    // the graph bakes in pointers, sizes and tensor maps: reuse it while they are unchanged
    char kb[256];
    snprintf(kb, sizeof(kb), "%p %p %p %p %lld %lld %lld %d %zu", (const void*)X, (void*)W, (void*)H, (void*)h->ws,
             (long long)m, (long long)n, (long long)ldx, r, oTr);
    if (!h->bcd_exec || h->bcd_key != kb) {
      if (h->bcd_exec) {
        cudaGraphExecDestroy(h->bcd_exec);
        h->bcd_exec = nullptr;
        h->bcd_key.clear();
      }
      cudaError_t e0 = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
      ntt_status si = e0 == cudaSuccess ? iteration() : NTT_ERR_CUDA;
      cudaGraph_t g = nullptr;
      cudaError_t e1 = cudaStreamEndCapture(st, &g);
      h->bcd_per_it = h->launches - l0;
      h->launches = l0;
      if (e0 != cudaSuccess || si != NTT_OK || e1 != cudaSuccess) {
        if (g) cudaGraphDestroy(g);
        if (si != NTT_OK) return si;
        return fail(h, NTT_ERR_CUDA, "BCD graph capture failed: %s", cudaGetErrorString(e0 ? e0 : e1));
      }
      cudaError_t e2 = cudaGraphInstantiate(&h->bcd_exec, g, 0);
      cudaGraphDestroy(g);
      if (e2 != cudaSuccess) {
        h->bcd_exec = nullptr;
        return fail(h, NTT_ERR_CUDA, "BCD graph instantiate: %s", cudaGetErrorString(e2));
      }
      h->bcd_key = kb;
    }
    cudaError_t el = cudaSuccess;
    for (int it = 0; it < iters && el == cudaSuccess; ++it) el = cudaGraphLaunch(h->bcd_exec, st);
    if (el != cudaSuccess) return fail(h, NTT_ERR_CUDA, "BCD graph launch: %s", cudaGetErrorString(el));
    h->launches = l0 + h->bcd_per_it * iters;
    CU(h, cudaEventRecord(h->gev_out, st));
    st = h->stream;
    CU(h, cudaStreamWaitEvent(st, h->gev_out, 0));
  } else {
    for (int it = 0; it < iters; ++it)
      if ((s = iteration())) return s;
  }
  // the last accepted iterates (l.28)
  CU(h, cudaMemcpyAsync(W, Wp, sizeof(float) * m * r, cudaMemcpyDeviceToDevice, st));
  if (cta && f1) LAUNCH(h, launch_bcd_hout_role(H, Hp, r, n, sH, bs, st));  // logical H_prev (role-swapped)
  else LAUNCH(h, launch_bcd_hout(Hp, r, n, sH, H, 0, bs, st));        // logical H_prev = diag(sHp) Hp
  if (objective_trace && iters > 0)
    CU(h, cudaMemcpyAsync(objective_trace, dtrace, sizeof(double) * iters, cudaMemcpyDeviceToHost, st));
  CU(h, cudaStreamSynchronize(st));
  return NTT_OK;
}

ntt_status ntt_decompose_eps(ntt_handle h, const float* A, int32_t d, const int64_t* dims, double tt_eps,
                             const int32_t* max_ranks, int32_t iters, uint64_t seed, float eps, float* cores,
                             int64_t cores_capacity, int32_t* ranks_out, double* rel_err) {
  if (!h) return NTT_ERR_INVALID_ARG;
  if (!A || !cores || !ranks_out) return fail(h, NTT_ERR_INVALID_ARG, "null A, cores or ranks_out");
  if (iters < 0) return fail(h, NTT_ERR_INVALID_ARG, "iters < 0");
  if (!(eps >= 0.0f)) return fail(h, NTT_ERR_INVALID_ARG, "eps must be >= 0");
  if (!(tt_eps >= 0.0)) return fail(h, NTT_ERR_INVALID_ARG, "tt_eps must be >= 0");
  if (h->nranks > 1)
    return fail(h, NTT_ERR_UNSUPPORTED, "ntt_decompose_eps runs on a single-GPU handle (rank rule per step)");
  // ---- shape, caps (upper bounds of the data-dependent ranks) and workspace plan
  TTShape s0;
  std::vector<int32_t> ones((size_t)std::max(d - 1, 1), 1);
  ntt_status st = check_tt(h, d, dims, ones.data(), &s0, false);
  if (st) return st;
  int64_t cap[65], mcap[65], ncol[65];
  cap[0] = 1;
  int64_t rest = s0.N;
  size_t hbuf[2] = {1, 1}, wmax = 1, mu_bytes = 0, rk_bytes = 0, cores_cap = 0;
  for (int l = 1; l < d; ++l) {
    mcap[l] = cap[l - 1] * s0.dims[l - 1];
    rest /= s0.dims[l - 1];
    ncol[l] = rest;
    int64_t c = std::min<int64_t>({(int64_t)kMaxRank, mcap[l], ncol[l]});
    if (max_ranks) {
      if (max_ranks[l - 1] < 1) return fail(h, NTT_ERR_RANK, "max_ranks[%d] < 1", l - 1);
      c = std::min<int64_t>(c, max_ranks[l - 1]);
    }
    cap[l] = c;
    hbuf[(l - 1) & 1] = std::max(hbuf[(l - 1) & 1], (size_t)(c * ncol[l]));
    wmax = std::max(wmax, (size_t)(mcap[l] * c));
    cores_cap += (size_t)(mcap[l] * c);
    // run_mu scratch for every (r_{l-1}, r_l) the rule may pick
    for (int64_t rp = 1; rp <= cap[l - 1]; ++rp)
      for (int64_t r = 1; r <= c && r <= rp * s0.dims[l - 1]; ++r)
        mu_bytes = std::max(mu_bytes, plan_mu(rp * s0.dims[l - 1], ncol[l], (int)r, h->num_sms, false).bytes);
    // rank-rule scratch for every Gram size the step can see (min(m, n) <= kRankMaxN is checked per step)
    const int64_t nmax = std::min<int64_t>({mcap[l], ncol[l], kRankMaxN});
    for (int64_t Nn = 1; Nn <= nmax; ++Nn)
      rk_bytes = std::max(rk_bytes, rank_rule_bytes(Nn, std::max(mcap[l], ncol[l]), h->num_sms));
  }
  cores_cap += (size_t)(cap[d - 1] * s0.dims[d - 1]);
  size_t o = 0;
  const size_t off_h0 = o;
  o = align_up(o + sizeof(float) * hbuf[0]);
  const size_t off_h1 = o;
  o = align_up(o + sizeof(float) * hbuf[1]);
  const size_t off_w = o;
  o = align_up(o + sizeof(float) * wmax);
  const size_t off_c = o;
  o = align_up(o + sizeof(float) * cores_cap);
  const size_t off_mu = o;
  o = align_up(o + mu_bytes);
  const size_t off_rk = o;
  o = align_up(o + rk_bytes);
  const size_t off_int = o;
  o = align_up(o + 64);
  CU(h, cudaSetDevice(h->device));
  if ((st = ensure_ws(h, o))) return st;
  char* ws = reinterpret_cast<char*>(h->ws);
  cudaStream_t cs = h->stream;
  const float* dA = A;
  if (!is_device_ptr(A)) {
    if ((st = ensure_stage(h, sizeof(float) * (size_t)s0.N))) return st;
    dA = reinterpret_cast<const float*>(h->stage);
    CU(h, cudaMemcpyAsync((void*)dA, A, sizeof(float) * (size_t)s0.N, cudaMemcpyHostToDevice, cs));
  }
  if ((st = check_nonneg(h, dA, 1, s0.N, s0.N, "A"))) return st;
  float* hb[2] = {reinterpret_cast<float*>(ws + off_h0), reinterpret_cast<float*>(ws + off_h1)};
  float* Wd = reinterpret_cast<float*>(ws + off_w);
  float* dcores = reinterpret_cast<float*>(ws + off_c);
  int* d_rank = reinterpret_cast<int*>(ws + off_int);
  // ---- the sweep: rank rule on the current unfolding, then MU NMF with that rank (Alg. 2 l.4-9)
  const float* X = dA;
  float* Hl = nullptr;
  int64_t rprev = 1, coff = 0;
  for (int l = 1; l < d; ++l) {
    const int64_t m = rprev * s0.dims[l - 1], n = ncol[l];
    h->cur_step = l;
    if (std::min(m, n) > kRankMaxN)
      return fail(h, NTT_ERR_UNSUPPORTED, "rank rule needs min(m, n) <= %d (step %d: %lld x %lld)", kRankMaxN, l,
                  (long long)m, (long long)n);
    LAUNCH(h, launch_rank_rule(X, m, n, n, tt_eps, ws + off_rk, h->num_sms, d_rank, nullptr, cs));
    int rk = 1;
    CU(h, cudaMemcpyAsync(&rk, d_rank, sizeof(int), cudaMemcpyDeviceToHost, cs));
    CU(h, cudaStreamSynchronize(cs));
    const int r = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)rk, cap[l], m, n}));
    ranks_out[l - 1] = r;
    Hl = hb[(l - 1) & 1];
    LAUNCH(h, launch_fill_uniform(Wd, m * r, seed, stream_w(l), 0, cs));
    LAUNCH(h, launch_fill_uniform(Hl, (int64_t)r * n, seed, stream_h(l), 0, cs));
    MuPlan p = plan_mu(m, n, r, h->num_sms, false);
    if (p.bytes > mu_bytes) return fail(h, NTT_ERR_WORKSPACE, "internal: MU scratch plan exceeded");
    if ((st = run_mu(h, p, X, n, iters, eps, Wd, Hl, ws + off_mu, nullptr))) return st;
    CU(h, cudaMemcpyAsync(dcores + coff, Wd, sizeof(float) * (size_t)(m * r), cudaMemcpyDeviceToDevice, cs));
    coff += m * r;
    X = Hl;
    rprev = r;
  }
  h->cur_step = 0;
  const int64_t ncl = rprev * s0.dims[d - 1];
  CU(h, cudaMemcpyAsync(dcores + coff, Hl, sizeof(float) * (size_t)ncl, cudaMemcpyDeviceToDevice, cs));
  coff += ncl;
  if (coff > cores_capacity)
    return fail(h, NTT_ERR_WORKSPACE, "cores_capacity %lld < %lld floats for the chosen ranks",
                (long long)cores_capacity, (long long)coff);
  CU(h, cudaMemcpyAsync(cores, dcores, sizeof(float) * (size_t)coff, cudaMemcpyDefault, cs));
  CU(h, cudaStreamSynchronize(cs));
  if (rel_err) {
    TTShape s;
    if ((st = check_tt(h, d, dims, ranks_out, &s, true))) return st;
    if ((st = contract_stream(h, s, cores, nullptr, 0.0f, 0, A, rel_err))) return st;
  }
  return NTT_OK;
}

// nTT sweep with the paper's BCD NMF at every step (Alg. 2 + Alg. 3).  Sweep buffers are
// stream-ordered allocations of their own, so the BCD calls may grow the handle workspace.
ntt_status ntt_decompose_bcd(ntt_handle h, const float* A, int32_t d, const int64_t* dims, const int32_t* ranks,
                             int32_t iters, uint64_t seed, double delta, float* cores, double* rel_err) {
  if (!h) return NTT_ERR_INVALID_ARG;
  if (!A || !cores) return fail(h, NTT_ERR_INVALID_ARG, "null A or cores");
  if (iters < 0) return fail(h, NTT_ERR_INVALID_ARG, "iters < 0");
  if (!(delta >= 0.0 && delta < 1.0)) return fail(h, NTT_ERR_INVALID_ARG, "delta must be in [0, 1)");
  if (h->nranks > 1) return fail(h, NTT_ERR_UNSUPPORTED, "ntt_decompose_bcd runs on a single-GPU handle");
  TTShape s;
  ntt_status st = check_tt(h, d, dims, ranks, &s, true);
  if (st) return st;
  for (int l = 0; l + 1 < d; ++l)
    if (ranks[l] > 32) return fail(h, NTT_ERR_RANK, "BCD sweep needs ranks <= 32 (rank %d = %d)", l, ranks[l]);
  CU(h, cudaSetDevice(h->device));
  cudaStream_t cs = h->stream;
  size_t hmax = 1, wmax = 1;
  {
    int64_t rest = s.N, rp = 1;
    for (int l = 1; l < d; ++l) {
      rest /= s.dims[l - 1];
      hmax = std::max(hmax, (size_t)(ranks[l - 1] * rest));
      wmax = std::max(wmax, (size_t)(rp * s.dims[l - 1] * ranks[l - 1]));
      rp = ranks[l - 1];
    }
  }
  const float* dA = A;
  if (!is_device_ptr(A)) {
    if ((st = ensure_stage(h, sizeof(float) * (size_t)s.N))) return st;
    dA = reinterpret_cast<const float*>(h->stage);
    CU(h, cudaMemcpyAsync((void*)dA, A, sizeof(float) * (size_t)s.N, cudaMemcpyHostToDevice, cs));
  }
  if ((st = check_nonneg(h, dA, 1, s.N, s.N, "A"))) return st;
  float* buf = nullptr;
  const size_t nfl = 2 * hmax + wmax + (size_t)s.cores;
  if (h->sweep_bytes < sizeof(float) * nfl) {  // grown once, reused by later calls
    CU(h, cudaStreamSynchronize(cs));
    if (h->sweep) CU(h, cudaFree(h->sweep));
    h->sweep = nullptr;
    h->sweep_bytes = 0;
    CU(h, cudaMalloc(&h->sweep, sizeof(float) * nfl));
    h->sweep_bytes = sizeof(float) * nfl;
  }
  buf = reinterpret_cast<float*>(h->sweep);
  float* hb[2] = {buf, buf + hmax};
  float* Wd = buf + 2 * hmax;
  float* dcores = Wd + wmax;
  const float* X = dA;
  float* Hl = nullptr;
  int64_t rprev = 1, coff = 0, rest = s.N;
  for (int l = 1; l < d; ++l) {
    const int64_t m = rprev * s.dims[l - 1];
    rest /= s.dims[l - 1];
    const int r = ranks[l - 1];
    h->cur_step = l;
    Hl = hb[(l - 1) & 1];
    LAUNCH(h, launch_fill_uniform(Wd, m * r, seed, stream_w(l), 0, cs));
    LAUNCH(h, launch_fill_uniform(Hl, (int64_t)r * rest, seed, stream_h(l), 0, cs));
    if ((st = ntt_nmf_bcd(h, X, m, rest, rest, r, iters, delta, Wd, Hl, nullptr))) return st;
    CU(h, cudaMemcpyAsync(dcores + coff, Wd, sizeof(float) * (size_t)(m * r), cudaMemcpyDeviceToDevice, cs));
    coff += m * r;
    X = Hl;
    rprev = r;
  }
  h->cur_step = 0;
  const int64_t ncl = rprev * s.dims[d - 1];
  CU(h, cudaMemcpyAsync(dcores + coff, Hl, sizeof(float) * (size_t)ncl, cudaMemcpyDeviceToDevice, cs));
  CU(h, cudaMemcpyAsync(cores, dcores, sizeof(float) * (size_t)s.cores, cudaMemcpyDefault, cs));
  CU(h, cudaStreamSynchronize(cs));
  if (rel_err) {
    if ((st = contract_stream(h, s, cores, nullptr, 0.0f, 0, A, rel_err))) return st;
  }
  return NTT_OK;
}

// TT-SVD baseline (SURVEY s.8(f) f4, reading R28; tt_svd.cu).  Same sweep, shapes and rank
// rule as ntt_decompose_eps; the NMF of each step is replaced by the truncated SVD.
ntt_status ntt_tt_svd(ntt_handle h, const float* A, int32_t d, const int64_t* dims, double tt_eps,
                      const int32_t* max_ranks, float* cores, int64_t cores_capacity, int32_t* ranks_out,
                      double* rel_err) {
  if (!h) return NTT_ERR_INVALID_ARG;
  if (!A || !cores || !ranks_out) return fail(h, NTT_ERR_INVALID_ARG, "null A, cores or ranks_out");
  if (!(tt_eps >= 0.0)) return fail(h, NTT_ERR_INVALID_ARG, "tt_eps must be >= 0");
  if (h->nranks > 1) return fail(h, NTT_ERR_UNSUPPORTED, "ntt_tt_svd runs on a single-GPU handle");
  TTShape s0;
  std::vector<int32_t> ones((size_t)std::max(d - 1, 1), 1);
  ntt_status st = check_tt(h, d, dims, ones.data(), &s0, false);
  if (st) return st;
  int64_t cap[65], mcap[65], ncol[65];
  cap[0] = 1;
  int64_t rest = s0.N;
  size_t hbuf[2] = {1, 1}, cores_cap = 0, stepb = 0;
  for (int l = 1; l < d; ++l) {
    mcap[l] = cap[l - 1] * s0.dims[l - 1];
    rest /= s0.dims[l - 1];
    ncol[l] = rest;
    int64_t c = std::min<int64_t>({(int64_t)kMaxRank, mcap[l], ncol[l]});
    if (max_ranks) {
      if (max_ranks[l - 1] < 1) return fail(h, NTT_ERR_RANK, "max_ranks[%d] < 1", l - 1);
      c = std::min<int64_t>(c, max_ranks[l - 1]);
    }
    cap[l] = c;
    hbuf[(l - 1) & 1] = std::max(hbuf[(l - 1) & 1], (size_t)(c * ncol[l]));
    cores_cap += (size_t)(mcap[l] * c);
    // per-step scratch for every m the previous rank allows
    for (int64_t rp = 1; rp <= cap[l - 1]; ++rp) {
      const int64_t m = rp * s0.dims[l - 1], n = ncol[l], N = std::min(m, n);
      if (N > kRankMaxN) continue;  // rejected at run time
      size_t b = align_up(rank_rule_bytes(N, std::max(m, n), h->num_sms)) + align_up(svd_eig_bytes(N)) +
                 align_up(sizeof(double) * (size_t)N * 64) + align_up(sizeof(double) * (size_t)(N + 64 * 4 + 8));
      if (m <= n) {
        b += align_up(sizeof(double) * (size_t)bcd_spart_splits(m, n, h->num_sms) * n * c);
      } else {
        const XhtPlan xp = plan_xht(m, n, h->num_sms);
        b += align_up(sizeof(double) * (size_t)xp.ncs * m * c) + align_up(sizeof(double) * (size_t)m * c) +
             align_up(sizeof(float) * (size_t)c * n);
      }
      stepb = std::max(stepb, b);
    }
  }
  cores_cap += (size_t)(cap[d - 1] * s0.dims[d - 1]);
  size_t o = 0;
  const size_t off_h0 = o;
  o = align_up(o + sizeof(float) * hbuf[0]);
  const size_t off_h1 = o;
  o = align_up(o + sizeof(float) * hbuf[1]);
  const size_t off_c = o;
  o = align_up(o + sizeof(float) * cores_cap);
  const size_t off_step = o;
  o = align_up(o + stepb);
  CU(h, cudaSetDevice(h->device));
  if ((st = ensure_ws(h, o))) return st;
  char* ws = reinterpret_cast<char*>(h->ws);
  cudaStream_t cs = h->stream;
  const float* dA = A;
  if (!is_device_ptr(A)) {
    if ((st = ensure_stage(h, sizeof(float) * (size_t)s0.N))) return st;
    dA = reinterpret_cast<const float*>(h->stage);
    CU(h, cudaMemcpyAsync((void*)dA, A, sizeof(float) * (size_t)s0.N, cudaMemcpyHostToDevice, cs));
  }
  float* hb[2] = {reinterpret_cast<float*>(ws + off_h0), reinterpret_cast<float*>(ws + off_h1)};
  float* dcores = reinterpret_cast<float*>(ws + off_c);
  const float* X = dA;
  float* Xn = nullptr;
  int64_t rprev = 1, coff = 0;
  for (int l = 1; l < d; ++l) {
    const int64_t m = rprev * s0.dims[l - 1], n = ncol[l], N = std::min(m, n);
    h->cur_step = l;
    if (N > kRankMaxN)
      return fail(h, NTT_ERR_UNSUPPORTED, "TT-SVD needs min(m, n) <= %d (step %d: %lld x %lld)", kRankMaxN, l, (long long)m,
                  (long long)n);
    const int rcap = (int)std::min<int64_t>(cap[l], N);
    // step scratch
    char* sp = ws + off_step;
    size_t so = 0;
    auto take = [&](size_t b) {
      char* at = sp + so;
      so = align_up(so + b);
      return at;
    };
    char* gws = take(rank_rule_bytes(N, std::max(m, n), h->num_sms));
    char* ews = take(svd_eig_bytes(N));
    double* Uv = reinterpret_cast<double*>(take(sizeof(double) * (size_t)N * 64));
    double* small = reinterpret_cast<double*>(take(sizeof(double) * (size_t)(N + 64 * 4 + 8)));
    double* eig = small;
    double* lam = eig + N;
    double* sv = lam + 64;
    double* inv = sv + 64;
    double* sgn = inv + 64;
    int* d_rank = reinterpret_cast<int*>(sgn + 64);
    double* C = nullptr;
    LAUNCH(h, launch_gram(X, m, n, n, gws, h->num_sms, &C, cs));
    LAUNCH(h, launch_svd_eig(C, (int)N, ews, tt_eps, rcap, eig, lam, d_rank, Uv, h->num_sms, cs));
    int rk = 1;
    CU(h, cudaMemcpyAsync(&rk, d_rank, sizeof(int), cudaMemcpyDeviceToHost, cs));
    CU(h, cudaStreamSynchronize(cs));
    const int r = std::max(1, std::min(rk, rcap));
    ranks_out[l - 1] = r;
    Xn = hb[(l - 1) & 1];
    float* core = dcores + coff;
    if (m <= n) {
      // core = U_r with the sign convention, X' = core^T X
      const int nS = bcd_spart_splits(m, n, h->num_sms);
      double* Spart = reinterpret_cast<double*>(take(sizeof(double) * (size_t)nS * n * r));
      LAUNCH(h, launch_sign_cols(Uv, m, r, nullptr, core, sgn, cs));
      LAUNCH(h, launch_bcd_spart(X, n, m, n, core, r, nS, Spart, cs));
      LAUNCH(h, launch_rows_from_spart(Spart, nS, n, r, Xn, cs));
    } else {
      // V_r = Uv (n x r): core = X V_r diag(1/s) with signs, X' = diag(sgn s) V_r^T
      const XhtPlan xp = plan_xht(m, n, h->num_sms);
      double* Ppart = reinterpret_cast<double*>(take(sizeof(double) * (size_t)xp.ncs * m * r));
      double* P = reinterpret_cast<double*>(take(sizeof(double) * (size_t)m * r));
      float* Vt = reinterpret_cast<float*>(take(sizeof(float) * (size_t)r * n));
      if (so > stepb) return fail(h, NTT_ERR_WORKSPACE, "internal: TT-SVD step scratch exceeded");
      LAUNCH(h, launch_sing(lam, r, sv, inv, cs));
      LAUNCH(h, launch_v_rows(Uv, n, r, nullptr, nullptr, Vt, cs));
      LAUNCH(h, launch_xht_partial(X, n, m, n, Vt, n, r, xp, Ppart, cs));
      LAUNCH(h, launch_sum_partials(Ppart, xp.ncs, m * r, P, cs));
      LAUNCH(h, launch_sign_cols(P, m, r, inv, core, sgn, cs));
      LAUNCH(h, launch_v_rows(Uv, n, r, sv, sgn, Xn, cs));
    }
    if (so > stepb) return fail(h, NTT_ERR_WORKSPACE, "internal: TT-SVD step scratch exceeded");
    coff += m * r;
    X = Xn;
    rprev = r;
  }
  h->cur_step = 0;
  const int64_t ncl = rprev * s0.dims[d - 1];
  CU(h, cudaMemcpyAsync(dcores + coff, Xn, sizeof(float) * (size_t)ncl, cudaMemcpyDeviceToDevice, cs));
  coff += ncl;
  if (coff > cores_capacity)
    return fail(h, NTT_ERR_WORKSPACE, "cores_capacity %lld < %lld floats for the chosen ranks",
                (long long)cores_capacity, (long long)coff);
  CU(h, cudaMemcpyAsync(cores, dcores, sizeof(float) * (size_t)coff, cudaMemcpyDefault, cs));
  CU(h, cudaStreamSynchronize(cs));
  if (rel_err) {
    TTShape s;
    if ((st = check_tt(h, d, dims, ranks_out, &s, true))) return st;
    if ((st = contract_stream(h, s, cores, nullptr, 0.0f, 0, A, rel_err))) return st;
  }
  return NTT_OK;
}

ntt_status ntt_rank_rule(ntt_handle h, const float* X, int64_t m, int64_t n, int64_t ldx, double tt_eps,
                         int32_t* rank, double* eig) {
  if (!h || !X || !rank) return NTT_ERR_INVALID_ARG;
  if (m < 1 || n < 1 || ldx < n) return fail(h, NTT_ERR_INVALID_ARG, "bad shape");
  if (!(tt_eps >= 0.0)) return fail(h, NTT_ERR_INVALID_ARG, "tt_eps must be >= 0");
  if (std::min(m, n) > kRankMaxN) return fail(h, NTT_ERR_UNSUPPORTED, "rank rule needs min(m, n) <= %d", kRankMaxN);
  if (!is_device_ptr(X)) return fail(h, NTT_ERR_INVALID_ARG, "X must be device memory");
  CU(h, cudaSetDevice(h->device));
  const int64_t N = std::min(m, n);
  const size_t rb = align_up(rank_rule_bytes(N, std::max(m, n), h->num_sms));
  ntt_status st = ensure_ws(h, rb + align_up(64) + align_up(sizeof(double) * (size_t)N));
  if (st) return st;
  char* ws = reinterpret_cast<char*>(h->ws);
  int* d_rank = reinterpret_cast<int*>(ws + rb);
  double* d_eig = reinterpret_cast<double*>(ws + rb + align_up(64));
  LAUNCH(h, launch_rank_rule(X, m, n, ldx, tt_eps, ws, h->num_sms, d_rank, d_eig, h->stream));
  int rk = 0;
  CU(h, cudaMemcpyAsync(&rk, d_rank, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  if (eig) CU(h, cudaMemcpyAsync(eig, d_eig, sizeof(double) * (size_t)N, cudaMemcpyDeviceToHost, h->stream));
  CU(h, cudaStreamSynchronize(h->stream));
  *rank = rk;
  return NTT_OK;
}

ntt_status ntt_reconstruct(ntt_handle h, int32_t d, const int64_t* dims, const int32_t* ranks, const float* cores,
                           float* out, const float* ref, double* rel_err) {
  if (!h) return NTT_ERR_INVALID_ARG;
  if (!cores) return fail(h, NTT_ERR_INVALID_ARG, "null cores");
  if (rel_err && !ref) return fail(h, NTT_ERR_INVALID_ARG, "rel_err needs ref");
  TTShape s;
  ntt_status st = check_tt(h, d, dims, ranks, &s, false);
  if (st) return st;
  CU(h, cudaSetDevice(h->device));
  return contract_stream(h, s, cores, out, 0.0f, 0, ref, rel_err);
}

ntt_status ntt_generate(ntt_handle h, int32_t d, const int64_t* dims, const int32_t* ranks, const float* cores,
                        float noise_amp, uint64_t seed, uint64_t noise_stream, float* out) {
  if (!h) return NTT_ERR_INVALID_ARG;
  if (!cores || !out) return fail(h, NTT_ERR_INVALID_ARG, "null cores or out");
  TTShape s;
  ntt_status st = check_tt(h, d, dims, ranks, &s, false);
  if (st) return st;
  CU(h, cudaSetDevice(h->device));
  return contract_stream(h, s, cores, out, noise_amp, rng_key(seed, noise_stream), nullptr, nullptr);
}

double ntt_compression_ratio(int32_t d, const int64_t* dims, const int32_t* ranks) {
  if (d < 1 || d > 64 || !dims || (d > 1 && !ranks)) return -1.0;
  double num = 1.0, den = 0.0;
  for (int i = 1; i <= d; ++i) {
    double rp = (i == 1) ? 1.0 : (double)ranks[i - 2];
    double rn = (i == d) ? 1.0 : (double)ranks[i - 1];
    if (dims[i - 1] < 1 || rp < 1 || rn < 1) return -1.0;
    num *= (double)dims[i - 1];
    den += (double)dims[i - 1] * rp * rn;
  }
  return num / den;
}

// ------------------------------------------------------------------- profiling
ntt_status ntt_profile_enable(ntt_handle h, int enable) {
  if (!h) return NTT_ERR_INVALID_ARG;
  CU(h, cudaStreamSynchronize(h->stream));
  if (h->gstream) CU(h, cudaStreamSynchronize(h->gstream));
  if (h->prof != (enable != 0)) {
    // the decompose graph records profile events only if captured with profiling on
    drop_graphs(h);
  }
  h->prof = enable != 0;
  h->ev_used = 0;
  h->recs.clear();
  for (auto& row : h->acc)
    for (auto& a : row) a = ntt_handle_s::Acc();
  return NTT_OK;
}

ntt_status ntt_profile_get(ntt_handle h, int cls, int64_t* launches, double* total_ms, double* total_bytes) {
  return ntt_profile_get_step(h, cls, -1, launches, total_ms, total_bytes);
}

ntt_status ntt_profile_get_step(ntt_handle h, int cls, int step, int64_t* launches, double* total_ms,
                                double* total_bytes) {
  if (!h || cls < 0 || cls >= NTT_PROF_CLASSES) return NTT_ERR_INVALID_ARG;
  CU(h, cudaStreamSynchronize(h->stream));
  prof_fold(h, h->recs, h->ev_pool);
  h->recs.clear();
  h->ev_used = 0;
  int64_t n = 0;
  double ms = 0.0, by = 0.0;
  for (int l = 0; l < 66; ++l) {
    if (step >= 0 && l != step) continue;
    n += h->acc[cls][l].n;
    ms += h->acc[cls][l].ms;
    by += h->acc[cls][l].bytes;
  }
  if (launches) *launches = n;
  if (total_ms) *total_ms = ms;
  if (total_bytes) *total_bytes = by;
  return NTT_OK;
}

// ------------------------------------------------------------------ distributed
int64_t ntt_dist_block(int64_t n_last, int nranks, int rank, int64_t* offset) {
  if (nranks < 1 || rank < 0 || rank >= nranks || n_last < 0) {
    if (offset) *offset = 0;
    return -1;
  }
  int64_t b0 = n_last * rank / nranks, b1 = n_last * (rank + 1) / nranks;
  if (offset) *offset = b0;
  return b1 - b0;
}

ntt_status ntt_get_unique_id(void* id128) {
  if (!id128) return NTT_ERR_INVALID_ARG;
  if (!load_nccl()) return NTT_ERR_UNSUPPORTED;
  ncclUniqueId id;
  if (g_nccl.GetUniqueId(&id) != ncclSuccess) return NTT_ERR_NCCL;
  memcpy(id128, &id, sizeof id);
  return NTT_OK;
}

// Exchange buffers of the persistent kernels' in-kernel cross-GPU reduction (PersistArgs::xpeers):
// every rank allocates xbuf_bytes(nranks), exports it with cudaIpcGetMemHandle, the handles are
// all-gathered by nranks ncclBroadcasts of 64 bytes, and every rank opens the others' buffers
// (NVLink peer access within one node).  The ranks then agree (ncclAllReduce of a 0/1 flag, min)
// so that either all of them run the in-kernel exchange or all keep the per-pass ncclAllReduce
// path (xready = false) -- a mixed outcome would deadlock the first pass.
static ntt_status setup_exchange(ntt_handle h) {
  const int p = h->nranks;
  const size_t bytes = xbuf_bytes(p);
  CU(h, cudaMalloc(&h->xbuf, bytes));
  CU(h, cudaMemset(h->xbuf, 0, bytes));
  std::vector<void*> bases(p, nullptr);
  bases[h->rank] = h->xbuf;
  bool ok = true;
  if (p > 1) {
    cudaIpcMemHandle_t mine;
    memset(&mine, 0, sizeof mine);
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    if (cudaIpcGetMemHandle(&mine, h->xbuf) != cudaSuccess) {
      ok = false;
      cudaGetLastError();
    }
    char* dh = nullptr;
    CU(h, cudaMalloc(&dh, 64 * (size_t)p));
    CU(h, cudaMemcpy(dh + 64 * (size_t)h->rank, &mine, 64, cudaMemcpyHostToDevice));
    for (int q = 0; q < p; ++q)
      NC(h, g_nccl.Broadcast(dh + 64 * (size_t)q, dh + 64 * (size_t)q, 64, ncclInt8, q, h->comm, h->stream));
    CU(h, cudaStreamSynchronize(h->stream));
    std::vector<cudaIpcMemHandle_t> all(p);
    CU(h, cudaMemcpy(all.data(), dh, 64 * (size_t)p, cudaMemcpyDeviceToHost));
    cudaFree(dh);
    for (int q = 0; q < p && ok; ++q) {
      if (q == h->rank) continue;
      if (cudaIpcOpenMemHandle(&bases[q], all[q], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        ok = false;
        cudaGetLastError();
        break;
      }
      h->xopened.push_back(bases[q]);
    }
    int* dflag = nullptr;
    CU(h, cudaMalloc(&dflag, sizeof(int)));
    const int mine_ok = ok ? 1 : 0;
    CU(h, cudaMemcpy(dflag, &mine_ok, sizeof(int), cudaMemcpyHostToDevice));
    NC(h, g_nccl.AllReduce(dflag, dflag, 1, ncclInt32, ncclMin, h->comm, h->stream));
    CU(h, cudaStreamSynchronize(h->stream));
    int all_ok = 0;
    CU(h, cudaMemcpy(&all_ok, dflag, sizeof(int), cudaMemcpyDeviceToHost));
    cudaFree(dflag);
    ok = all_ok == 1;
  }
  if (!ok) {  // every rank: per-pass ncclAllReduce path
    for (void* pp : h->xopened) cudaIpcCloseMemHandle(pp);
    h->xopened.clear();
    cudaFree(h->xbuf);
    h->xbuf = nullptr;
    h->xmode = 0;
    return NTT_OK;
  }
  CU(h, cudaMalloc(reinterpret_cast<void**>(&h->xpeers), sizeof(double*) * (size_t)p));
  CU(h, cudaMemcpy(h->xpeers, bases.data(), sizeof(double*) * (size_t)p, cudaMemcpyHostToDevice));
  h->xready = true;
  return NTT_OK;
}

ntt_status ntt_create_dist(ntt_handle* out, int device, void* cuda_stream, const void* id128, int nranks, int rank) {
  return ntt_create_dist_grid(out, device, cuda_stream, id128, nranks, rank, 1, nranks);
}

ntt_status ntt_create_dist_grid(ntt_handle* out, int device, void* cuda_stream, const void* id128, int nranks, int rank,
                                int pr, int pc) {
  if (!out || !id128 || nranks < 1 || rank < 0 || rank >= nranks) return NTT_ERR_INVALID_ARG;
  if (pr < 1 || pc < 1 || pr * pc != nranks) return NTT_ERR_INVALID_ARG;
  if (!load_nccl()) return NTT_ERR_UNSUPPORTED;
  ntt_status s = create_common(out, device, cuda_stream);
  if (s) return s;
  ntt_handle h = *out;
  ncclUniqueId id;
  memcpy(&id, id128, sizeof id);
  ncclResult_t r = g_nccl.CommInitRank(&h->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    delete h;
    *out = nullptr;
    return NTT_ERR_NCCL;
  }
  h->nranks = nranks;
  h->rank = rank;
  h->pr = pr;
  h->pc = pc;
  h->ga = rank / pc;
  h->gb = rank % pc;
  // row / column communicators (Alg. 5 / Alg. 6 groups)
  ncclResult_t r1 = g_nccl.CommSplit(h->comm, h->ga, h->gb, &h->comm_row, nullptr);
  ncclResult_t r2 = (r1 == ncclSuccess) ? g_nccl.CommSplit(h->comm, h->gb, h->ga, &h->comm_col, nullptr) : r1;
  if (r2 != ncclSuccess) {
    ntt_destroy(h);
    *out = nullptr;
    return NTT_ERR_NCCL;
  }
  if ((s = setup_exchange(h))) {
    ntt_destroy(h);
    *out = nullptr;
    return s;
  }
  return NTT_OK;
}

int ntt_dist_grid(ntt_handle h, int* pr, int* pc, int* ga, int* gb) {
  if (!h) return -1;
  if (pr) *pr = h->pr;
  if (pc) *pc = h->pc;
  if (ga) *ga = h->ga;
  if (gb) *gb = h->gb;
  return 0;
}

int ntt_dist_rank(ntt_handle h) { return h ? h->rank : -1; }
int ntt_dist_size(ntt_handle h) { return h ? h->nranks : -1; }

}  // extern "C"

extern "C" int64_t ntt_collective_count(ntt_handle h) { return h ? h->collectives : -1; }

extern "C" ntt_status ntt_set_dist_exchange(ntt_handle h, int mode) {
  if (!h || (mode != 0 && mode != 1)) return NTT_ERR_INVALID_ARG;
  if (!h->comm) return fail(h, NTT_ERR_INVALID_ARG, "ntt_set_dist_exchange needs an ntt_create_dist* handle");
  if (mode == 1 && !h->xready) return fail(h, NTT_ERR_UNSUPPORTED, "exchange buffers are not mapped");
  CU(h, cudaStreamSynchronize(h->stream));
  if (h->gstream) CU(h, cudaStreamSynchronize(h->gstream));
  drop_graphs(h);  // the decompose graph bakes in the path
  h->xmode = mode;
  return NTT_OK;
}

extern "C" int64_t ntt_peer_exchange_count(ntt_handle h) {
  if (!h || !h->xready) return -1;
  if (cudaStreamSynchronize(h->stream) != cudaSuccess) return -1;
  if (h->gstream && cudaStreamSynchronize(h->gstream) != cudaSuccess) return -1;
  unsigned long long v = 0;
  const char* seqp = reinterpret_cast<const char*>(h->xbuf) + xbuf_bytes(h->nranks) - sizeof(unsigned long long) * 8;
  if (cudaMemcpy(&v, seqp, sizeof v, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  return (int64_t)v;
}

extern "C" ntt_status ntt_stream_ceiling(ntt_handle h, const void* buf, int64_t bytes, int32_t reps, double* gbps) {
  if (!h || !buf || !gbps || bytes < 16 || (bytes & 15) || reps < 1 || (reinterpret_cast<uintptr_t>(buf) & 15))
    return NTT_ERR_INVALID_ARG;
  cudaPointerAttributes pa;
  if (cudaPointerGetAttributes(&pa, buf) != cudaSuccess || pa.type != cudaMemoryTypeDevice)
    return fail(h, NTT_ERR_INVALID_ARG, "ntt_stream_ceiling: buf must be device memory");
  float* sink = nullptr;
  CU(h, cudaMallocAsync(reinterpret_cast<void**>(&sink), 16, h->stream));
  cudaEvent_t e0, e1;
  CU(h, cudaEventCreate(&e0));
  CU(h, cudaEventCreate(&e1));
  LAUNCH(h, launch_read_stream(buf, bytes, sink, h->num_sms, h->stream));  // warm-up
  CU(h, cudaEventRecord(e0, h->stream));
  for (int i = 0; i < reps; ++i) LAUNCH(h, launch_read_stream(buf, bytes, sink, h->num_sms, h->stream));
  CU(h, cudaEventRecord(e1, h->stream));
  CU(h, cudaEventSynchronize(e1));
  float ms = 0.f;
  CU(h, cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  CU(h, cudaFreeAsync(sink, h->stream));
  *gbps = (double)bytes * reps / (ms * 1e-3) / 1e9;
  return NTT_OK;
}

extern "C" ntt_status ntt_debug_fill_uniform_cols(ntt_handle h, float* H, int32_t r, int64_t nloc, int64_t b,
                                                  int64_t nd, int64_t off, int64_t nglob, uint64_t seed,
                                                  uint64_t stream) {
  if (!h) return NTT_ERR_INVALID_ARG;
  if (!H || r < 1 || nloc < 0 || b < 1 || nd < b || off < 0 || off + b > nd || nloc % b || nglob < nloc ||
      !is_device_ptr(H))
    return fail(h, NTT_ERR_INVALID_ARG, "bad fill_uniform_cols layout");
  CU(h, cudaSetDevice(h->device));
  LAUNCH(h, launch_fill_uniform_cols(H, r, nloc, b, nd, off, nglob, seed, stream, h->stream));
  return NTT_OK;
}

extern "C" ntt_status ntt_debug_gather_last_core(ntt_handle h, const float* gath, int64_t r, int64_t nd,
                                                 int32_t nranks, float* core) {
  if (!h) return NTT_ERR_INVALID_ARG;
  if (!gath || !core || r < 1 || nd < nranks || nranks < 1 || !is_device_ptr(gath) || !is_device_ptr(core))
    return fail(h, NTT_ERR_INVALID_ARG, "bad gather_last_core arguments");
  CU(h, cudaSetDevice(h->device));
  LAUNCH(h, launch_gather_last_core(gath, r, nd, nranks, core, h->stream));
  return NTT_OK;
}

extern "C" ntt_status ntt_set_validation(ntt_handle h, int flags) {
  if (!h) return NTT_ERR_INVALID_ARG;
  if (flags & ~NTT_VALIDATE_NONNEG) return fail(h, NTT_ERR_INVALID_ARG, "unknown validation flags 0x%x", flags);
  h->validate = flags;
  return NTT_OK;
}

extern "C" ntt_status ntt_debug_bcd_force_correct(ntt_handle h, uint64_t mask) {
  if (!h) return NTT_ERR_INVALID_ARG;
  h->bcd_force = mask & ((1ull << 52) - 1);
  return NTT_OK;
}

extern "C" ntt_status ntt_prefetch_input(ntt_handle h, const float* src, int64_t count) {
  if (!h) return NTT_ERR_INVALID_ARG;
  if (!src || count < 1) return fail(h, NTT_ERR_INVALID_ARG, "null source or count < 1");
  if (is_device_ptr(src)) return fail(h, NTT_ERR_INVALID_ARG, "ntt_prefetch_input takes a host pointer");
  CU(h, cudaSetDevice(h->device));
  if (!h->cstream) {
    CU(h, cudaStreamCreateWithFlags(&h->cstream, cudaStreamNonBlocking));
    for (int q = 0; q < 2; ++q) {
      CU(h, cudaEventCreateWithFlags(&h->cev[q], cudaEventDisableTiming));
      CU(h, cudaEventCreateWithFlags(&h->uev[q], cudaEventDisableTiming));
    }
  }
  const int q = h->next_slot;
  const size_t bytes = sizeof(float) * (size_t)count;
  if (h->slot_cap[q] < bytes) {
    CU(h, cudaStreamSynchronize(h->cstream));
    CU(h, cudaStreamSynchronize(h->stream));
    if (h->gstream) CU(h, cudaStreamSynchronize(h->gstream));
    if (h->slot[q]) CU(h, cudaFree(h->slot[q]));
    h->slot[q] = nullptr;
    h->slot_cap[q] = 0;
    CU(h, cudaMalloc(&h->slot[q], bytes));
    h->slot_cap[q] = bytes;
  }
  // not before the last decompose that read this slot is done (a never-recorded event is no wait)
  CU(h, cudaStreamWaitEvent(h->cstream, h->uev[q], 0));
  CU(h, cudaMemcpyAsync(h->slot[q], src, bytes, cudaMemcpyHostToDevice, h->cstream));
  CU(h, cudaEventRecord(h->cev[q], h->cstream));
  h->slot_src[q] = src;
  h->slot_n[q] = count;
  h->slot_ready[q] = true;
  h->slot_seq[q] = ++h->fills;
  h->next_slot = q ^ 1;
  return NTT_OK;
}

extern "C" int32_t ntt_debug_mu_path(ntt_handle h, int64_t m, int64_t n, int32_t r) {
  if (!h || r < 1 || m < 1 || n < 1) return -1;
  const bool dist = h->comm != nullptr;
  const MuPlan p = plan_mu(m, n, r, h->num_sms, dist, h->xready && h->xmode == 1);
  if (p.tiny && !dist) return 1;
  if (p.clu && !dist) return 2;
  if (p.fused && p.persist && (!dist || (h->xready && h->xmode == 1))) return 3;
  if (p.fused) return 4;
  if (p.tc) return 5;
  return 6;
}

extern "C" const unsigned long long* ntt_debug_persist_trace(ntt_handle h) {
  if (!h) return nullptr;
  cudaStreamSynchronize(h->stream);
  return h->ptrace;
}
