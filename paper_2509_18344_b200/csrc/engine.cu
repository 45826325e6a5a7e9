// libsubspec engine: context, capped arena, placement, pinned host store, K7 layer streaming,
// draft loop (CUDA graph + PDL), verification, acceptance, and the C-ABI (include/subspec.h).
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>
#include <unistd.h>
#include <cuda.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges for nsys/ncu timelines (no link dependency)

#include "subspec.h"
#include "common.cuh"
#include "kernels.h"

using namespace ss;

namespace {

constexpr uint64_t kTidMul = 0xD1B54A32D192ED03ull;
uint64_t splitmix64_host(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
uint64_t tensor_key(uint64_t seed, uint64_t tid) { return splitmix64_host(seed ^ (tid * kTidMul)); }
float scale_c32(double sigma) { return float((sigma * std::sqrt(12.0)) / 262144.0); }

struct Arena {
  uint8_t* base = nullptr;
  size_t cap = 0, used = 0;
  void* alloc(size_t bytes, size_t align = 256) {
    size_t off = (used + align - 1) / align * align;
    if (off + bytes > cap) return nullptr;
    used = off + bytes;
    return base + off;
  }
};

struct LayerW {
  uint16_t* attn_norm = nullptr;
  uint16_t* mlp_norm = nullptr;
  uint16_t* bias = nullptr;
  bool resident = false;
  uint8_t* bf16[4] = {nullptr, nullptr, nullptr, nullptr};
  uint8_t* q4[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t host_off[4] = {0, 0, 0, 0};
  // K7 stream codec (zstream.cu): -1 plain bf16 (no header), 0 raw blob, 1 exponent-coded blob; the
  // bytes streamed per step and the offset of the raw bf16 data inside a blob
  int zmode[4] = {-1, -1, -1, -1};
  size_t host_used[4] = {0, 0, 0, 0};
  size_t host_a0[4] = {0, 0, 0, 0};
};

struct StreamItem {
  int64_t seq;
  int layer, group;
  size_t off, bytes;
  int ev;
  bool consumed;
};

enum State { ST_CREATED = 0, ST_LOADED = 1, ST_READY = 2, ST_SESSION = 3, ST_DRAFTED = 4, ST_VERIFIED = 5 };

}  // namespace

struct ss_ctx {
  ss_model_config cfg{};
  ss_limits lim{};
  int device = 0;
  cudaStream_t cs = nullptr, xs = nullptr;
  Arena ar;
  std::string err;
  bool poisoned = false;
  int state = ST_CREATED;
  int H = 0, F = 0, qd = 0, kvd = 0, qkv_rows = 0, L = 0, V = 0, d = 0, nh = 0, nkv = 0, C = 0;
  int gN[4] = {0}, gK[4] = {0};
  // weights
  uint16_t* embed = nullptr;
  uint16_t* h_embed = nullptr;   // embedding in mapped pinned host memory (zero-copy row gather)
  uint8_t* head = nullptr;
  uint16_t* final_norm = nullptr;
  std::vector<LayerW> lw;
  int n_resident = 0;
  uint64_t seed = 0;
  uint8_t* host = nullptr;
  bool host_external = false;   // caller-owned store (ss_load_weights_shared), registered here
  size_t host_bytes = 0;
  bool substitutes_built = false;
  // kv + tree
  uint16_t *kc = nullptr, *vc = nullptr, *kt = nullptr, *vt = nullptr;
  int64_t kc_layer = 0, kt_layer = 0;
  uint16_t *kcd = nullptr, *vcd = nullptr, *ktd = nullptr, *vtd = nullptr;   // NEXT-4 separate draft KV (else null)
  int max_nodes = 0, anc_stride = 0;
  int *tok = nullptr, *parent = nullptr, *depth = nullptr, *anc = nullptr;
  float* score = nullptr;
  int *committed_len = nullptr, *root_tok = nullptr, *tokbuf = nullptr;
  int P = 0, n_nodes = 0, cur_k = 0, cur_deff = 0;
  // batched requests (NEXT-2): slots [0, B) of Bmax; per-slot tree arrays of max_nodes and committed
  // KV of C rows, so the kv-head strides of the KV buffers are kv_nodes = Bmax*max_nodes, kv_ctx = Bmax*C
  int Bmax = 1, B = 1, kv_nodes = 0, kv_ctx = 0;
  std::vector<int> Pb;                 // committed length per slot (host mirror)
  std::vector<char> slot_ready;        // slot prefilled in this batch session
  ReqMap cur_rq{0, 0, 0, 0};           // request map of the pass being enqueued
  // activations
  float* x = nullptr;
  uint16_t *hfrag = nullptr, *attnfrag = nullptr, *actfrag = nullptr, *qbuf = nullptr;
  float *hxs = nullptr, *attnxs = nullptr, *actxs = nullptr;   // group sums of the FragX inputs
  float* logits = nullptr;
  unsigned long long* tracebuf = nullptr;   // debug: %globaltimer events [512][kTraceEvents]
  int mpad_max = 0;
  float2* rope = nullptr;
  // gemv scratch
  float* gv_part = nullptr;
  int* gv_cnt = nullptr;
  int gv_grid = 148;
  size_t gv_part_floats = 0;
  // attention scratch
  float* at_o = nullptr;        // debug output scratch (ss_debug_matmul / ss_debug_time_matmul)
  void* dbg_mem = nullptr;      // at_o (+ logits outside fp32 mode): debug-only, outside the arena
  size_t at_o_floats = 0;
  // topk scratch
  float *tk_max = nullptr, *tk_sum = nullptr, *tk_val = nullptr;
  int* tk_idx = nullptr;
  // verify
  float *am_val = nullptr, *am_sec = nullptr, *gap = nullptr;
  int *am_idx = nullptr, *argmax = nullptr;
  int vtiles = 0;
  // accept
  int *out_tokens = nullptr, *out_n = nullptr, *out_path = nullptr, *commit_meta = nullptr;
  int* h_out = nullptr;   // pinned: [0] n, [1..] tokens
  // streaming ring (K7)
  uint8_t* ring = nullptr;
  size_t ring_bytes = 0, ring_head = 0;
  std::deque<StreamItem> inflight;
  int64_t next_issue = 0, next_consume = 0;
  // ss_debug_step_timeline: extra timing events per streamed item while on (seq -> copy start/end on
  // the copy stream, compute start (after the copy wait) / end (ring release) on the compute stream)
  bool tl_on = false;
  std::map<int64_t, std::array<cudaEvent_t, 4>> tl_ev;
  std::vector<std::pair<int, int>> cycle;
  std::vector<cudaEvent_t> ev_copied, ev_consumed, ev_t0, ev_t1;
  std::vector<bool> ev_pending;
  std::deque<int> timing_queue;
  int ev_pool = 0;
  int sub_bits = 4;           // substitute code bits (ss_set_substitute_bits; 2 = NEXT-3)
  ss_options opt{};           // per-context options (ss_create)
  bool l2_prefetch = false;
  float* sumsq = nullptr;     // fused RMSNorm: per-tile sums of squares [H/128][32]
  unsigned long long* norm_ctr = nullptr;
  int* h_root = nullptr;      // pinned staging word for draft_tree's root token
  bool serial_stream = false; // ablation: no copy/compute overlap in the verify streaming
  int last_consumed_ev = -1;
  cudaEvent_t ev_root = nullptr;
  bool fuse_norm = true;
  int k6_variant = 0;         // K6 kernel variant (ss_debug_set_knob 2; launch_gemm; A/B only)
  bool zcomp = false;         // ss_options.compress_stream (bf16 mode): the host store holds coded blobs
  uint16_t* dbuf = nullptr;   // decoded bf16 row tiles of the group being verified (K6 reads them)
  size_t dbuf_bytes = 0;      // decode buffer: >= one row tile of every group; a group decodes and
                              // runs K6 in row blocks of <= dbuf_bytes (the rest of the cap feeds the ring)
  // NEXT-1 cooperative streaming (ss_coop_*): rank r of `coop_world` copies slice r of every streamed
  // group from its host store and pushes it into every peer's ring at the same offset; flags[h] =
  // "rank h's slice of item seq landed here" (= seq + 1), flags[kCoopMax + h] = "rank h consumed
  // items < value" (both monotonic, written by the peers' streams)
  int coop_world = 1, coop_rank = 0;
  bool coop_exported = false;
  uint32_t* flags = nullptr;
  std::vector<uint8_t*> peer_ring;
  std::vector<uint32_t*> peer_flags;
  std::vector<void*> ipc_opened;
  std::deque<std::tuple<size_t, size_t, int64_t>> placed;   // ring occupancy (off, bytes, seq)
  // graphs
  std::map<std::tuple<int, int, uint32_t>, cudaGraphExec_t> graphs;
  std::map<std::tuple<int, int, uint32_t>, int64_t> graph_launches;
  bool use_graphs = true, use_pdl = true;
  // SS_FP32 precision mode (f32.cu): fp32 activations, q, attention output, KV cache, logits
  bool f32 = false;
  int kv_es = 2;                         // bytes per K/V element (2 bf16, 4 fp32)
  float *h32 = nullptr, *q32 = nullptr, *o32 = nullptr, *y32 = nullptr, *a32 = nullptr, *logits32 = nullptr;
  uint8_t* host_dev = nullptr;           // fp32 mode: device-mapped view of the pinned host store
  // stats
  ss_stats st{};
  cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr, e3 = nullptr;
  // copy-busy accounting: every copy interval is clipped to start no earlier than the last
  // ss_reset_stats (ev_region), all times measured from ev_ref (recorded once at creation)
  cudaEvent_t ev_ref = nullptr, ev_region = nullptr;
  bool region_set = false;
  int64_t launches = 0;
  bool capturing = false;
};

// ------------------------------------------------------------------------------------------
namespace {

ss_status fail(ss_ctx* c, ss_status s, const std::string& msg) {
  if (c) {
    c->err = msg;
    if (s == SS_ERR_CUDA) c->poisoned = true;
  }
  return s;
}

#define CK(call)                                                                               \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess) return fail(c, SS_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

ss_status check_launch(ss_ctx* c, const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(c, SS_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return SS_OK;
}

size_t sub_bytes(int N, int K, int bits) { return size_t(N / 128) * (K / 128) * size_t(qtile_bytes(bits)); }
size_t bf16_bytes(int N, int K) { return size_t(N) * K * 2; }

// token groups of 8 for a draft GEMV over M <= 32 rows: the tcgen05 MMA's N is 16 or 32 (M = 128)
int gemv_nt(int M) { return M <= 16 ? 2 : 4; }
int gemm_nt(int M) { return ((M + 127) / 128) * 16; }

// busy ms of copy slot ev, clipped to the current stats region
static float copy_busy_ms(ss_ctx* c, int ev) {
  float a = 0.f, b = 0.f, r = 0.f;
  if (cudaEventElapsedTime(&a, c->ev_ref, c->ev_t0[ev]) != cudaSuccess ||
      cudaEventElapsedTime(&b, c->ev_ref, c->ev_t1[ev]) != cudaSuccess) {
    cudaGetLastError();
    return 0.f;
  }
  if (c->region_set && cudaEventElapsedTime(&r, c->ev_ref, c->ev_region) == cudaSuccess) a = std::max(a, r);
  cudaGetLastError();
  return std::max(0.f, b - a);
}

// ---------------------------------- K7 streaming ------------------------------------------
// Stream memory operations (driver API, fetched at run time: no libcuda link dependency)
namespace {
constexpr int kCoopMax = 64;
typedef CUresult (*PFN_wait32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_write32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_range)(CUdeviceptr*, size_t*, CUdeviceptr);
PFN_wait32 g_wait32 = nullptr;
PFN_write32 g_write32 = nullptr;
PFN_range g_range = nullptr;
bool load_driver_fns() {
  static std::once_flag once;
  static bool ok = false;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    ok = cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", (void**)&g_wait32, 12000, cudaEnableDefault, &q) == cudaSuccess &&
         q == cudaDriverEntryPointSuccess &&
         cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", (void**)&g_write32, 12000, cudaEnableDefault, &q) == cudaSuccess &&
         q == cudaDriverEntryPointSuccess &&
         cudaGetDriverEntryPointByVersion("cuMemGetAddressRange", (void**)&g_range, 12000, cudaEnableDefault, &q) == cudaSuccess &&
         q == cudaDriverEntryPointSuccess;
    cudaGetLastError();
  });
  return ok;
}
}  // namespace
#define CKD(x)                                                                         \
  do {                                                                                 \
    CUresult r_ = (x);                                                                 \
    if (r_ != CUDA_SUCCESS) return fail(c, SS_ERR_CUDA, std::string("driver: ") + #x); \
  } while (0)
static size_t coop_slice_lo(size_t B, int h, int G) { return h >= G ? B : (B * size_t(h) / size_t(G)) & ~size_t(4095); }

static void tl_record(ss_ctx* c, int64_t seq, int k, cudaStream_t st) {
  auto it = c->tl_ev.find(seq);
  if (it == c->tl_ev.end()) it = c->tl_ev.emplace(seq, std::array<cudaEvent_t, 4>{}).first;
  if (!it->second[k] && cudaEventCreate(&it->second[k]) != cudaSuccess) {
    cudaGetLastError();
    it->second[k] = nullptr;
    return;
  }
  cudaEventRecord(it->second[k], st);
}

ss_status pump(ss_ctx* c) {
  if (c->cycle.empty()) return SS_OK;
  const int n_items = int(c->cycle.size());
  while (true) {
    const int64_t seq = c->next_issue;
    // never run more than one cycle ahead of consumption
    if (seq >= c->next_consume + n_items) return SS_OK;
    // ablation (ss_options.async_stream = 0, the paper's "async transfer" off, P:172-176 / Table 2): copy a
    // group only when it is the next one consumed and after the previous group's compute
    if (c->serial_stream && seq > c->next_consume) return SS_OK;
    const auto [l, g] = c->cycle[seq % n_items];
    const size_t B = c->lw[l].host_used[g];   // the group's host-store bytes (a codec blob or plain bf16)
    size_t off = c->ring_head;
    if (off + B > c->ring_bytes) off = 0;
    const int ev = int(seq % c->ev_pool);
    for (size_t i = 0; i < c->inflight.size(); ++i)
      if (c->inflight[i].ev == ev) {   // event slot still owned by an old item
        if (!c->inflight[i].consumed) return SS_OK;
        // consumed long ago (the pool is 4 cycles deep): order the copy stream after it and drop it
        CK(cudaStreamWaitEvent(c->xs, c->ev_consumed[ev], 0));
        c->inflight.erase(c->inflight.begin() + i);
        break;
      }
    // regions of older items that the new copy overwrites must have been consumed
    std::vector<size_t> dead;
    for (size_t i = 0; i < c->inflight.size(); ++i) {
      const auto& it = c->inflight[i];
      const bool overlap = it.off < off + B && off < it.off + it.bytes;
      if (overlap) {
        if (!it.consumed) return SS_OK;
        dead.push_back(i);
      }
    }
    if (c->ev_pending[ev]) {   // timing of a previous copy with this slot not yet harvested
      CK(cudaEventSynchronize(c->ev_t1[ev]));
      c->st.stream_busy_ms += copy_busy_ms(c, ev);
      c->ev_pending[ev] = false;
    }
    for (size_t i : dead) CK(cudaStreamWaitEvent(c->xs, c->ev_consumed[c->inflight[i].ev], 0));
    if (c->serial_stream && c->last_consumed_ev >= 0) CK(cudaStreamWaitEvent(c->xs, c->ev_consumed[c->last_consumed_ev], 0));
    for (size_t k = dead.size(); k-- > 0;) c->inflight.erase(c->inflight.begin() + dead[k]);
    CK(cudaEventRecord(c->ev_t0[ev], c->xs));
    if (c->tl_on) tl_record(c, seq, 0, c->xs);
    if (c->coop_world > 1) {
      // NEXT-1: the items that occupied [off, off + B) before must have been consumed by every peer
      int64_t need = 0;
      for (auto it = c->placed.begin(); it != c->placed.end();) {
        if (std::get<0>(*it) < off + B && off < std::get<0>(*it) + std::get<1>(*it)) {
          need = std::max(need, std::get<2>(*it) + 1);
          it = c->placed.erase(it);
        } else {
          ++it;
        }
      }
      c->placed.emplace_back(off, B, seq);
      const int G = c->coop_world, me = c->coop_rank;
      const size_t lo = coop_slice_lo(B, me, G), hi = coop_slice_lo(B, me + 1, G);
      if (hi > lo)
        CK(cudaMemcpyAsync(c->ring + off + lo, c->host + c->lw[l].host_off[g] + lo, hi - lo, cudaMemcpyHostToDevice, c->xs));
      for (int h = 0; h < G; ++h) {
        if (h == me) continue;
        if (need > 0) CKD(g_wait32((CUstream)c->xs, (CUdeviceptr)(c->flags + kCoopMax + h), cuuint32_t(need), CU_STREAM_WAIT_VALUE_GEQ));
        if (hi > lo) CK(cudaMemcpyAsync(c->peer_ring[h] + off + lo, c->ring + off + lo, hi - lo, cudaMemcpyDeviceToDevice, c->xs));
      }
      for (int h = 0; h < G; ++h)   // my slice of item seq is in every ring
        CKD(g_write32((CUstream)c->xs, (CUdeviceptr)(c->peer_flags[h] + me), cuuint32_t(seq + 1), 0));
      c->st.stream_bytes += double(hi - lo);
      c->st.stream_raw_bytes += double(bf16_bytes(c->gN[g], c->gK[g]));
      c->st.peer_bytes += double(hi - lo) * (G - 1);
    } else {
      CK(cudaMemcpyAsync(c->ring + off, c->host + c->lw[l].host_off[g], B, cudaMemcpyHostToDevice, c->xs));
      c->st.stream_bytes += double(B);
      c->st.stream_raw_bytes += double(bf16_bytes(c->gN[g], c->gK[g]));
    }
    CK(cudaEventRecord(c->ev_t1[ev], c->xs));
    if (c->tl_on) tl_record(c, seq, 1, c->xs);
    CK(cudaEventRecord(c->ev_copied[ev], c->xs));
    c->ev_pending[ev] = true;
    c->timing_queue.push_back(ev);
    c->inflight.push_back({seq, l, g, off, B, ev, false});
    c->ring_head = off + B;
    c->next_issue = seq + 1;
  }
}

void harvest_timing(ss_ctx* c) {
  while (!c->timing_queue.empty()) {
    const int ev = c->timing_queue.front();
    if (!c->ev_pending[ev]) {
      c->timing_queue.pop_front();
      continue;
    }
    if (cudaEventQuery(c->ev_t1[ev]) != cudaSuccess) break;
    c->st.stream_busy_ms += copy_busy_ms(c, ev);
    c->ev_pending[ev] = false;
    c->timing_queue.pop_front();
  }
  cudaGetLastError();
}

// returns the staged weights of the next item in the cycle (must be (l, g)); compute waits on its copy
ss_status consume_begin(ss_ctx* c, int l, int g, const uint8_t** w, int* ev_out) {
  ss_status s = pump(c);
  if (s != SS_OK) return s;
  const int64_t seq = c->next_consume;
  const int n_items = int(c->cycle.size());
  if (c->cycle[seq % n_items] != std::make_pair(l, g)) return fail(c, SS_ERR_STRUCTURE, "stream order mismatch");
  for (auto& it : c->inflight)
    if (it.seq == seq) {
      CK(cudaStreamWaitEvent(c->cs, c->ev_copied[it.ev], 0));
      for (int h = 0; h < c->coop_world && c->coop_world > 1; ++h)   // every rank's slice landed
        if (h != c->coop_rank)
          CKD(g_wait32((CUstream)c->cs, (CUdeviceptr)(c->flags + h), cuuint32_t(seq + 1), CU_STREAM_WAIT_VALUE_GEQ));
      *w = c->ring + it.off;
      *ev_out = it.ev;
      if (c->tl_on) tl_record(c, seq, 2, c->cs);
      return SS_OK;
    }
  return fail(c, SS_ERR_BUDGET, "staging ring cannot hold the next layer group");
}
ss_status consume_end(ss_ctx* c, int ev) {
  if (c->tl_on) tl_record(c, c->next_consume, 3, c->cs);
  CK(cudaEventRecord(c->ev_consumed[ev], c->cs));
  for (int h = 0; h < c->coop_world && c->coop_world > 1; ++h)   // tell every peer: item consumed here
    if (h != c->coop_rank)
      CKD(g_write32((CUstream)c->cs, (CUdeviceptr)(c->peer_flags[h] + kCoopMax + c->coop_rank),
                    cuuint32_t(c->next_consume + 1), 0));
  c->last_consumed_ev = ev;
  for (auto& it : c->inflight)
    if (it.ev == ev) it.consumed = true;
  c->next_consume++;
  return pump(c);
}

// ----------------------------------- passes -------------------------------------------------
struct PassOut {
  bool logits = false;        // draft: logits to c->logits [M x V]
  bool argmax = false;        // target: per-node argmax + gap
  bool topk = false;          // draft: per vocab-tile top-k statistics (EPI_TOPK), no logits in HBM
  int tk_k = 0;
  float tk_inv_t = 1.f;
};
// debug timing only (ss_debug_time_pass): skip kernel classes to attribute pass time
int g_skip = 0;
unsigned long long* g_trace = nullptr;   // device buffer [launch][kTraceEvents] for ss_debug_trace_pass
int g_trace_n = 0, g_trace_cap = 0;
unsigned long long* g_cta_trace = nullptr;   // per-CTA trace of GEMV launch number g_cta_launch
int g_cta_launch = -1, g_gemv_n = 0;
enum { SKIP_ATTN = 1, SKIP_NORM = 2, SKIP_GEMV = 4, SKIP_HEAD = 8 };

// the draft's weight stream in pass order: qkv, o, gate_up, down of each layer, then the head
static void next_weights(ss_ctx* c, int l, int g, const uint8_t** ptr, int64_t* bytes) {
  int nl = l, ng = g + 1;
  if (ng == 4) {
    ng = 0;
    ++nl;
  }
  if (nl >= c->L) {   // after the last layer: the head (prefetch its first part only)
    *ptr = c->head;
    *bytes = std::min<int64_t>(int64_t(64) << 20, int64_t(bf16_bytes(c->V, c->H)));
    return;
  }
  const LayerW& w = c->lw[nl];
  *ptr = w.resident ? w.bf16[ng] : w.q4[ng];
  *bytes = int64_t(w.resident ? bf16_bytes(c->gN[ng], c->gK[ng]) : sub_bytes(c->gN[ng], c->gK[ng], c->sub_bits));
  if (ng == 0) {   // qkv is small: let it cover o as well (two kernels ahead)
    const uint8_t* p2 = w.resident ? w.bf16[1] : w.q4[1];
    if (p2 == *ptr + *bytes) *bytes += int64_t(w.resident ? bf16_bytes(c->gN[1], c->gK[1]) : sub_bytes(c->gN[1], c->gK[1], c->sub_bits));
  }
}

ss_status matmul(ss_ctx* c, bool target, int l, int g, const uint16_t* X, int M, const EpiParams& epi) {
  if (!target && (g_skip & SKIP_GEMV)) return SS_OK;
  const int N = c->gN[g], K = c->gK[g];
  const LayerW& w = c->lw[l];
  if (!target) {
    GemvParams p{};
    p.W = w.resident ? w.bf16[g] : w.q4[g];
    p.X = X;
    p.XS = X == c->hfrag ? c->hxs : (X == c->attnfrag ? c->attnxs : c->actxs);
    p.N = N;
    p.K = K;
    p.NT = gemv_nt(M);
    p.partials = c->gv_part;
    p.counters = c->gv_cnt;
    p.max_seg = gemv_max_segments(N, K, gemv_streamk_grid(!w.resident, N, K, c->gv_grid));
    p.epi = epi;
    if (c->l2_prefetch) next_weights(c, l, g, &p.pf, &p.pf_bytes);
    // qkv substitutes: planned at one CTA per SM (the 16-warp K2 plans one CTA per SM for every group;
    // the hint matters for the 8-warp build, SS_K2_CW = 8, whose default is two per SM)
    p.ctas_per_sm = (g == 0 && !w.resident) ? 1 : 0;
    p.qbits = c->sub_bits;
    if (g_trace && g_trace_n < g_trace_cap) p.trace = g_trace + kTraceEvents * (g_trace_n++);
    if (g_cta_trace && g_gemv_n++ == g_cta_launch) p.cta_trace = g_cta_trace;
    launch_gemv(!w.resident, p, c->gv_grid, c->use_pdl, c->cs);
    c->launches++;
    return check_launch(c, "gemv");
  }
  GemmParams p{};
  p.X = X;
  p.N = N;
  p.K = K;
  p.NT = gemm_nt(M);
  p.epi = epi;
  if (w.resident) {
    p.W = w.bf16[g];
    launch_gemm(p, c->use_pdl, c->cs, c->k6_variant);
    c->launches++;
    return check_launch(c, "gemm");
  }
  const uint8_t* wp = nullptr;
  int ev = -1;
  ss_status s = consume_begin(c, l, g, &wp, &ev);
  if (s != SS_OK) return s;
  if (w.zmode[g] == 1) {
    // K7 codec: decode the streamed blob into bf16 row tiles and run K6 on them, in row blocks of at
    // most dbuf_bytes (a row block is a contiguous chunk range of the blob); the ring region is released
    // after the last block's decode.  Every block keeps the whole matrix's K-split plan (split_n), so
    // the products are bitwise those of one launch over the matrix.
    const int nC = K / 128, tiles = N / 128;
    const int per_max = std::max<int>(1, int(c->dbuf_bytes / (size_t(nC) * kBF16TileBytes)));
    const int parts = (tiles + per_max - 1) / per_max, per = (tiles + parts - 1) / parts;
    for (int t0 = 0; t0 < tiles; t0 += per) {
      const int nt = std::min(per, tiles - t0);
      launch_zdecode_range(wp, c->dbuf, t0 * nC, nt * nC, c->cs);
      c->launches++;
      if ((s = check_launch(c, "zdecode")) != SS_OK) return s;
      if (t0 + nt == tiles && (s = consume_end(c, ev)) != SS_OK) return s;
      GemmParams q = p;
      q.W = reinterpret_cast<const uint8_t*>(c->dbuf);
      q.N = nt * 128;
      q.tile0 = t0;
      q.split_n = N;
      launch_gemm(q, false, c->cs, c->k6_variant);
      c->launches++;
      if ((s = check_launch(c, "gemm")) != SS_OK) return s;
    }
    return SS_OK;
  }
  p.W = wp + w.host_a0[g];
  launch_gemm(p, false, c->cs, c->k6_variant);   // follows a cross-stream event wait: plain serialisation
  c->launches++;
  s = check_launch(c, "gemm");
  if (s != SS_OK) return s;
  return consume_end(c, ev);
}

EpiParams base_epi(ss_ctx* c, int M) {
  EpiParams e{};
  e.M = M;
  e.committed_len = c->committed_len;
  e.depth = c->depth;
  e.rope = c->rope;
  e.q_dim = c->qd;
  e.kv_dim = c->kvd;
  e.head_dim = c->d;
  e.max_nodes = c->kv_nodes;
  e.rq = c->cur_rq;
  e.x = c->x;
  e.ldx = c->H;
  e.ffn = c->F;
  return e;
}

// SS_FP32: the forward of M nodes in fp32 on the f32.cu kernels.  Weights: resident bf16; offloaded
// layers: the draft's substitutes (4/2-bit tiles) and the target's bf16 tiles read in place from the
// device-mapped pinned host store (parity mode: no staging ring).  Output: draft logits -> c->logits,
// target logits -> c->logits32 (+ argmax/gap when out.argmax).
static const uint8_t* weights_f32(ss_ctx* c, bool target, int l, int g, int* fmt) {
  const LayerW& w = c->lw[l];
  if (w.resident) {
    *fmt = 0;
    return w.bf16[g];
  }
  if (!target) {
    *fmt = c->sub_bits;
    return w.q4[g];
  }
  *fmt = 0;
  return c->host_dev + w.host_off[g];
}

ss_status forward_pass_f32(ss_ctx* c, bool target, int M, int node_base, const PassOut& out) {
  const float eps = c->cfg.rms_eps;
  const int H = c->H, F = c->F;
  launch_rmsnorm_f32(c->tok, node_base, c->embed, c->x, M, H, c->lw[0].attn_norm, eps, c->h32, c->cs);
  float* kc = reinterpret_cast<float*>(c->kc);
  float* vc = reinterpret_cast<float*>(c->vc);
  float* kt = reinterpret_cast<float*>(c->kt);
  float* vt = reinterpret_cast<float*>(c->vt);
  for (int l = 0; l < c->L; ++l) {
    const LayerW& w = c->lw[l];
    if (l > 0) launch_rmsnorm_f32(nullptr, 0, nullptr, c->x, M, H, w.attn_norm, eps, c->h32, c->cs);
    int fmt = 0;
    const uint8_t* W = weights_f32(c, target, l, 0, &fmt);
    launch_linear_f32(c->h32, M, H, W, fmt, c->qkv_rows, c->y32, c->cs);
    launch_qkv_post_f32(c->y32, M, w.bias, c->qd, c->kvd, c->d, c->rope, c->committed_len, c->depth, node_base, c->q32,
                        kt + l * c->kt_layer, vt + l * c->kt_layer, c->kv_nodes, c->cs);
    launch_attention_f32(c->q32, kc + l * c->kc_layer, vc + l * c->kc_layer, kt + l * c->kt_layer, vt + l * c->kt_layer,
                         c->committed_len, c->anc, c->depth, c->anc_stride, c->kv_ctx, c->kv_nodes, node_base, M, c->nh,
                         c->nkv, c->d, c->o32, c->cs);
    W = weights_f32(c, target, l, 1, &fmt);
    launch_linear_f32(c->o32, M, c->qd, W, fmt, H, c->y32, c->cs);
    launch_add_f32(c->x, c->y32, int64_t(M) * H, c->cs);
    launch_rmsnorm_f32(nullptr, 0, nullptr, c->x, M, H, w.mlp_norm, eps, c->h32, c->cs);
    W = weights_f32(c, target, l, 2, &fmt);
    launch_linear_f32(c->h32, M, H, W, fmt, 2 * F, c->y32, c->cs);
    launch_silu_mul_f32(c->y32, M, F, c->a32, c->cs);
    W = weights_f32(c, target, l, 3, &fmt);
    launch_linear_f32(c->a32, M, F, W, fmt, H, c->y32, c->cs);
    launch_add_f32(c->x, c->y32, int64_t(M) * H, c->cs);
    c->launches += 10;
  }
  launch_rmsnorm_f32(nullptr, 0, nullptr, c->x, M, H, c->final_norm, eps, c->h32, c->cs);
  float* lg = target ? c->logits32 : c->logits;
  launch_linear_f32(c->h32, M, H, c->head, 0, c->V, lg, c->cs);
  c->launches += 3;
  if (out.argmax) {
    launch_argmax_f32(c->logits32, M, c->V, c->argmax, c->gap, c->cs);
    c->launches++;
  }
  return check_launch(c, "forward_f32");
}

// Forward M nodes [node_base, node_base + M) through the draft (GEMV path) or the target (GEMM
// path, streamed).  Tree slots of these nodes receive their K/V.
ss_status forward_pass(ss_ctx* c, bool target, int M, int node_base, const PassOut& out) {
  if (c->f32) return forward_pass_f32(c, target, M, node_base, out);
  const int NT = target ? gemm_nt(M) : gemv_nt(M);
  const float eps = c->cfg.rms_eps;
  ss_status s;
  launch_embed_rmsnorm(c->tok, node_base, M, c->embed, c->x, c->H, c->lw[0].attn_norm, eps, c->hfrag, c->hxs, NT,
                       c->use_pdl, c->cs, c->cur_rq);
  c->launches++;
  if ((s = check_launch(c, "embed_rmsnorm")) != SS_OK) return s;
  for (int l = 0; l < c->L; ++l) {
    EpiParams e = base_epi(c, M);
    e.kind = EPI_QKV;
    e.bias = c->lw[l].bias;
    e.q_out = c->qbuf;
    const bool own = !target && c->ktd;   // NEXT-4: the draft's own K/V (tree scratch and cache)
    e.k_tree = (own ? c->ktd : c->kt) + l * c->kt_layer;
    e.v_tree = (own ? c->vtd : c->vt) + l * c->kt_layer;
    e.node_base = node_base;
    if ((s = matmul(c, target, l, 0, c->hfrag, M, e)) != SS_OK) return s;
    AttnParams a{};
    a.q = c->qbuf;
    a.k_cache = (own ? c->kcd : c->kc) + l * c->kc_layer;
    a.v_cache = (own ? c->vcd : c->vc) + l * c->kc_layer;
    a.k_tree = e.k_tree;
    a.v_tree = e.v_tree;
    a.committed_len = c->committed_len;
    a.anc = c->anc;
    a.depth = c->depth;
    a.anc_stride = c->anc_stride;
    a.max_ctx = c->kv_ctx;
    a.max_nodes = c->kv_nodes;
    a.rq = c->cur_rq;
    a.n_q = M;
    a.node_base = node_base;
    a.n_heads = c->nh;
    a.n_kv = c->nkv;
    a.head_dim = c->d;
    a.out_fragx = c->attnfrag;
    a.out_xs = c->attnxs;
    a.out_nt = NT;
    if (g_trace && g_trace_n < g_trace_cap) a.trace = g_trace + kTraceEvents * (g_trace_n++);
    if (!(g_skip & SKIP_ATTN)) launch_attention(a, c->use_pdl, c->cs);
    c->launches++;
    if ((s = check_launch(c, "attention")) != SS_OK) return s;
    const bool fnorm = !target && c->fuse_norm && !(g_skip & SKIP_NORM) &&
                       gemv_tiles_all_resident(true, NT, c->gN[1], c->gK[1], c->gv_grid, c->sub_bits) &&
                       gemv_tiles_all_resident(true, NT, c->gN[3], c->gK[3], c->gv_grid, c->sub_bits) &&
                       (c->n_resident == 0 || (gemv_tiles_all_resident(false, NT, c->gN[1], c->gK[1], c->gv_grid) &&
                                               gemv_tiles_all_resident(false, NT, c->gN[3], c->gK[3], c->gv_grid)));
    // one monotonic barrier counter per (matrix, weight format, NT): every launch on a counter has
    // the same number of arrivals (tiles x cluster size), so generations stay aligned
    auto resid_norm = [&](const uint16_t* gain, int which) {
      EpiParams r = base_epi(c, M);
      r.kind = EPI_RESID_NORM;
      r.sumsq = c->sumsq;
      r.sumsq_ld = NT * 8;
      r.norm_gain = gain;
      r.norm_out = c->hfrag;
      r.norm_xs = c->hxs;
      r.norm_ctr = c->norm_ctr + (which * 2 + (c->lw[l].resident ? 1 : 0)) * 4 + (NT - 1);   // NT in 1..4
      r.n_tiles = c->H / 128;
      r.eps = eps;
      r.act_nt = NT;
      return r;
    };
    e = base_epi(c, M);
    e.kind = EPI_RESID;
    if (fnorm) e = resid_norm(c->lw[l].mlp_norm, 0);
    if ((s = matmul(c, target, l, 1, c->attnfrag, M, e)) != SS_OK) return s;
    if (!fnorm && !(g_skip & SKIP_NORM))
      launch_rmsnorm(c->x, M, c->H, c->lw[l].mlp_norm, eps, c->hfrag, c->hxs, NT, c->use_pdl, c->cs);
    c->launches += fnorm ? 0 : 1;
    if ((s = check_launch(c, "rmsnorm")) != SS_OK) return s;
    e = base_epi(c, M);
    e.kind = EPI_SILU;
    e.act = c->actfrag;
    e.act_xs = c->actxs;
    e.act_nt = NT;
    const uint16_t* nextg = (l + 1 < c->L) ? c->lw[l + 1].attn_norm : c->final_norm;
    if ((s = matmul(c, target, l, 2, c->hfrag, M, e)) != SS_OK) return s;
    e = base_epi(c, M);
    e.kind = EPI_RESID;
    if (fnorm) e = resid_norm(nextg, 1);
    if ((s = matmul(c, target, l, 3, c->actfrag, M, e)) != SS_OK) return s;
    if (fnorm) {
    } else if ((!target || out.argmax) && !(g_skip & SKIP_NORM)) {
      launch_rmsnorm(c->x, M, c->H, nextg, eps, c->hfrag, c->hxs, NT, c->use_pdl, c->cs);
      c->launches++;
      if ((s = check_launch(c, "rmsnorm")) != SS_OK) return s;
    } else if (l + 1 < c->L) {
      launch_rmsnorm(c->x, M, c->H, nextg, eps, c->hfrag, c->hxs, NT, c->use_pdl, c->cs);
      c->launches++;
      if ((s = check_launch(c, "rmsnorm")) != SS_OK) return s;
    }
  }
  if (out.argmax) {
    GemmParams p{};
    p.W = c->head;
    p.X = c->hfrag;
    p.N = c->V;
    p.K = c->H;
    p.NT = NT;
    p.epi = base_epi(c, M);
    p.epi.kind = EPI_ARGMAX;
    p.epi.am_val = c->am_val;
    p.epi.am_idx = c->am_idx;
    p.epi.am_second = c->am_sec;
    p.epi.am_tiles = c->vtiles;
    launch_gemm(p, c->use_pdl, c->cs, c->k6_variant);
    launch_argmax_merge(c->am_val, c->am_idx, c->am_sec, M, c->vtiles, c->argmax, c->gap, c->use_pdl, c->cs);
    c->launches += 2;
    return check_launch(c, "verify head");
  }
  if (out.logits || out.topk) {
    // head over the final normed rows (GEMV, <= 32 rows at a time); topk: the K5 statistics are
    // produced in the GEMV's epilogue and the logits never leave the SMs
    for (int r0 = 0; r0 < M && !target && !(g_skip & SKIP_HEAD); r0 += 32) {
      const int m = std::min(32, M - r0);
      GemvParams p{};
      p.W = c->head;
      p.X = c->hfrag;
      p.N = c->V;
      p.K = c->H;
      p.NT = gemv_nt(m);
      p.partials = c->gv_part;
      p.counters = c->gv_cnt;
      p.max_seg = gemv_max_segments(c->V, c->H, gemv_streamk_grid(false, c->V, c->H, c->gv_grid));
      p.epi = base_epi(c, m);
      p.epi.kind = EPI_LOGITS;
      p.epi.out = c->logits;
      p.epi.ldo = c->V;
      if (out.topk) {
        p.epi.kind = EPI_TOPK;
        p.epi.tk_max = c->tk_max;
        p.epi.tk_sum = c->tk_sum;
        p.epi.tk_val = c->tk_val;
        p.epi.tk_idx = c->tk_idx;
        p.epi.tk_k = out.tk_k;
        p.epi.tk_tiles = c->V / 128;
        p.epi.tk_inv_t = out.tk_inv_t;
      }
      launch_gemv(false, p, c->gv_grid, c->use_pdl, c->cs);
      c->launches++;
      if ((s = check_launch(c, "head gemv")) != SS_OK) return s;
    }
  }
  return SS_OK;
}

// request map of a pass over `rows` rows per request of all B slots (zero map for one request)
static ReqMap batch_map(ss_ctx* c, int rows) {
  return c->B > 1 ? ReqMap{rows, 0, c->max_nodes, c->C} : ReqMap{0, 0, 0, 0};
}

ss_status draft_loop(ss_ctx* c, int D, int k, float T) {
  ss_status s;
  launch_tree_init(c->root_tok, c->tok, c->parent, c->depth, c->score, c->anc, c->use_pdl, c->cs, c->B, c->max_nodes,
                   c->anc_stride);
  c->launches++;
  if ((s = check_launch(c, "tree_init")) != SS_OK) return s;
  for (int dd = 0; dd < D; ++dd) {
    const int Mr = dd == 0 ? 1 : k;   // frontier rows per request
    const int M = c->B * Mr;
    const int base = dd == 0 ? 0 : 1 + (dd - 1) * k;
    PassOut o;
    // bf16: the head GEMV's epilogue produces the per-tile top-k statistics (K5 folded);
    // fp32 parity mode: logits, then the two-stage top-k kernels
    o.topk = !c->f32;
    o.logits = c->f32;
    o.tk_k = k;
    o.tk_inv_t = float(1.0 / double(T));
    c->cur_rq = batch_map(c, Mr);
    s = forward_pass(c, false, M, base, o);
    c->cur_rq = ReqMap{0, 0, 0, 0};
    if (s != SS_OK) return s;
    TopkParams t{};
    t.req_rows = c->B > 1 ? Mr : 0;
    t.node_stride = c->max_nodes;
    t.logits = c->logits;
    t.M = M;
    t.V = c->V;
    t.k = k;
    t.inv_t = float(1.0 / double(T));
    t.blocks_per_row = std::max(1, std::min(64, 296 / M));
    t.blk_max = c->tk_max;
    t.blk_sum = c->tk_sum;
    t.blk_val = c->tk_val;
    t.blk_idx = c->tk_idx;
    t.tok = c->tok;
    t.parent = c->parent;
    t.depth = c->depth;
    t.score = c->score;
    t.anc = c->anc;
    t.anc_stride = c->anc_stride;
    t.node_base = base;
    t.child_base = 1 + dd * k;
    t.child_depth = dd + 1;
    if (o.topk) {
      t.blocks_per_row = c->V / 128;
      launch_topk_select(t, c->use_pdl, c->cs);
      c->launches += 1;
    } else {
      launch_topk(t, c->use_pdl, c->cs);
      c->launches += 2;
    }
    if ((s = check_launch(c, "topk")) != SS_OK) return s;
  }
  if (c->ktd) {
    // NEXT-4 separate draft KV: the depth-D nodes (the root when D = 0) are never a draft frontier; one
    // KV-only pass (no head) gives every tree node its draft K/V, so whatever path is accepted can be
    // committed to the draft's cache
    s = forward_pass(c, false, D > 0 ? k : 1, D > 0 ? 1 + (D - 1) * k : 0, PassOut{});
    if (s != SS_OK) return s;
  }
  return SS_OK;
}

ss_status run_draft(ss_ctx* c, int D, int k, float T) {
  uint32_t tb;
  std::memcpy(&tb, &T, 4);
  const auto key = std::make_tuple(D + (c->B << 16), k, tb);   // one graph per (D, batch, k, T)
  if (c->use_graphs) {
    auto it = c->graphs.find(key);
    if (it == c->graphs.end()) {
      // first use: run eagerly (sets kernel attributes), then capture for later steps
      const int64_t l0 = c->launches;
      ss_status s = draft_loop(c, D, k, T);
      if (s != SS_OK) return s;
      const int64_t nl = c->launches - l0;
      cudaGraph_t g = nullptr;
      if (cudaStreamBeginCapture(c->cs, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
        c->capturing = true;
        const int64_t lsave = c->launches;
        ss_status s2 = draft_loop(c, D, k, T);
        c->launches = lsave;
        c->capturing = false;
        cudaError_t e = cudaStreamEndCapture(c->cs, &g);
        cudaGraphExec_t ge = nullptr;
        if (s2 == SS_OK && e == cudaSuccess && cudaGraphInstantiate(&ge, g, 0) == cudaSuccess) {
          c->graphs[key] = ge;
          c->graph_launches[key] = nl;
        } else {
          c->use_graphs = false;
        }
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        c->poisoned = false;
        c->err.clear();
      } else {
        cudaGetLastError();
        c->use_graphs = false;
      }
      return SS_OK;
    }
    CK(cudaGraphLaunch(it->second, c->cs));
    c->launches += c->graph_launches[key];
    return SS_OK;
  }
  return draft_loop(c, D, k, T);
}

ss_status do_verify(ss_ctx* c) {
  PassOut o;
  o.argmax = true;
  c->cur_rq = batch_map(c, c->n_nodes);   // rows request-major: request b's nodes at b * n_nodes
  ss_status s = forward_pass(c, true, c->B * c->n_nodes, 0, o);
  c->cur_rq = ReqMap{0, 0, 0, 0};
  return s;
}

// prefill chunk of slot b: a chain of m nodes of that request (rows all belong to request b)
ss_status do_verify_slot(ss_ctx* c, int b) {
  PassOut o;
  o.argmax = true;
  c->cur_rq = c->Bmax > 1 ? ReqMap{0, b, c->max_nodes, c->C} : ReqMap{0, 0, 0, 0};
  ss_status s = forward_pass(c, true, c->n_nodes, 0, o);
  c->cur_rq = ReqMap{0, 0, 0, 0};
  return s;
}

ss_status do_accept(ss_ctx* c, bool chain, int slot = 0) {
  AcceptParams a{};
  a.n_req = chain ? 1 : c->B;   // a prefill chunk commits one slot
  a.req0 = chain ? slot : 0;
  a.node_stride = c->max_nodes;
  a.ctx_stride = c->C;
  a.out_stride = c->max_nodes + 1;
  a.argmax = c->argmax;
  a.tok = c->tok;
  a.parent = c->parent;
  a.commit_meta = c->commit_meta;
  a.n_nodes = c->n_nodes;
  a.k = std::max(1, c->cur_k);
  a.depth_max = c->cur_deff;
  a.committed_len = c->committed_len;
  a.root_tok = c->root_tok;
  a.out_tokens = c->out_tokens;
  a.out_n = c->out_n;
  a.out_path = c->out_path;
  a.k_cache = c->kc;
  a.v_cache = c->vc;
  a.k_tree = c->kt;
  a.v_tree = c->vt;
  // the commit copies 16-bit units: fp32 K/V rows are 2 head_dim units (strides in units too)
  const int u = c->kv_es / 2;
  a.cache_layer_stride = c->kc_layer * u;
  a.tree_layer_stride = c->kt_layer * u;
  a.n_layers = c->L;
  a.n_kv = c->nkv;
  a.head_dim = c->d * u;
  a.max_ctx = c->kv_ctx;
  a.max_nodes = c->kv_nodes;
  a.chain = chain ? 1 : 0;
  launch_accept_commit(a, c->use_pdl, c->cs);
  c->launches += 2;
  if (c->kcd) {   // NEXT-4: the same path's draft K/V into the draft's own cache (same commit meta)
    AcceptParams d = a;
    d.k_cache = c->kcd;
    d.v_cache = c->vcd;
    d.k_tree = c->ktd;
    d.v_tree = c->vtd;
    launch_commit(d, c->use_pdl, c->cs);
    c->launches++;
  }
  return check_launch(c, "accept_commit");
}

ss_status read_outputs(ss_ctx* c, int cap, int32_t* out_tokens, int32_t* out_n, int32_t* opt_path, int slot = 0) {
  const int64_t so = int64_t(slot) * (c->max_nodes + 1);
  CK(cudaMemcpyAsync(c->h_out, c->out_n + slot, 4, cudaMemcpyDeviceToHost, c->cs));
  CK(cudaMemcpyAsync(c->h_out + 1, c->out_tokens + so, size_t(cap) * 4, cudaMemcpyDeviceToHost, c->cs));
  if (opt_path) CK(cudaMemcpyAsync(c->h_out + 1 + cap, c->out_path + so, size_t(cap) * 4, cudaMemcpyDeviceToHost, c->cs));
  CK(cudaStreamSynchronize(c->cs));
  const int n = c->h_out[0];
  if (out_n) *out_n = n;
  if (out_tokens) std::memcpy(out_tokens, c->h_out + 1, size_t(std::min(n, cap)) * 4);
  if (opt_path) std::memcpy(opt_path, c->h_out + 1 + cap, size_t(std::min(n, cap)) * 4);
  return SS_OK;
}

bool valid_cfg(const ss_model_config* m, const ss_limits* l) {
  if (!m || !l) return false;
  if (m->n_layers < 1 || m->hidden % 128 || m->ffn % 128 || m->vocab % 128 || m->n_heads < 1 || m->n_kv_heads < 1)
    return false;
  if (m->n_heads % m->n_kv_heads) return false;
  if (m->head_dim != 64 && m->head_dim != 128) return false;
  if (((m->n_heads + 2 * m->n_kv_heads) * m->head_dim) % 128) return false;
  if ((m->n_heads * m->head_dim) % 128) return false;
  if (m->max_context < 2 || m->max_context > 8192) return false;
  if (m->n_heads / m->n_kv_heads > 16) return false;
  if (m->precision != SS_BF16 && m->precision != SS_FP32) return false;
  if (l->max_depth < 0 || l->max_top_k < 1 || l->max_top_k > 32 || l->max_chunk < 1 || l->max_chunk > 1024) return false;
  // batched slots: a draft pass forwards max_batch * k <= 32 frontier rows (GEMV token tiles)
  if (l->max_batch < 0 || l->max_batch > 32 || (l->max_batch > 1 && l->max_batch * l->max_top_k > 32)) return false;
  return true;
}

// NVTX range over one phase of the step (host side; nsys shows the kernels it enqueues beneath it)
struct NvtxRange {
  explicit NvtxRange(const char* name, uint32_t argb) {
    nvtxEventAttributes_t a = {};
    a.version = NVTX_VERSION;
    a.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
    a.colorType = NVTX_COLOR_ARGB;
    a.color = argb;
    a.messageType = NVTX_MESSAGE_TYPE_ASCII;
    a.message.ascii = name;
    nvtxRangePushEx(&a);
  }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

#define GUARD(c)                                                                 \
  do {                                                                           \
    if (!(c)) return SS_ERR_INVALID;                                             \
    if ((c)->poisoned) return SS_ERR_CUDA;                                       \
    cudaSetDevice((c)->device);                                                  \
  } while (0)

}  // namespace

// ================================== C-ABI ===================================================
extern "C" {

void ss_default_options(ss_options* o) {
  if (!o) return;
  o->embed_on_host = 1;
  o->async_stream = 1;
  o->cuda_graphs = 1;
  o->fuse_norm = 1;
  o->separate_draft_kv = 0;
  o->compress_stream = 1;
}

ss_status ss_create(const ss_model_config* cfg, const ss_limits* lim, const ss_options* opt, int device, void* dev_arena,
                    size_t arena_bytes, void* compute_stream, void* copy_stream, ss_ctx** out) {
  if (!out || !valid_cfg(cfg, lim) || !dev_arena) return SS_ERR_INVALID;
  *out = nullptr;
  ss_ctx* c = new ss_ctx();
  c->cfg = *cfg;
  c->lim = *lim;
  ss_default_options(&c->opt);
  if (opt) c->opt = *opt;
  c->serial_stream = !c->opt.async_stream;
  c->use_graphs = c->opt.cuda_graphs != 0;
  c->f32 = cfg->precision == SS_FP32;
  if (c->f32) {
    if (lim->max_batch > 1) {   // the fp32 parity mode serves one request
      delete c;
      return SS_ERR_INVALID;
    }
    c->kv_es = 4;
    c->use_graphs = false;
  }
  c->fuse_norm = c->opt.fuse_norm != 0;
  c->zcomp = c->opt.compress_stream != 0 && !c->f32;   // the fp32 parity mode reads the store in place
  if (c->opt.separate_draft_kv && (c->f32 || lim->max_batch > 1)) {   // NEXT-4 variant: one bf16 request
    delete c;
    return SS_ERR_INVALID;
  }
  c->device = device;
  if (cudaSetDevice(device) != cudaSuccess) {
    delete c;
    return SS_ERR_CUDA;
  }
  c->cs = reinterpret_cast<cudaStream_t>(compute_stream);
  c->xs = reinterpret_cast<cudaStream_t>(copy_stream);
  c->ar.base = reinterpret_cast<uint8_t*>(dev_arena);
  c->ar.cap = arena_bytes;
  c->H = cfg->hidden;
  c->F = cfg->ffn;
  c->nh = cfg->n_heads;
  c->nkv = cfg->n_kv_heads;
  c->d = cfg->head_dim;
  c->qd = c->nh * c->d;
  c->kvd = c->nkv * c->d;
  c->qkv_rows = c->qd + 2 * c->kvd;
  c->L = cfg->n_layers;
  c->V = cfg->vocab;
  c->C = cfg->max_context;
  c->gN[0] = c->qkv_rows; c->gK[0] = c->H;
  c->gN[1] = c->H;        c->gK[1] = c->qd;
  c->gN[2] = 2 * c->F;    c->gK[2] = c->H;
  c->gN[3] = c->H;        c->gK[3] = c->F;
  int dev_sms = 148;
  cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, device);
  c->gv_grid = dev_sms;
  const int k = lim->max_top_k, D = lim->max_depth;
  c->max_nodes = std::max(1 + k * D, lim->max_chunk);
  c->anc_stride = std::max(D + 1, lim->max_chunk);
  c->Bmax = std::max(1, int(lim->max_batch));
  c->B = 1;
  c->Pb.assign(size_t(c->Bmax), 0);
  c->slot_ready.assign(size_t(c->Bmax), 0);
  c->kv_nodes = c->Bmax * c->max_nodes;
  c->kv_ctx = c->Bmax * c->C;
  // rows of a pass: a prefill chunk, or a verify over every slot's tree
  c->mpad_max = std::max(32, ((std::max(c->max_nodes, c->Bmax * (1 + k * D)) + 127) / 128) * 128);
  Arena& a = c->ar;
  auto A = [&](size_t bytes) { return a.alloc(bytes); };
  bool ok = true;
  auto chk = [&](void* p) { ok = ok && p != nullptr; return p; };
  // The embedding is only ever gathered (<= max_nodes rows per pass).  opt.embed_on_host = 1 keeps it
  // in mapped, portable pinned host memory and reads rows over the host link (zero-copy), which
  // leaves its 2*V*H bytes of the VRAM cap to the streaming ring (reading R24); 0 keeps it
  // in the arena, PAPER.md:534's GPU-resident placement.
  {
    if (c->opt.embed_on_host &&
        cudaHostAlloc(&c->h_embed, size_t(c->V) * c->H * 2, cudaHostAllocMapped | cudaHostAllocPortable) == cudaSuccess) {
      void* dptr = nullptr;
      cudaHostGetDevicePointer(&dptr, c->h_embed, 0);
      c->embed = reinterpret_cast<uint16_t*>(dptr);
    } else {
      cudaGetLastError();
      c->h_embed = nullptr;
      c->embed = (uint16_t*)chk(A(size_t(c->V) * c->H * 2));
    }
  }
  c->head = (uint8_t*)chk(A(bf16_bytes(c->V, c->H)));
  c->final_norm = (uint16_t*)chk(A(size_t(c->H) * 2));
  c->lw.resize(c->L);
  for (auto& w : c->lw) {
    w.attn_norm = (uint16_t*)chk(A(size_t(c->H) * 2));
    w.mlp_norm = (uint16_t*)chk(A(size_t(c->H) * 2));
    if (cfg->qkv_bias) w.bias = (uint16_t*)chk(A(size_t(c->qkv_rows) * 2));
  }
  c->kc_layer = int64_t(c->nkv) * c->kv_ctx * c->d;
  c->kt_layer = int64_t(c->nkv) * c->kv_nodes * c->d;
  c->kc = (uint16_t*)chk(A(size_t(c->L) * c->kc_layer * c->kv_es));
  c->vc = (uint16_t*)chk(A(size_t(c->L) * c->kc_layer * c->kv_es));
  c->kt = (uint16_t*)chk(A(size_t(c->L) * c->kt_layer * c->kv_es));
  c->vt = (uint16_t*)chk(A(size_t(c->L) * c->kt_layer * c->kv_es));
  if (c->opt.separate_draft_kv) {
    c->kcd = (uint16_t*)chk(A(size_t(c->L) * c->kc_layer * 2));
    c->vcd = (uint16_t*)chk(A(size_t(c->L) * c->kc_layer * 2));
    c->ktd = (uint16_t*)chk(A(size_t(c->L) * c->kt_layer * 2));
    c->vtd = (uint16_t*)chk(A(size_t(c->L) * c->kt_layer * 2));
  }
  if (c->f32) {
    const size_t rows = size_t(c->mpad_max);
    c->h32 = (float*)chk(A(rows * std::max(c->H, c->qd) * 4));
    c->q32 = (float*)chk(A(rows * c->qd * 4));
    c->o32 = (float*)chk(A(rows * c->qd * 4));
    c->y32 = (float*)chk(A(rows * std::max({c->qkv_rows, 2 * c->F, c->H}) * 4));
    c->a32 = (float*)chk(A(rows * c->F * 4));
    c->logits32 = (float*)chk(A(rows * c->V * 4));
  }
  c->tok = (int*)chk(A(size_t(c->kv_nodes) * 4));
  c->parent = (int*)chk(A(size_t(c->kv_nodes) * 4));
  c->depth = (int*)chk(A(size_t(c->kv_nodes) * 4));
  c->score = (float*)chk(A(size_t(c->kv_nodes) * 4));
  c->anc = (int*)chk(A(size_t(c->kv_nodes) * c->anc_stride * 4));
  c->committed_len = (int*)chk(A(std::max<size_t>(64, size_t(c->Bmax) * 4)));
  c->root_tok = (int*)chk(A(std::max<size_t>(64, size_t(c->Bmax) * 4)));
  c->tokbuf = (int*)chk(A(size_t(lim->max_chunk) * 4));
  const int fx_cols = std::max({c->H, c->qd, c->F});
  c->x = (float*)chk(A(size_t(c->mpad_max) * c->H * 4));
  c->hfrag = (uint16_t*)chk(A(size_t(c->mpad_max) * fx_cols * 2));
  c->attnfrag = (uint16_t*)chk(A(size_t(c->mpad_max) * c->qd * 2));
  c->actfrag = (uint16_t*)chk(A(size_t(c->mpad_max) * c->F * 2));
  c->qbuf = (uint16_t*)chk(A(size_t(c->mpad_max) * c->qd * 2));
  c->hxs = (float*)chk(A(size_t(c->mpad_max) * (fx_cols / 64) * 4));
  c->attnxs = (float*)chk(A(size_t(c->mpad_max) * (c->qd / 64) * 4));
  c->actxs = (float*)chk(A(size_t(c->mpad_max) * (c->F / 64) * 4));
  // draft logits [32 x V]: written only by the fp32 parity mode and the debug entry points (the bf16
  // draft keeps per-tile top-k statistics instead); outside fp32 mode they live in a debug buffer
  // allocated on first debug use, outside the VRAM cap
  if (c->f32) c->logits = (float*)chk(A(size_t(32) * c->V * 4));
  c->tracebuf = (unsigned long long*)chk(A(size_t(512) * kTraceEvents * 8));
  c->sumsq = (float*)chk(A(size_t(c->H / 128) * 32 * 4));
  c->norm_ctr = (unsigned long long*)chk(A(256));   // 24 monotonic counters (3 x 2 formats x NT 1..4), zeroed below
  c->flags = (uint32_t*)chk(A(2 * kCoopMax * 4));   // NEXT-1 stream flags, zeroed by ss_coop_export
  c->rope = (float2*)chk(A(size_t(c->C) * (c->d / 2) * 8));
  // gemv partials: worst case over groups and the head at Mpad = 32
  size_t gvf = 0;
  int max_tiles = 0;
  for (int g = 0; g < 5; ++g) {
    const int N = g < 4 ? c->gN[g] : c->V, K = g < 4 ? c->gK[g] : c->H;
    for (int q4 = 0; q4 < 2; ++q4)
      gvf = std::max(gvf, size_t(N / 128) * gemv_max_segments(N, K, gemv_streamk_grid(q4, N, K, c->gv_grid)) * 128 * 32);
    max_tiles = std::max(max_tiles, N / 128);
  }
  c->gv_part_floats = gvf;
  c->gv_part = (float*)chk(A(gvf * 4));
  c->gv_cnt = (int*)chk(A(size_t(max_tiles) * 4));
  {
    // debug output scratch of ss_debug_matmul / ss_debug_time_matmul: one request's rows x the widest
    // matrix group, or 32 rows of logits
    const size_t mpad_one = size_t(std::max(32, ((c->max_nodes + 127) / 128) * 128));
    c->at_o_floats = std::max(mpad_one * std::max({c->gN[0], c->gN[1], c->gN[2], c->gN[3]}), size_t(32) * c->V);
    // allocated on first debug use (ensure_debug_bufs), outside the VRAM cap: not a product buffer
  }
  {   // top-k statistics: [32 rows][blocks] of the two-stage kernels (296) or of the head's vocab tiles
    const size_t nb = std::max<size_t>(296, size_t(c->V / 128));
    c->tk_max = (float*)chk(A(size_t(32) * nb * 4));
    c->tk_sum = (float*)chk(A(size_t(32) * nb * 4));
    c->tk_val = (float*)chk(A(size_t(32) * nb * lim->max_top_k * 4));
    c->tk_idx = (int*)chk(A(size_t(32) * nb * lim->max_top_k * 4));
  }
  c->vtiles = c->V / 128;
  c->am_val = (float*)chk(A(size_t(c->mpad_max) * c->vtiles * 4));
  c->am_sec = (float*)chk(A(size_t(c->mpad_max) * c->vtiles * 4));
  c->am_idx = (int*)chk(A(size_t(c->mpad_max) * c->vtiles * 4));
  c->argmax = (int*)chk(A(size_t(c->mpad_max) * 4));
  c->gap = (float*)chk(A(size_t(c->mpad_max) * 4));
  c->out_tokens = (int*)chk(A(size_t(c->Bmax) * (c->max_nodes + 1) * 4));
  c->out_n = (int*)chk(A(std::max<size_t>(64, size_t(c->Bmax) * 4)));
  c->out_path = (int*)chk(A(size_t(c->Bmax) * (c->max_nodes + 1) * 4));
  c->commit_meta = (int*)chk(A(std::max<size_t>(64, size_t(c->Bmax) * 8)));
  if (!ok) {
    delete c;
    return SS_ERR_BUDGET;
  }
  // zero everything carved so far (padding rows of FragX buffers must be finite; counters 0)
  if (cudaMemsetAsync(a.base, 0, a.used, c->cs) != cudaSuccess) {
    delete c;
    return SS_ERR_CUDA;
  }
  // RoPE table (cos, sin) of pos * theta^(-2j/d), computed in double
  std::vector<float2> rope(size_t(c->C) * (c->d / 2));
  for (int p = 0; p < c->C; ++p)
    for (int j = 0; j < c->d / 2; ++j) {
      const double ang = double(p) * std::pow(double(cfg->rope_theta), -2.0 * j / c->d);
      rope[size_t(p) * (c->d / 2) + j] = make_float2(float(std::cos(ang)), float(std::sin(ang)));
    }
  cudaMemcpyAsync(c->rope, rope.data(), rope.size() * 8, cudaMemcpyHostToDevice, c->cs);
  cudaStreamSynchronize(c->cs);
  cudaHostAlloc(&c->h_out, (size_t(2 * c->Bmax) * (c->max_nodes + 1) + c->Bmax + 8) * 4, cudaHostAllocPortable);
  cudaEventCreate(&c->e0);
  cudaEventCreate(&c->e1);
  cudaEventCreate(&c->e2);
  cudaEventCreate(&c->e3);
  cudaEventCreateWithFlags(&c->ev_root, cudaEventDisableTiming);
  cudaEventCreate(&c->ev_ref);
  cudaEventCreate(&c->ev_region);
  cudaEventRecord(c->ev_ref, c->cs);
  cudaHostAlloc(&c->h_root, 64, cudaHostAllocPortable);
  if (cudaDeviceSynchronize() != cudaSuccess || cudaGetLastError() != cudaSuccess || !c->h_out || !c->h_root) {
    delete c;
    return SS_ERR_CUDA;
  }
  c->st.arena_cap = int64_t(arena_bytes);
  *out = c;
  return SS_OK;
}

// Caller-owned host stores are page-locked with cudaHostRegister once per process (refcounted:
// several contexts of one process may share a store).
static std::mutex g_reg_mu;
static std::map<void*, int> g_reg_count;
static bool host_register(void* p, size_t bytes) {
  std::lock_guard<std::mutex> lk(g_reg_mu);
  int& n = g_reg_count[p];
  if (n == 0) {
    cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterPortable);
    if (e == cudaErrorHostMemoryAlreadyRegistered) {
      cudaGetLastError();
      n = 1 << 20;   // registered by someone else: never unregister it here
    } else if (e != cudaSuccess) {
      cudaGetLastError();
      g_reg_count.erase(p);
      return false;
    }
  }
  ++n;
  return true;
}
static void host_unregister(void* p) {
  std::lock_guard<std::mutex> lk(g_reg_mu);
  auto it = g_reg_count.find(p);
  if (it == g_reg_count.end()) return;
  if (--it->second == 0) {
    cudaHostUnregister(p);
    cudaGetLastError();
    g_reg_count.erase(it);
  }
}

// host-store bytes of one offloaded group: plain bf16, or a codec blob's capacity (raw fallback fits)
static size_t group_store_bytes(ss_ctx* c, int g) {
  const int64_t n = int64_t(c->gN[g]) * c->gK[g];
  return c->zcomp ? (zblob_cap(n) + 4095) / 4096 * 4096 : size_t(n) * 2;
}
static size_t host_store_bytes(ss_ctx* c, int nr) {
  size_t layer = 0;
  for (int g = 0; g < 4; ++g) layer += group_store_bytes(c, g);
  return size_t(c->L - nr) * layer;
}

// the offloaded group (l, g) whose tiled bf16 is at ring[0, 2n) -> the host store (blob or plain)
static ss_status store_group(ss_ctx* c, int l, int g) {
  LayerW& w = c->lw[l];
  const int64_t n = int64_t(c->gN[g]) * c->gK[g];
  if (!c->zcomp) {
    CK(cudaMemcpyAsync(c->host + w.host_off[g], c->ring, size_t(n) * 2, cudaMemcpyDeviceToHost, c->cs));
    CK(cudaStreamSynchronize(c->cs));
    w.zmode[g] = -1;
    w.host_used[g] = size_t(n) * 2;
    w.host_a0[g] = 0;
    return SS_OK;
  }
  const size_t a2n = (size_t(n) * 2 + 4095) / 4096 * 4096;
  uint8_t* blob = c->ring + a2n;
  uint8_t* scratch = blob + (zblob_cap(n) + 4095) / 4096 * 4096;
  if (size_t(scratch - c->ring) + 4 * (256 + size_t(n / kZChunk)) > c->ring_bytes)
    return fail(c, SS_ERR_BUDGET, "ring too small to encode a matrix group");
  ZHeader hd{};
  CK(zencode(reinterpret_cast<const uint16_t*>(c->ring), n, blob, scratch, c->cs, &hd));
  CK(cudaMemcpyAsync(c->host + w.host_off[g], blob, hd.used, cudaMemcpyDeviceToHost, c->cs));
  CK(cudaStreamSynchronize(c->cs));
  w.zmode[g] = int(hd.mode);
  w.host_used[g] = hd.used;
  w.host_a0[g] = hd.a0;
  return SS_OK;
}

// a group already in a shared host store (attach): its blob header says how it is stored
static ss_status attach_group(ss_ctx* c, int l, int g) {
  LayerW& w = c->lw[l];
  const int64_t n = int64_t(c->gN[g]) * c->gK[g];
  if (!c->zcomp) {
    w.zmode[g] = -1;
    w.host_used[g] = size_t(n) * 2;
    w.host_a0[g] = 0;
    return SS_OK;
  }
  ZHeader hd;
  std::memcpy(&hd, c->host + w.host_off[g], sizeof(hd));
  if (hd.magic != kZMagic || hd.n != uint64_t(n) || hd.used > group_store_bytes(c, g))
    return fail(c, SS_ERR_INVALID, "shared host store: not filled by a context with the same model and codec");
  w.zmode[g] = int(hd.mode);
  w.host_used[g] = hd.used;
  w.host_a0[g] = hd.a0;
  return SS_OK;
}

ss_status ss_host_store_bytes(ss_ctx* c, int32_t n_resident, size_t* out) {
  GUARD(c);
  if (!out || n_resident < 0 || n_resident > c->L) return fail(c, SS_ERR_INVALID, "host_store_bytes args");
  *out = host_store_bytes(c, n_resident);
  return SS_OK;
}

// Synthetic weights (SURVEY O.1 generator; tensor ids as synth/weights.py), generated on the device.
static ss_status fill_synthetic(ss_ctx* c, uint64_t seed, bool fill) {
  const double H = c->H;
  if (c->h_embed) {   // generate on the device (ring scratch), then place in the host copy
    // in ring-sized pieces (a planner-max placement leaves a ring of only two matrix groups)
    const uint64_t total = uint64_t(c->V) * c->H, piece = uint64_t(c->ring_bytes / 2);
    for (uint64_t first = 0; first < total; first += piece) {
      const uint64_t n = std::min(piece, total - first);
      launch_gen_natural(reinterpret_cast<uint16_t*>(c->ring), tensor_key(seed, 0), n, scale_c32(1.0), 0, c->cs, first);
      CK(cudaMemcpyAsync(reinterpret_cast<uint16_t*>(c->h_embed) + first, c->ring, n * 2, cudaMemcpyDeviceToHost, c->cs));
      CK(cudaStreamSynchronize(c->cs));
    }
  } else {
    launch_gen_natural(c->embed, tensor_key(seed, 0), uint64_t(c->V) * c->H, scale_c32(1.0), 0, c->cs);
  }
  launch_gen_tiled(c->head, tensor_key(seed, 2 + 16 * c->L), c->V, c->H, scale_c32(1.0 / std::sqrt(H)), 0, 0, c->cs);
  launch_gen_natural(c->final_norm, tensor_key(seed, 1 + 16 * c->L), c->H, scale_c32(0.05), 1, c->cs);
  for (int l = 0; l < c->L; ++l) {
    LayerW& w = c->lw[l];
    const uint64_t b = 1 + 16 * uint64_t(l);
    launch_gen_natural(w.attn_norm, tensor_key(seed, b + 0), c->H, scale_c32(0.05), 1, c->cs);
    launch_gen_natural(w.mlp_norm, tensor_key(seed, b + 8), c->H, scale_c32(0.05), 1, c->cs);
    if (w.bias) {
      launch_gen_natural(w.bias, tensor_key(seed, b + 2), c->qd, scale_c32(0.02), 0, c->cs);
      launch_gen_natural(w.bias + c->qd, tensor_key(seed, b + 4), c->kvd, scale_c32(0.02), 0, c->cs);
      launch_gen_natural(w.bias + c->qd + c->kvd, tensor_key(seed, b + 6), c->kvd, scale_c32(0.02), 0, c->cs);
    }
    for (int g = 0; g < 4; ++g) {
      if (!w.resident && !fill) {   // shared store already holds this matrix
        ss_status s = attach_group(c, l, g);
        if (s != SS_OK) return s;
        continue;
      }
      uint8_t* dst = w.resident ? w.bf16[g] : c->ring;
      const int K = c->gK[g];
      const float cin = scale_c32(1.0 / std::sqrt(double(K)));
      if (g == 0) {
        launch_gen_tiled(dst, tensor_key(seed, b + 1), c->qd, K, cin, 0, 0, c->cs);
        launch_gen_tiled(dst, tensor_key(seed, b + 3), c->kvd, K, cin, 0, c->qd, c->cs);
        launch_gen_tiled(dst, tensor_key(seed, b + 5), c->kvd, K, cin, 0, c->qd + c->kvd, c->cs);
      } else if (g == 1) {
        launch_gen_tiled(dst, tensor_key(seed, b + 7), c->H, K, cin, 0, 0, c->cs);
      } else if (g == 2) {
        launch_gen_tiled(dst, tensor_key(seed, b + 9), c->F, K, cin, 1, 0, c->cs);
        launch_gen_tiled(dst, tensor_key(seed, b + 10), c->F, K, cin, 2, 0, c->cs);
      } else {
        launch_gen_tiled(dst, tensor_key(seed, b + 11), c->H, K, cin, 0, 0, c->cs);
      }
      if (!w.resident && fill) {
        ss_status s = store_group(c, l, g);
        if (s != SS_OK) return s;
      }
    }
  }
  return SS_OK;
}

static ss_status load_impl(ss_ctx* c, const ss_host_weights* hw, uint64_t seed, int32_t n_resident, void* ext_host,
                           size_t ext_bytes, bool fill);

ss_status ss_set_substitute_bits(ss_ctx* c, int32_t bits) {
  GUARD(c);
  if (c->state != ST_CREATED) return fail(c, SS_ERR_STRUCTURE, "set_substitute_bits: only before load_weights");
  if (bits != 4 && bits != 3 && bits != 2) return fail(c, SS_ERR_INVALID, "set_substitute_bits: 4, 3 or 2");
  c->sub_bits = bits;
  return SS_OK;
}

ss_status ss_load_weights(ss_ctx* c, const ss_host_weights* w, int32_t n_resident) {
  GUARD(c);
  if (!w || !w->embed || !w->layers || !w->final_norm || !w->head) return fail(c, SS_ERR_INVALID, "load_weights: NULL tensor");
  for (int l = 0; l < c->L; ++l) {
    const ss_host_layer& h = w->layers[l];
    if (!h.attn_norm || !h.wq || !h.wk || !h.wv || !h.wo || !h.mlp_norm || !h.wg || !h.wu || !h.wd)
      return fail(c, SS_ERR_INVALID, "load_weights: NULL layer tensor");
    const bool b = h.bq && h.bk && h.bv, any = h.bq || h.bk || h.bv;
    if (c->cfg.qkv_bias ? !b : any) return fail(c, SS_ERR_INVALID, "load_weights: biases must match cfg.qkv_bias");
  }
  return load_impl(c, w, 0, n_resident, nullptr, 0, true);
}

ss_status ss_load_weights_synthetic(ss_ctx* c, uint64_t seed, int32_t n_resident) {
  GUARD(c);
  return load_impl(c, nullptr, seed, n_resident, nullptr, 0, true);
}

ss_status ss_load_weights_synthetic_shared(ss_ctx* c, uint64_t seed, int32_t n_resident, void* host_store,
                                           size_t host_bytes, int32_t fill) {
  GUARD(c);
  if (!host_store || n_resident < 0) return fail(c, SS_ERR_INVALID, "load_weights_shared: store and n_resident >= 0");
  return load_impl(c, nullptr, seed, n_resident, host_store, host_bytes, fill != 0);
}

// Place one matrix group (layer l, group g) from the caller's natural row-major host arrays: each
// source matrix is copied to the device (staging) and tiled into dst (resident buffer or ring).
static ss_status fill_group_from_host(ss_ctx* c, const ss_host_layer& h, int g, uint8_t* dst, uint16_t* staging) {
  const int K = c->gK[g];
  struct Piece { const uint16_t* src; int64_t rows; int map; int64_t row_off; };
  std::vector<Piece> pieces;
  if (g == 0) pieces = {{h.wq, c->qd, 0, 0}, {h.wk, c->kvd, 0, c->qd}, {h.wv, c->kvd, 0, c->qd + c->kvd}};
  else if (g == 1) pieces = {{h.wo, c->H, 0, 0}};
  else if (g == 2) pieces = {{h.wg, c->F, 1, 0}, {h.wu, c->F, 2, 0}};
  else pieces = {{h.wd, c->H, 0, 0}};
  for (const Piece& p : pieces) {
    CK(cudaMemcpyAsync(staging, p.src, size_t(p.rows) * K * 2, cudaMemcpyHostToDevice, c->cs));
    launch_tile_from_natural(dst, staging, p.rows, K, p.map, p.row_off, c->cs);
    CK(cudaStreamSynchronize(c->cs));   // the staging buffer is reused by the next piece
  }
  return check_launch(c, "tile_from_natural");
}

static ss_status load_impl(ss_ctx* c, const ss_host_weights* hw, uint64_t seed, int32_t n_resident, void* ext_host,
                           size_t ext_bytes, bool fill) {
  if (c->state != ST_CREATED) return fail(c, SS_ERR_STRUCTURE, "load_weights: already loaded");
  if (c->f32 && ext_host) return fail(c, SS_ERR_INVALID, "the fp32 parity mode keeps its own host store");
  c->seed = seed;
  const size_t layer_bf16 = [&] { size_t s = 0; for (int g = 0; g < 4; ++g) s += bf16_bytes(c->gN[g], c->gK[g]); return s; }();
  const size_t layer_q4 = [&] { size_t s = 0; for (int g = 0; g < 4; ++g) s += sub_bytes(c->gN[g], c->gK[g], c->sub_bits); return s; }();
  size_t max_group = 0, max_tile_row = 0;
  for (int g = 0; g < 4; ++g) {
    max_group = std::max(max_group, bf16_bytes(c->gN[g], c->gK[g]));
    max_tile_row = std::max(max_tile_row, size_t(c->gK[g] / 128) * kBF16TileBytes);
  }
  // K7 codec decode buffer: 64 MiB (the small groups fit whole; gate_up / down decode in row blocks)
  c->dbuf_bytes = std::min(max_group, std::max(size_t(64) << 20, max_tile_row));
  const size_t avail = c->ar.cap - c->ar.used - 4096 * 8;
  auto need = [&](int nr) {
    const int off = c->L - nr;
    // offloaded layers: a ring of >= two groups (+ codec scratch) and, with the codec, the decode buffer
    return size_t(nr) * layer_bf16 + size_t(off) * layer_q4 +
           (off > 0 ? 2 * max_group + (c->zcomp ? c->dbuf_bytes + (8u << 20) : 0) : max_group);
  };
  int nr = n_resident;
  if (nr < 0) {
    nr = 0;
    while (nr < c->L && need(nr + 1) <= avail) ++nr;
  }
  if (nr > c->L) return fail(c, SS_ERR_INVALID, "n_resident > n_layers");
  if (need(nr) > avail) return fail(c, SS_ERR_BUDGET, "arena below the minimum footprint for this placement");
  c->n_resident = nr;
  for (int l = 0; l < c->L; ++l) {
    LayerW& w = c->lw[l];
    w.resident = l < nr;
    for (int g = 0; g < 4; ++g) {
      if (w.resident)
        w.bf16[g] = (uint8_t*)c->ar.alloc(bf16_bytes(c->gN[g], c->gK[g]), 1024);
      else
        w.q4[g] = (uint8_t*)c->ar.alloc(sub_bytes(c->gN[g], c->gK[g], c->sub_bits), 1024);
    }
  }
  if (c->zcomp && nr < c->L) {
    c->dbuf = (uint16_t*)c->ar.alloc(c->dbuf_bytes, 4096);
    if (!c->dbuf) return fail(c, SS_ERR_BUDGET, "no room for the stream decode buffer");
  }
  // the staging ring takes what is left
  c->ring_bytes = (c->ar.cap - c->ar.used - 4096) / 4096 * 4096;
  c->ring = (uint8_t*)c->ar.alloc(c->ring_bytes, 4096);
  if (!c->ring || c->ring_bytes < max_group) return fail(c, SS_ERR_BUDGET, "no room for the staging ring");
  // pinned host store for offloaded layers (device layout)
  c->host_bytes = host_store_bytes(c, nr);
  if (ext_host) {
    if (ext_bytes < c->host_bytes) return fail(c, SS_ERR_BUDGET, "shared host store smaller than ss_host_store_bytes");
    if (c->host_bytes && !host_register(ext_host, c->host_bytes))
      return fail(c, SS_ERR_CUDA, "cudaHostRegister of the shared host store failed");
    c->host = reinterpret_cast<uint8_t*>(ext_host);
    c->host_external = true;
  }
  if (c->host_bytes) {
    // fp32 parity mode: the target reads offloaded layers in place through a device-mapped view
    const unsigned flags = cudaHostAllocPortable | (c->f32 ? cudaHostAllocMapped : 0u);
    if (!c->host_external && cudaHostAlloc(&c->host, c->host_bytes, flags) != cudaSuccess)
      return fail(c, SS_ERR_CUDA, "cudaHostAlloc of the pinned host store failed");
    if (c->f32) {
      void* dp = nullptr;
      CK(cudaHostGetDevicePointer(&dp, c->host, 0));
      c->host_dev = reinterpret_cast<uint8_t*>(dp);
    }
    size_t off = 0;
    for (int l = nr; l < c->L; ++l)
      for (int g = 0; g < 4; ++g) {
        c->lw[l].host_off[g] = off;
        off += group_store_bytes(c, g);
      }
  }
  if (hw) {
    // caller weights: norms/biases/embedding copied as they are, matrices tiled on the device through
    // the ring (second half = natural staging, first half = tiled group when the layer is offloaded)
    const size_t E = size_t(c->V) * c->H * 2;
    if (c->h_embed) std::memcpy(c->h_embed, hw->embed, E);
    else CK(cudaMemcpyAsync(c->embed, hw->embed, E, cudaMemcpyHostToDevice, c->cs));
    CK(cudaMemcpyAsync(c->final_norm, hw->final_norm, size_t(c->H) * 2, cudaMemcpyHostToDevice, c->cs));
    uint16_t* staging = reinterpret_cast<uint16_t*>(c->ring + (c->ring_bytes >= 2 * max_group ? max_group : 0));
    if (c->ring_bytes < 2 * max_group && c->n_resident < c->L)
      return fail(c, SS_ERR_BUDGET, "load_weights: ring below two matrix groups");
    {   // head [V x H]: tiled in ring-sized row blocks
      const int64_t rows_per = std::max<int64_t>(128, int64_t(c->ring_bytes / (size_t(c->H) * 2)) / 128 * 128);
      for (int64_t r0 = 0; r0 < c->V; r0 += rows_per) {
        const int64_t n = std::min<int64_t>(rows_per, c->V - r0);
        uint16_t* st16 = reinterpret_cast<uint16_t*>(c->ring);
        CK(cudaMemcpyAsync(st16, hw->head + r0 * c->H, size_t(n) * c->H * 2, cudaMemcpyHostToDevice, c->cs));
        launch_tile_from_natural(c->head, st16, n, c->H, 0, r0, c->cs);
        CK(cudaStreamSynchronize(c->cs));
      }
    }
    for (int l = 0; l < c->L; ++l) {
      LayerW& w = c->lw[l];
      const ss_host_layer& h = hw->layers[l];
      CK(cudaMemcpyAsync(w.attn_norm, h.attn_norm, size_t(c->H) * 2, cudaMemcpyHostToDevice, c->cs));
      CK(cudaMemcpyAsync(w.mlp_norm, h.mlp_norm, size_t(c->H) * 2, cudaMemcpyHostToDevice, c->cs));
      if (w.bias) {
        CK(cudaMemcpyAsync(w.bias, h.bq, size_t(c->qd) * 2, cudaMemcpyHostToDevice, c->cs));
        CK(cudaMemcpyAsync(w.bias + c->qd, h.bk, size_t(c->kvd) * 2, cudaMemcpyHostToDevice, c->cs));
        CK(cudaMemcpyAsync(w.bias + c->qd + c->kvd, h.bv, size_t(c->kvd) * 2, cudaMemcpyHostToDevice, c->cs));
      }
      for (int g = 0; g < 4; ++g) {
        uint8_t* dst = w.resident ? w.bf16[g] : c->ring;
        ss_status s = fill_group_from_host(c, h, g, dst, w.resident ? reinterpret_cast<uint16_t*>(c->ring) : staging);
        if (s != SS_OK) return s;
        if (!w.resident && (s = store_group(c, l, g)) != SS_OK) return s;
      }
    }
  } else {
    ss_status s = fill_synthetic(c, seed, fill);
    if (s != SS_OK) return s;
  }
  CK(cudaStreamSynchronize(c->cs));
  ss_status s = check_launch(c, "load_weights");
  if (s != SS_OK) return s;
  // streaming cycle: offloaded layers in order, groups qkv, o, gate_up, down (none in fp32 mode)
  c->cycle.clear();
  for (int l = nr; l < c->L && !c->f32; ++l)
    for (int g = 0; g < 4; ++g) c->cycle.emplace_back(l, g);
  c->ev_pool = 4 * int(c->cycle.size()) + 64;
  for (int i = 0; i < c->ev_pool; ++i) {
    cudaEvent_t e1, e2, t0, t1;
    cudaEventCreateWithFlags(&e1, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&e2, cudaEventDisableTiming);
    cudaEventCreate(&t0);
    cudaEventCreate(&t1);
    c->ev_copied.push_back(e1);
    c->ev_consumed.push_back(e2);
    c->ev_t0.push_back(t0);
    c->ev_t1.push_back(t1);
  }
  c->ev_pending.assign(c->ev_pool, false);
  c->st.n_resident = nr;
  c->st.n_offloaded = c->L - nr;
  c->st.host_pinned_bytes = int64_t(c->host_bytes) + (c->h_embed ? int64_t(c->V) * c->H * 2 : 0);
  c->st.ring_bytes = int64_t(c->ring_bytes);
  c->st.arena_used = int64_t(c->ar.used);
  c->st.substitute_bytes = int64_t(size_t(c->L - nr) * layer_q4);
  c->state = ST_LOADED;
  return SS_OK;
}

ss_status ss_build_substitutes(ss_ctx* c, const ss_quant_spec* q) {
  NvtxRange nvtx_range("ss.build_substitutes", 0xFFF39C12u);
  GUARD(c);
  if (!q || (q->bits != 4 && q->bits != 3 && q->bits != 2) || q->group_size != 64)
    return fail(c, SS_ERR_INVALID, "substitutes are 4-, 3- or 2-bit with group 64");
  if ((q->method != SS_QUANT_RTN && q->method != SS_QUANT_HQQ) || q->hqq_iters < 0 || q->hqq_iters > 1000)
    return fail(c, SS_ERR_INVALID, "quantizer method is SS_QUANT_RTN or SS_QUANT_HQQ, hqq_iters in [0, 1000]");
  const int hqq_iters = q->method == SS_QUANT_HQQ ? (q->hqq_iters ? q->hqq_iters : 20) : 0;
  if (q->bits != c->sub_bits)
    return fail(c, SS_ERR_INVALID, "quant bits differ from the layout sized at load (ss_set_substitute_bits)");
  if (c->state != ST_LOADED) return fail(c, SS_ERR_STRUCTURE, "build_substitutes before load_weights");
  for (int l = c->n_resident; l < c->L; ++l)
    for (int g = 0; g < 4; ++g) {
      const LayerW& w = c->lw[l];
      const int64_t n = int64_t(c->gN[g]) * c->gK[g];
      const uint8_t* src = c->ring;   // the target's tiled bf16 (decoded from the host store's blob)
      if (w.zmode[g] < 0) {
        CK(cudaMemcpyAsync(c->ring, c->host + w.host_off[g], size_t(n) * 2, cudaMemcpyHostToDevice, c->cs));
      } else {
        uint8_t* blob = c->ring + (size_t(n) * 2 + 4095) / 4096 * 4096;
        CK(cudaMemcpyAsync(blob, c->host + w.host_off[g], w.host_used[g], cudaMemcpyHostToDevice, c->cs));
        if (w.zmode[g] == 1) launch_zdecode(blob, reinterpret_cast<uint16_t*>(c->ring), n, c->cs);
        else src = blob + w.host_a0[g];
      }
      launch_quantize(src, w.q4[g], c->gN[g], c->gK[g], c->sub_bits, hqq_iters, c->cs);
      CK(cudaStreamSynchronize(c->cs));
    }
  ss_status s = check_launch(c, "quantize");
  if (s != SS_OK) return s;
  c->substitutes_built = true;
  c->state = ST_READY;
  c->ring_head = 0;
  return pump(c);   // start streaming the first verify's layers right away
}

static ss_status prefill_slot_impl(ss_ctx* c, int slot, const int32_t* prompt, int32_t n, int32_t chunk,
                                   int32_t* out_first) {
  NvtxRange nvtx_range("ss.prefill", 0xFF8E44ADu);
  if (c->state < ST_READY) return fail(c, SS_ERR_STRUCTURE, "prefill before build_substitutes");
  if (c->state == ST_DRAFTED || c->state == ST_VERIFIED) return fail(c, SS_ERR_STRUCTURE, "prefill inside a step");
  if (slot < 0 || slot >= c->B) return fail(c, SS_ERR_INVALID, "prefill: slot outside the active batch");
  if (!prompt || n < 1 || chunk < 1 || chunk > c->lim.max_chunk) return fail(c, SS_ERR_INVALID, "prefill: bad prompt/chunk");
  if (n > c->C) return fail(c, SS_ERR_CAPACITY, "prompt longer than max_context");
  for (int i = 0; i < n; ++i)
    if (prompt[i] < 0 || prompt[i] >= c->V) return fail(c, SS_ERR_INVALID, "token id out of range");
  CK(cudaMemsetAsync(c->committed_len + slot, 0, 4, c->cs));
  c->Pb[slot] = 0;
  const int64_t no = int64_t(slot) * c->max_nodes;
  for (int c0 = 0; c0 < n; c0 += chunk) {
    const int m = std::min(chunk, n - c0);
    CK(cudaMemcpyAsync(c->tokbuf, prompt + c0, size_t(m) * 4, cudaMemcpyHostToDevice, c->cs));
    launch_chain_init(c->tokbuf, m, c->tok + no, c->parent + no, c->depth + no, c->score + no,
                      c->anc + no * c->anc_stride, c->anc_stride, c->cs);
    c->n_nodes = m;
    c->cur_k = 1;
    c->cur_deff = 0;
    for (int r0 = 0; c->kcd && r0 < m; r0 += 32) {   // NEXT-4: the draft's own K/V of the chunk (GEMV: <= 32 rows)
      ss_status s = forward_pass(c, false, std::min(32, m - r0), r0, PassOut{});
      if (s != SS_OK) return s;
    }
    ss_status s = do_verify_slot(c, slot);
    if (s != SS_OK) return s;
    if ((s = do_accept(c, true, slot)) != SS_OK) return s;
    c->Pb[slot] += m;
    // the pageable prompt buffer is reused next chunk: make the H2D copy complete
    CK(cudaStreamSynchronize(c->cs));
  }
  int32_t first = 0, nn = 0;
  ss_status s = read_outputs(c, 1, &first, &nn, nullptr, slot);
  if (s != SS_OK) return s;
  if (out_first) *out_first = first;
  c->st.prefill_tokens += n;
  c->P = c->Pb[0];
  c->st.committed_len = c->P;
  c->slot_ready[slot] = 1;
  bool all = true;
  for (int b = 0; b < c->B; ++b) all = all && c->slot_ready[b];
  c->state = all ? ST_SESSION : ST_READY;
  harvest_timing(c);
  return SS_OK;
}

ss_status ss_prefill(ss_ctx* c, const int32_t* prompt, int32_t n, int32_t chunk, int32_t* out_first) {
  GUARD(c);
  return prefill_slot_impl(c, 0, prompt, n, chunk, out_first);
}

ss_status ss_prefill_slot(ss_ctx* c, int32_t slot, const int32_t* prompt, int32_t n, int32_t chunk, int32_t* out_first) {
  GUARD(c);
  return prefill_slot_impl(c, slot, prompt, n, chunk, out_first);
}

ss_status ss_set_batch(ss_ctx* c, int32_t n_req) {
  GUARD(c);
  if (n_req < 1 || n_req > c->Bmax) return fail(c, SS_ERR_INVALID, "set_batch: n_req outside [1, max_batch]");
  if (c->state == ST_DRAFTED || c->state == ST_VERIFIED) return fail(c, SS_ERR_STRUCTURE, "set_batch inside a step");
  // every check above precedes any state change (a rejected call leaves the session intact)
  if (c->B > 1 || n_req > 1) {
    // a batch session starts over: every active slot is prefilled again
    std::fill(c->slot_ready.begin(), c->slot_ready.end(), 0);
    if (c->state == ST_SESSION) c->state = ST_READY;
  }
  c->B = n_req;
  return SS_OK;
}

static ss_status draft_impl(ss_ctx* c, int32_t root_token, const ss_draft_params* p) {
  NvtxRange nvtx_range("ss.draft_tree", 0xFF2E86C1u);
  if (!p || p->top_k < 1 || p->top_k > c->lim.max_top_k || p->depth < 0 || p->depth > c->lim.max_depth ||
      !(p->sharpen_t > 0.f) || !std::isfinite(p->sharpen_t))
    return fail(c, SS_ERR_INVALID, "draft params");
  if (c->state != ST_SESSION) return fail(c, SS_ERR_STRUCTURE, "draft_tree needs a prefilled session (and no pending step)");
  if (c->B > 1 && root_token >= 0) return fail(c, SS_ERR_INVALID, "batched draft: roots come from the previous step");
  int Pmax = 0;
  for (int b = 0; b < c->B; ++b) Pmax = std::max(Pmax, c->Pb[b]);
  if (Pmax + 1 > c->C) return fail(c, SS_ERR_CAPACITY, "context full");
  if (root_token >= c->V) return fail(c, SS_ERR_INVALID, "root token out of range");
  const int k = p->top_k;
  // O.10 capacity clamp; a batch shares one tree shape, clamped by its longest request
  const int deff = std::max(0, std::min(p->depth, (c->C - Pmax - 1) / k));
  if (root_token >= 0) {
    // pinned staging word: the copy is ordered on the compute stream and the host does not wait for
    // the draft (a blocked host would stop feeding the streaming ring during the draft)
    CK(cudaEventSynchronize(c->ev_root));   // the previous root copy has left the staging word
    *c->h_root = root_token;
    CK(cudaMemcpyAsync(c->root_tok, c->h_root, 4, cudaMemcpyHostToDevice, c->cs));
    CK(cudaEventRecord(c->ev_root, c->cs));
  }
  CK(cudaEventRecord(c->e0, c->cs));
  ss_status s;
  if (deff == 0) {
    launch_tree_init(c->root_tok, c->tok, c->parent, c->depth, c->score, c->anc, c->use_pdl, c->cs, c->B, c->max_nodes,
                     c->anc_stride);
    c->launches++;
    s = check_launch(c, "tree_init");
  } else {
    s = run_draft(c, deff, k, p->sharpen_t);
  }
  if (s != SS_OK) return s;
  CK(cudaEventRecord(c->e1, c->cs));
  c->cur_k = k;
  c->cur_deff = deff;
  c->n_nodes = 1 + k * deff;
  c->st.last_d_eff = deff;
  c->state = ST_DRAFTED;
  return SS_OK;
}

ss_status ss_draft_tree(ss_ctx* c, int32_t root_token, const ss_draft_params* p, int32_t* ot, int32_t* op, int32_t* od,
                        float* os, int32_t* on) {
  GUARD(c);
  ss_status s = draft_impl(c, root_token, p);
  if (s != SS_OK) return s;
  const int n = c->n_nodes;
  if (on) *on = n;
  for (int b = 0; b < c->B; ++b) {   // batched: [B][n] over the active slots
    const int64_t so = int64_t(b) * c->max_nodes, ho = int64_t(b) * n;
    if (ot) CK(cudaMemcpyAsync(ot + ho, c->tok + so, size_t(n) * 4, cudaMemcpyDeviceToHost, c->cs));
    if (op) CK(cudaMemcpyAsync(op + ho, c->parent + so, size_t(n) * 4, cudaMemcpyDeviceToHost, c->cs));
    if (od) CK(cudaMemcpyAsync(od + ho, c->depth + so, size_t(n) * 4, cudaMemcpyDeviceToHost, c->cs));
    if (os) CK(cudaMemcpyAsync(os + ho, c->score + so, size_t(n) * 4, cudaMemcpyDeviceToHost, c->cs));
  }
  if (ot || op || od || os) CK(cudaStreamSynchronize(c->cs));
  return SS_OK;
}

static ss_status verify_impl(ss_ctx* c) {
  NvtxRange nvtx_range("ss.verify_tree", 0xFFC0392Bu);
  if (c->state != ST_DRAFTED) return fail(c, SS_ERR_STRUCTURE, "verify_tree before draft_tree");
  ss_status s = do_verify(c);
  if (s != SS_OK) return s;
  CK(cudaEventRecord(c->e2, c->cs));
  c->state = ST_VERIFIED;
  return SS_OK;
}

ss_status ss_verify_tree(ss_ctx* c, int32_t* opt_argmax, float* opt_gap) {
  GUARD(c);
  ss_status s = verify_impl(c);
  if (s != SS_OK) return s;
  const size_t nn = size_t(c->B) * c->n_nodes;   // batched: [B][n_nodes], request-major rows
  if (opt_argmax) CK(cudaMemcpyAsync(opt_argmax, c->argmax, nn * 4, cudaMemcpyDeviceToHost, c->cs));
  if (opt_gap) CK(cudaMemcpyAsync(opt_gap, c->gap, nn * 4, cudaMemcpyDeviceToHost, c->cs));
  if (opt_argmax || opt_gap) CK(cudaStreamSynchronize(c->cs));
  return SS_OK;
}

// out_tokens/opt_path: [B][stride] (stride >= D_eff + 1), out_n: [B]
static ss_status accept_impl(ss_ctx* c, int32_t* out_tokens, int32_t* out_n, int32_t* opt_path, int stride) {
  NvtxRange nvtx_range("ss.accept_and_commit", 0xFF27AE60u);
  if (c->state != ST_VERIFIED) return fail(c, SS_ERR_STRUCTURE, "accept before verify");
  ss_status s = do_accept(c, false);
  if (s != SS_OK) return s;
  CK(cudaEventRecord(c->e3, c->cs));
  const int cap = c->cur_deff + 1;
  int total = 0;
  if (c->B == 1) {
    int32_t n = 0;
    if ((s = read_outputs(c, cap, out_tokens, &n, opt_path)) != SS_OK) return s;
    if (out_n) *out_n = n;
    c->Pb[0] += n;
    total = n;
  } else {
    // every slot's count and tokens in two copies (outputs are [B][max_nodes + 1] on the device)
    const int os = c->max_nodes + 1, B = c->B;
    int* hn = c->h_out;
    int* ht = c->h_out + B;
    CK(cudaMemcpyAsync(hn, c->out_n, size_t(B) * 4, cudaMemcpyDeviceToHost, c->cs));
    CK(cudaMemcpyAsync(ht, c->out_tokens, size_t(B) * os * 4, cudaMemcpyDeviceToHost, c->cs));
    if (opt_path) CK(cudaMemcpyAsync(ht + size_t(B) * os, c->out_path, size_t(B) * os * 4, cudaMemcpyDeviceToHost, c->cs));
    CK(cudaStreamSynchronize(c->cs));
    for (int b = 0; b < B; ++b) {
      const int n = hn[b];
      if (out_n) out_n[b] = n;
      if (out_tokens) std::memcpy(out_tokens + size_t(b) * stride, ht + size_t(b) * os, size_t(std::min(n, cap)) * 4);
      if (opt_path)
        std::memcpy(opt_path + size_t(b) * stride, ht + size_t(B) * os + size_t(b) * os, size_t(std::min(n, cap)) * 4);
      c->Pb[b] += n;
      total += n;
    }
  }
  c->P = c->Pb[0];
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, c->e0, c->e1) == cudaSuccess) c->st.draft_ms += ms;
  if (cudaEventElapsedTime(&ms, c->e1, c->e2) == cudaSuccess) c->st.verify_ms += ms;
  if (cudaEventElapsedTime(&ms, c->e2, c->e3) == cudaSuccess) c->st.accept_ms += ms;
  cudaGetLastError();
  c->st.steps++;
  c->st.tokens_emitted += total;
  c->st.committed_len = c->P;
  c->st.gpu_launches = c->launches;
  harvest_timing(c);
  c->state = ST_SESSION;
  return SS_OK;
}

ss_status ss_accept_and_commit(ss_ctx* c, int32_t* out_tokens, int32_t* out_n, int32_t* opt_path) {
  GUARD(c);
  return accept_impl(c, out_tokens, out_n, opt_path, c->cur_deff + 1);
}

ss_status ss_step(ss_ctx* c, const ss_draft_params* p, int32_t* out_tokens, int32_t* out_n) {
  GUARD(c);
  if (c->B != 1) return fail(c, SS_ERR_STRUCTURE, "ss_step is the one-request step; use ss_step_batch");
  ss_status s = draft_impl(c, -1, p);
  if (s != SS_OK) return s;
  if ((s = verify_impl(c)) != SS_OK) return s;
  return accept_impl(c, out_tokens, out_n, nullptr, c->cur_deff + 1);
}

ss_status ss_step_batch(ss_ctx* c, const ss_draft_params* p, int32_t stride, int32_t* out_tokens, int32_t* out_n) {
  GUARD(c);
  if (!p || !out_tokens || !out_n || stride < p->depth + 1) return fail(c, SS_ERR_INVALID, "step_batch args");
  ss_status s = draft_impl(c, -1, p);
  if (s != SS_OK) return s;
  if ((s = verify_impl(c)) != SS_OK) return s;
  return accept_impl(c, out_tokens, out_n, nullptr, stride);
}

ss_status ss_generate(ss_ctx* c, const int32_t* prompt, int32_t n, int32_t max_new, int32_t chunk,
                      const ss_draft_params* p, int32_t* out_tokens, int32_t* out_n, int32_t* tau_hist) {
  GUARD(c);
  if (!p || !out_tokens || max_new < 1) return fail(c, SS_ERR_INVALID, "generate args");
  if (c->state == ST_DRAFTED || c->state == ST_VERIFIED) return fail(c, SS_ERR_STRUCTURE, "generate inside a step");
  if (c->B != 1) return fail(c, SS_ERR_STRUCTURE, "ss_generate is the one-request loop; use ss_generate_batch");
  int32_t first = 0;
  ss_status s = ss_prefill(c, prompt, n, chunk, &first);
  if (s != SS_OK) return s;
  int produced = 0;
  out_tokens[produced++] = first;
  std::vector<int32_t> buf(size_t(c->lim.max_depth) + 2);
  ss_draft_params q = *p;
  const bool ar = p->depth == 0;
  if (ar) {
    q.depth = 0;
    q.top_k = 1;
  }
  while (produced < max_new) {
    if (c->P + 1 > c->C) break;
    int32_t m = 0;
    if ((s = ss_step(c, &q, buf.data(), &m)) != SS_OK) return s;
    if (tau_hist && m >= 0 && m <= p->depth + 1) tau_hist[m]++;
    for (int i = 0; i < m && produced < max_new; ++i) out_tokens[produced++] = buf[i];
  }
  if (out_n) *out_n = produced;
  return SS_OK;
}

ss_status ss_generate_batch(ss_ctx* c, int32_t n_req, const int32_t* prompts, const int32_t* prompt_lens,
                            int32_t max_new, int32_t chunk, const ss_draft_params* p, int32_t* out_tokens,
                            int32_t* out_n, int32_t* tau_hist) {
  GUARD(c);
  if (!p || !prompts || !prompt_lens || !out_tokens || !out_n || max_new < 1)
    return fail(c, SS_ERR_INVALID, "generate_batch args");
  ss_status s = ss_set_batch(c, n_req);
  if (s != SS_OK) return s;
  std::vector<int> produced(size_t(n_req), 0);
  int64_t off = 0;
  for (int b = 0; b < n_req; ++b) {
    int32_t first = 0;
    if ((s = prefill_slot_impl(c, b, prompts + off, prompt_lens[b], chunk, &first)) != SS_OK) return s;
    off += prompt_lens[b];
    out_tokens[size_t(b) * max_new] = first;
    produced[b] = 1;
  }
  ss_draft_params q = *p;
  if (p->depth == 0) q.top_k = 1;
  const int stride = q.depth + 1;
  std::vector<int32_t> buf(size_t(n_req) * stride);
  std::vector<int32_t> m(static_cast<size_t>(n_req));
  // every slot steps until the slowest one has max_new tokens (the others' surplus is dropped)
  while (*std::min_element(produced.begin(), produced.end()) < max_new) {
    int Pmax = 0;
    for (int b = 0; b < n_req; ++b) Pmax = std::max(Pmax, c->Pb[b]);
    if (Pmax + 1 > c->C) break;
    if ((s = ss_step_batch(c, &q, stride, buf.data(), m.data())) != SS_OK) return s;
    for (int b = 0; b < n_req; ++b) {
      if (produced[b] >= max_new) continue;
      if (tau_hist && m[b] >= 0 && m[b] <= p->depth + 1) tau_hist[m[b]]++;
      for (int i = 0; i < m[b] && produced[b] < max_new; ++i) out_tokens[size_t(b) * max_new + produced[b]++] = buf[size_t(b) * stride + i];
    }
  }
  for (int b = 0; b < n_req; ++b) out_n[b] = produced[b];
  return SS_OK;
}

ss_status ss_get_stats(ss_ctx* c, ss_stats* out) {
  if (!c || !out) return SS_ERR_INVALID;
  harvest_timing(c);
  c->st.gpu_launches = c->launches;
  *out = c->st;
  return SS_OK;
}

ss_status ss_reset_stats(ss_ctx* c) {
  if (!c) return SS_ERR_INVALID;
  harvest_timing(c);
  // copies still in flight count only from here on (the stats region starts on the compute stream now)
  cudaEventRecord(c->ev_region, c->cs);
  c->region_set = true;
  const ss_stats keep = c->st;
  c->st = ss_stats{};
  c->st.arena_used = keep.arena_used;
  c->st.arena_cap = keep.arena_cap;
  c->st.ring_bytes = keep.ring_bytes;
  c->st.host_pinned_bytes = keep.host_pinned_bytes;
  c->st.substitute_bytes = keep.substitute_bytes;
  c->st.n_resident = keep.n_resident;
  c->st.n_offloaded = keep.n_offloaded;
  c->st.committed_len = keep.committed_len;
  c->launches = 0;
  return SS_OK;
}

const char* ss_last_error(ss_ctx* c) { return c ? c->err.c_str() : "null context"; }

void ss_destroy(ss_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  if (c->dbg_mem) cudaFree(c->dbg_mem);
  for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
  for (auto e : c->ev_copied) cudaEventDestroy(e);
  for (auto e : c->ev_consumed) cudaEventDestroy(e);
  for (auto e : c->ev_t0) cudaEventDestroy(e);
  for (auto e : c->ev_t1) cudaEventDestroy(e);
  for (auto e : {c->e0, c->e1, c->e2, c->e3, c->ev_root, c->ev_ref, c->ev_region})
    if (e) cudaEventDestroy(e);
  for (void* b : c->ipc_opened) cudaIpcCloseMemHandle(b);
  if (c->h_root) cudaFreeHost(c->h_root);
  if (c->host && c->host_external) host_unregister(c->host);
  else if (c->host) cudaFreeHost(c->host);
  if (c->h_embed) cudaFreeHost(c->h_embed);
  if (c->h_out) cudaFreeHost(c->h_out);
  cudaGetLastError();
  delete c;
}

// ------------------------- NEXT-1: cooperative weight streaming -----------------------------
namespace {
struct CoopBlob {
  uint32_t magic, version;
  int32_t pid, device;
  uint64_t ring_off, flags_off, ring_bytes, n_items, host_bytes, cycle_bytes;
  uint64_t ring_ptr, flags_ptr;
  cudaIpcMemHandle_t ipc;
};
constexpr uint32_t kCoopMagic = 0x53534350u;   // "SSCP"
static_assert(sizeof(CoopBlob) <= sizeof(ss_coop_handle), "coop handle size");
}  // namespace

ss_status ss_coop_export(ss_ctx* c, ss_coop_handle* out) {
  GUARD(c);
  if (!out) return fail(c, SS_ERR_INVALID, "coop_export: null handle");
  if (c->state < ST_READY || c->state == ST_DRAFTED || c->state == ST_VERIFIED)
    return fail(c, SS_ERR_STRUCTURE, "coop_export: after build_substitutes, outside a step");
  if (c->cycle.empty() || c->f32 || c->serial_stream || c->coop_world > 1)
    return fail(c, SS_ERR_STRUCTURE, "coop_export: needs streamed layers, bf16, async streaming, not yet enabled");
  if (!load_driver_fns()) return fail(c, SS_ERR_CUDA, "coop_export: stream memory operations unavailable");
  CK(cudaMemsetAsync(c->flags, 0, 2 * kCoopMax * 4, c->cs));
  CK(cudaStreamSynchronize(c->cs));
  CUdeviceptr base = 0;
  size_t size = 0;
  CKD(g_range(&base, &size, (CUdeviceptr)c->ar.base));
  CoopBlob b{};
  b.magic = kCoopMagic;
  b.version = 1;
  b.pid = int32_t(getpid());
  b.device = c->device;
  b.ring_off = uint64_t(reinterpret_cast<uintptr_t>(c->ring) - base);
  b.flags_off = uint64_t(reinterpret_cast<uintptr_t>(c->flags) - base);
  b.ring_bytes = c->ring_bytes;
  b.n_items = c->cycle.size();
  b.host_bytes = c->host_bytes;
  for (auto& lg : c->cycle) b.cycle_bytes += c->lw[lg.first].host_used[lg.second];
  b.ring_ptr = uint64_t(reinterpret_cast<uintptr_t>(c->ring));
  b.flags_ptr = uint64_t(reinterpret_cast<uintptr_t>(c->flags));
  CK(cudaIpcGetMemHandle(&b.ipc, c->ar.base));
  std::memset(out, 0, sizeof(*out));
  std::memcpy(out, &b, sizeof(b));
  c->coop_exported = true;
  return SS_OK;
}

ss_status ss_coop_enable(ss_ctx* c, int32_t rank, int32_t world, const ss_coop_handle* all) {
  GUARD(c);
  if (!all || world < 2 || world > kCoopMax || rank < 0 || rank >= world)
    return fail(c, SS_ERR_INVALID, "coop_enable: rank/world/handles");
  if (!c->coop_exported || c->coop_world > 1) return fail(c, SS_ERR_STRUCTURE, "coop_enable: export first, once");
  if (c->state == ST_DRAFTED || c->state == ST_VERIFIED) return fail(c, SS_ERR_STRUCTURE, "coop_enable inside a step");
  if (c->next_consume % int64_t(c->cycle.size()) != 0) return fail(c, SS_ERR_STRUCTURE, "coop_enable: mid-pass");
  std::vector<CoopBlob> bl(world);
  for (int h = 0; h < world; ++h) std::memcpy(&bl[h], &all[h], sizeof(CoopBlob));
  for (int h = 0; h < world; ++h) {
    if (bl[h].magic != kCoopMagic || bl[h].version != 1) return fail(c, SS_ERR_INVALID, "coop_enable: bad handle");
    if (bl[h].ring_bytes != c->ring_bytes || bl[h].n_items != c->cycle.size() || bl[h].host_bytes != c->host_bytes ||
        bl[h].cycle_bytes != bl[rank].cycle_bytes) {
      char msg[320];
      std::snprintf(msg, sizeof msg,
                    "coop_enable: rank %d differs in model, placement or ring (ring %llu/%llu items %llu/%zu host %llu/%zu "
                    "cycle %llu/%llu)", h, (unsigned long long)bl[h].ring_bytes, (unsigned long long)c->ring_bytes,
                    (unsigned long long)bl[h].n_items, c->cycle.size(), (unsigned long long)bl[h].host_bytes, c->host_bytes,
                    (unsigned long long)bl[h].cycle_bytes, (unsigned long long)bl[rank].cycle_bytes);
      return fail(c, SS_ERR_INVALID, msg);
    }
  }
  if (bl[rank].ring_ptr != uint64_t(reinterpret_cast<uintptr_t>(c->ring)))
    return fail(c, SS_ERR_INVALID, "coop_enable: handle `rank` is not this context's");
  // drain the non-cooperative stream: every prefetched item is dropped, the ring restarts at 0
  CK(cudaStreamSynchronize(c->cs));
  CK(cudaStreamSynchronize(c->xs));
  harvest_timing(c);
  c->inflight.clear();
  c->placed.clear();
  c->ring_head = 0;
  c->next_issue = c->next_consume = 0;
  c->peer_ring.assign(world, nullptr);
  c->peer_flags.assign(world, nullptr);
  for (int h = 0; h < world; ++h) {
    if (h == rank) {
      c->peer_ring[h] = c->ring;
      c->peer_flags[h] = c->flags;
      continue;
    }
    uint8_t* base = nullptr;
    if (bl[h].pid == int32_t(getpid())) {   // another context of this process: its pointers as they are
      c->peer_ring[h] = reinterpret_cast<uint8_t*>(uintptr_t(bl[h].ring_ptr));
      c->peer_flags[h] = reinterpret_cast<uint32_t*>(uintptr_t(bl[h].flags_ptr));
      continue;
    }
    void* vb = nullptr;
    CK(cudaIpcOpenMemHandle(&vb, bl[h].ipc, cudaIpcMemLazyEnablePeerAccess));
    c->ipc_opened.push_back(vb);
    base = reinterpret_cast<uint8_t*>(vb);
    c->peer_ring[h] = base + bl[h].ring_off;
    c->peer_flags[h] = reinterpret_cast<uint32_t*>(base + bl[h].flags_off);
  }
  c->coop_world = world;
  c->coop_rank = rank;
  return SS_OK;   // streaming resumes at the next target pass (after the caller's barrier)
}

ss_status ss_coop_finish(ss_ctx* c) {
  GUARD(c);
  if (c->coop_world < 2) return fail(c, SS_ERR_STRUCTURE, "coop_finish: cooperative streaming not enabled");
  if (c->state == ST_DRAFTED || c->state == ST_VERIFIED) return fail(c, SS_ERR_STRUCTURE, "coop_finish inside a step");
  // release every peer's pending ring writes into this rank (they wait for our consumption), then
  // wait for our own pending pushes, which the peers release the same way
  for (int h = 0; h < c->coop_world; ++h)
    if (h != c->coop_rank)
      CKD(g_write32((CUstream)c->cs, (CUdeviceptr)(c->peer_flags[h] + kCoopMax + c->coop_rank), 0x7fffffffu, 0));
  CK(cudaStreamSynchronize(c->cs));
  CK(cudaStreamSynchronize(c->xs));
  harvest_timing(c);
  c->inflight.clear();
  c->placed.clear();
  c->ring_head = 0;
  c->next_issue = c->next_consume = 0;
  for (void* b : c->ipc_opened) CK(cudaIpcCloseMemHandle(b));
  c->ipc_opened.clear();
  c->peer_ring.clear();
  c->peer_flags.clear();
  c->coop_world = 1;
  c->coop_rank = 0;
  c->coop_exported = false;   // a new cooperative epoch starts with ss_coop_export again
  return SS_OK;   // streaming resumes alone at the next target pass (after the caller's barrier)
}

// ---------------------------------- debug ---------------------------------------------------
static ss_status drain_stream(ss_ctx* c) {
  CK(cudaStreamSynchronize(c->cs));
  CK(cudaStreamSynchronize(c->xs));
  return SS_OK;
}

ss_status ss_debug_gen_tensor(ss_ctx* c, uint64_t seed, int32_t tid, int64_t rows, int64_t cols, int32_t kind,
                              double sigma, uint16_t* out) {
  GUARD(c);
  if (!out || rows < 1 || cols < 1) return fail(c, SS_ERR_INVALID, "gen_tensor args");
  if (c->state != ST_CREATED && c->state < ST_READY) return fail(c, SS_ERR_STRUCTURE, "gen_tensor needs a free ring");
  const size_t bytes = size_t(rows) * cols * 2;
  uint8_t* buf = c->ring ? c->ring : c->ar.base + c->ar.used;
  const size_t room = c->ring ? c->ring_bytes : c->ar.cap - c->ar.used;
  if (bytes > room) return fail(c, SS_ERR_BUDGET, "gen_tensor: tensor larger than free arena");
  if (c->ring && !c->inflight.empty()) {   // ring busy with prefetches: drain them first
    CK(cudaStreamSynchronize(c->xs));
    return fail(c, SS_ERR_STRUCTURE, "gen_tensor: ring in use by streaming");
  }
  launch_gen_natural(reinterpret_cast<uint16_t*>(buf), tensor_key(seed, uint64_t(tid)), uint64_t(rows) * cols,
                     scale_c32(sigma), kind == 1, c->cs);
  CK(cudaMemcpyAsync(out, buf, bytes, cudaMemcpyDeviceToHost, c->cs));
  CK(cudaStreamSynchronize(c->cs));
  return check_launch(c, "gen_tensor");
}

ss_status ss_debug_read_group(ss_ctx* c, int32_t layer, int32_t group, uint16_t* out) {
  GUARD(c);
  if (c->state < ST_LOADED || layer < 0 || layer >= c->L || group < 0 || group > 3 || !out)
    return fail(c, SS_ERR_INVALID, "read_group args");
  const int N = c->gN[group], K = c->gK[group];
  const LayerW& w = c->lw[layer];
  ss_status s = drain_stream(c);
  if (s != SS_OK) return s;
  // tiled source: resident buffer, or the host store copied to the device
  uint8_t* src = w.resident ? w.bf16[group] : nullptr;
  std::vector<uint8_t> tmp;
  if (!w.resident) {
    tmp.resize(bf16_bytes(N, K));
    if (w.zmode[group] < 0) std::memcpy(tmp.data(), c->host + w.host_off[group], tmp.size());
    else zdecode_host(c->host + w.host_off[group], reinterpret_cast<uint16_t*>(tmp.data()));   // the K7 codec's blob
  } else {
    tmp.resize(bf16_bytes(N, K));
    CK(cudaMemcpyAsync(tmp.data(), src, tmp.size(), cudaMemcpyDeviceToHost, c->cs));
    CK(cudaStreamSynchronize(c->cs));
  }
  for (int64_t n = 0; n < N; ++n)
    for (int64_t k = 0; k < K; ++k)
      std::memcpy(out + n * K + k, tmp.data() + bf16_tiled_offset(n, k, K), 2);
  return SS_OK;
}

ss_status ss_debug_decode_group(ss_ctx* c, int32_t layer, int32_t group, uint16_t* out, int32_t* out_mode,
                                uint64_t* out_stream_bytes) {
  GUARD(c);
  if (c->state < ST_LOADED || layer < 0 || layer >= c->L || group < 0 || group > 3 || !out || c->lw[layer].resident)
    return fail(c, SS_ERR_INVALID, "decode_group args (an offloaded group)");
  const LayerW& w = c->lw[layer];
  const int N = c->gN[group], K = c->gK[group];
  const int64_t n = int64_t(N) * K;
  ss_status s = drain_stream(c);
  if (s != SS_OK) return s;
  if (c->ring && !c->inflight.empty()) return fail(c, SS_ERR_STRUCTURE, "decode_group: ring in use by streaming");
  // the blob as streamed (H2D into the ring), decoded by the GPU kernel the verify uses
  uint8_t* blob = c->ring + (size_t(n) * 2 + 4095) / 4096 * 4096;
  const uint16_t* tiles = reinterpret_cast<const uint16_t*>(c->ring);
  if (w.zmode[group] < 0) {
    CK(cudaMemcpyAsync(c->ring, c->host + w.host_off[group], size_t(n) * 2, cudaMemcpyHostToDevice, c->cs));
  } else {
    CK(cudaMemcpyAsync(blob, c->host + w.host_off[group], w.host_used[group], cudaMemcpyHostToDevice, c->cs));
    if (w.zmode[group] == 1) launch_zdecode(blob, reinterpret_cast<uint16_t*>(c->ring), n, c->cs);
    else tiles = reinterpret_cast<const uint16_t*>(blob + w.host_a0[group]);
  }
  std::vector<uint8_t> tmp(size_t(n) * 2);
  CK(cudaMemcpyAsync(tmp.data(), tiles, tmp.size(), cudaMemcpyDeviceToHost, c->cs));
  CK(cudaStreamSynchronize(c->cs));
  for (int64_t r = 0; r < N; ++r)
    for (int64_t k = 0; k < K; ++k) std::memcpy(out + r * K + k, tmp.data() + bf16_tiled_offset(r, k, K), 2);
  if (out_mode) *out_mode = w.zmode[group];
  if (out_stream_bytes) *out_stream_bytes = w.host_used[group];
  return check_launch(c, "decode_group");
}

ss_status ss_debug_get_substitute(ss_ctx* c, int32_t layer, int32_t group, uint8_t* codes, uint16_t* s, uint16_t* z) {
  GUARD(c);
  if (c->state < ST_READY || layer < 0 || layer >= c->L || group < 0 || group > 3 || c->lw[layer].resident)
    return fail(c, SS_ERR_INVALID, "get_substitute: not an offloaded layer (or substitutes not built)");
  const int N = c->gN[group], K = c->gK[group];
  const bool q2 = c->sub_bits == 2, q3 = c->sub_bits == 3;
  std::vector<uint8_t> q(sub_bytes(N, K, c->sub_bits));
  CK(cudaMemcpyAsync(q.data(), c->lw[layer].q4[group], q.size(), cudaMemcpyDeviceToHost, c->cs));
  CK(cudaStreamSynchronize(c->cs));
  for (int64_t n = 0; n < N; ++n)
    for (int64_t k = 0; k < K; ++k) {
      uint64_t off;
      int sh;
      if (q3) {
        uint64_t hoff;
        int hbit;
        q3_code_pos(n, k, K, &off, &sh, &hoff, &hbit);
        if (codes) codes[n * K + k] = uint8_t(((q[off] >> sh) & 3) | (((q[hoff] >> hbit) & 1) << 2));
      } else {
        if (q2) q2_code_pos(n, k, K, &off, &sh);
        else q4_code_pos(n, k, K, &off, &sh);
        if (codes) codes[n * K + k] = (q[off] >> sh) & (q2 ? 3 : 15);
      }
      if ((k & 63) == 0) {
        uint32_t m;
        std::memcpy(&m, q.data() + (q2 ? q2_meta_offset(n, k, K) : (q3 ? q3_meta_offset(n, k, K) : q4_meta_offset(n, k, K))), 4);
        if (s) s[n * (K / 64) + k / 64] = uint16_t(m & 0xFFFF);
        if (z) z[n * (K / 64) + k / 64] = uint16_t(m >> 16);
      }
    }
  return SS_OK;
}

// debug scratch (ss_debug_* only): allocated once, outside the arena, so the product path's VRAM cap
// holds no test-only buffer
static ss_status ensure_debug_bufs(ss_ctx* c) {
  if (c->dbg_mem) return SS_OK;
  const size_t lg = c->logits ? 0 : size_t(32) * c->V * 4;
  const size_t ao = (c->at_o_floats * 4 + 255) / 256 * 256;
  if (cudaMalloc(&c->dbg_mem, ao + lg) != cudaSuccess) {
    cudaGetLastError();
    c->dbg_mem = nullptr;
    return fail(c, SS_ERR_BUDGET, "debug scratch: device allocation failed");
  }
  c->at_o = reinterpret_cast<float*>(c->dbg_mem);
  if (!c->logits) c->logits = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(c->dbg_mem) + ao);
  return SS_OK;
}

ss_status ss_debug_matmul(ss_ctx* c, int32_t which, int32_t layer, int32_t group, const uint16_t* x, int32_t M, float* y) {
  GUARD(c);
  if (ensure_debug_bufs(c) != SS_OK) return SS_ERR_BUDGET;
  if (c->state < ST_READY || layer < 0 || layer >= c->L || group < 0 || group > 3 || !x || !y || M < 1)
    return fail(c, SS_ERR_INVALID, "debug_matmul args");
  if (which == 0 && M > 32) return fail(c, SS_ERR_INVALID, "draft GEMV: M <= 32");
  if (which == 1 && M > c->mpad_max) return fail(c, SS_ERR_INVALID, "target GEMM: M too large");
  const int N = c->gN[group], K = c->gK[group];
  const int NT = which == 0 ? gemv_nt(M) : gemm_nt(M);
  ss_status s = drain_stream(c);
  if (s != SS_OK) return s;
  // X -> FragX (host side), into hfrag/actfrag scratch
  std::vector<uint16_t> fx(size_t(NT) * 8 * K, 0);
  for (int m = 0; m < M; ++m)
    for (int k = 0; k < K; ++k) fx[fragx_offset(m, k, NT)] = x[int64_t(m) * K + k];
  uint16_t* X = K == c->F ? c->actfrag : c->hfrag;
  float* XS = K == c->F ? c->actxs : c->hxs;
  std::vector<float> xs(size_t(K / 64) * NT * 8, 0.f);
  for (int m = 0; m < M; ++m)
    for (int k = 0; k < K; ++k) {
      uint32_t b = uint32_t(x[int64_t(m) * K + k]) << 16;
      float f;
      std::memcpy(&f, &b, 4);
      xs[size_t(k / 64) * NT * 8 + m] += f;
    }
  CK(cudaMemcpyAsync(X, fx.data(), fx.size() * 2, cudaMemcpyHostToDevice, c->cs));
  if (which == 0) CK(cudaMemcpyAsync(XS, xs.data(), xs.size() * 4, cudaMemcpyHostToDevice, c->cs));
  float* Y = c->at_o;   // debug output scratch: the attention partial buffer
  if (size_t(M) * N > c->at_o_floats) return fail(c, SS_ERR_BUDGET, "debug_matmul: output too large");
  EpiParams e = base_epi(c, M);
  e.kind = EPI_STORE;
  e.out = Y;
  e.ldo = N;
  const LayerW& w = c->lw[layer];
  if (which == 0) {
    GemvParams p{};
    p.W = w.resident ? w.bf16[group] : w.q4[group];
    p.X = X;
    p.XS = XS;
    p.N = N;
    p.K = K;
    p.NT = NT;
    p.partials = c->gv_part;
    p.counters = c->gv_cnt;
    p.max_seg = gemv_max_segments(N, K, gemv_streamk_grid(!w.resident, N, K, c->gv_grid));
    p.epi = e;
    p.qbits = c->sub_bits;
    p.ctas_per_sm = (group == 0 && !w.resident) ? 1 : 0;   // the draft pass's plan (matmul)
    launch_gemv(!w.resident, p, c->gv_grid, false, c->cs);
  } else {
    GemmParams p{};
    p.X = X;
    p.N = N;
    p.K = K;
    p.NT = NT;
    p.epi = e;
    if (w.resident) {
      p.W = w.bf16[group];
    } else {
      return fail(c, SS_ERR_STRUCTURE, "debug target matmul on an offloaded layer: use a resident layer");
    }
    launch_gemm(p, false, c->cs, c->k6_variant);
  }
  CK(cudaMemcpyAsync(y, Y, size_t(M) * N * 4, cudaMemcpyDeviceToHost, c->cs));
  CK(cudaStreamSynchronize(c->cs));
  return check_launch(c, "debug_matmul");
}

ss_status ss_debug_time_matmul(ss_ctx* c, int32_t which, int32_t layer, int32_t group, int32_t M, int32_t iters,
                               float* out_ms) {
  GUARD(c);
  if (ensure_debug_bufs(c) != SS_OK) return SS_ERR_BUDGET;
  // layer >= 0: that layer only; layer == -1: every layer in turn (weights stream from HBM, not L2).
  // group 0..3: that matrix group; -1: the bf16 head; -2: the four groups of each layer in pass order.
  // which 0: the draft GEMV (K2 / bf16 head), M <= 32; which 1: the target GEMM (K6) on resident
  // layers (EPI_STORE) or the head (group -1, EPI_ARGMAX as in the verify), M <= the verify rows
  if (c->state < ST_READY || which < 0 || which > 1 || layer < -1 || layer >= c->L || group < -2 || group > 3 || M < 1 ||
      M > (which == 0 ? 32 : c->mpad_max) || iters < 1 || !out_ms)
    return fail(c, SS_ERR_INVALID, "time_matmul args");
  std::vector<std::pair<int, int>> seq;
  for (int l = (layer < 0 ? 0 : layer); l < (layer < 0 ? c->L : layer + 1); ++l) {
    if (group == -2)
      for (int g = 0; g < 4; ++g) seq.emplace_back(l, g);
    else
      seq.emplace_back(l, group);
  }
  if (group == -1) seq.assign(1, {0, -1});
  if (which == 1)
    for (auto& lg : seq)
      if (lg.second >= 0 && (!c->lw[lg.first].resident || size_t(M) * c->gN[lg.second] > c->at_o_floats))
        return fail(c, SS_ERR_STRUCTURE, "time_matmul: the target GEMM is timed on resident layers");
  auto launch = [&](int l, int g) {
    const bool head = g == -1;
    const int N = head ? c->V : c->gN[g], K = head ? c->H : c->gK[g];
    const LayerW& w = c->lw[l];
    if (which == 1) {
      GemmParams q{};
      q.W = head ? c->head : w.bf16[g];
      q.X = K == c->F ? c->actfrag : c->hfrag;
      q.N = N;
      q.K = K;
      q.NT = gemm_nt(M);
      q.epi = base_epi(c, M);
      if (head) {
        q.epi.kind = EPI_ARGMAX;
        q.epi.am_val = c->am_val;
        q.epi.am_idx = c->am_idx;
        q.epi.am_second = c->am_sec;
        q.epi.am_tiles = c->vtiles;
      } else {
        q.epi.kind = EPI_STORE;
        q.epi.out = c->at_o;
        q.epi.ldo = N;
      }
      launch_gemm(q, c->use_pdl, c->cs, c->k6_variant);
      return;
    }
    GemvParams p{};
    p.W = head ? c->head : (w.resident ? w.bf16[g] : w.q4[g]);
    p.X = K == c->F ? c->actfrag : c->hfrag;
    p.XS = K == c->F ? c->actxs : c->hxs;
    p.N = N;
    p.K = K;
    p.NT = gemv_nt(M);
    p.partials = c->gv_part;
    p.counters = c->gv_cnt;
    p.max_seg = gemv_max_segments(N, K, gemv_streamk_grid(!head && !w.resident, N, K, c->gv_grid));
    p.epi = base_epi(c, M);
    p.epi.kind = EPI_STORE;
    p.ctas_per_sm = (!head && g == 0 && !w.resident) ? 1 : 0;   // the draft pass's plan (matmul)
    p.qbits = c->sub_bits;
    p.epi.out = c->at_o;
    p.epi.ldo = N;
    launch_gemv(!head && !w.resident, p, c->gv_grid, c->use_pdl, c->cs);
  };
  ss_status s = drain_stream(c);
  if (s != SS_OK) return s;
  for (auto& lg : seq) launch(lg.first, lg.second);   // warm-up (attributes, instruction cache)
  CK(cudaEventRecord(c->e0, c->cs));
  for (int i = 0; i < iters; ++i)
    for (auto& lg : seq) launch(lg.first, lg.second);
  CK(cudaEventRecord(c->e1, c->cs));
  CK(cudaEventSynchronize(c->e1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, c->e0, c->e1));
  *out_ms = ms / float(iters * seq.size());
  return check_launch(c, "time_matmul");
}

ss_status ss_debug_set_knob(ss_ctx* c, int32_t knob, int32_t value) {
  GUARD(c);
  switch (knob) {
    case 2: c->k6_variant = value; break;
    default: return fail(c, SS_ERR_INVALID, "unknown knob");
  }
  CK(cudaStreamSynchronize(c->cs));
  for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
  c->graphs.clear();   // captured graphs hold the old launch parameters
  c->graph_launches.clear();
  return SS_OK;
}

ss_status ss_debug_time_pass(ss_ctx* c, int32_t M, int32_t iters, int32_t skip, float* out_ms) {
  GUARD(c);
  if (ensure_debug_bufs(c) != SS_OK) return SS_ERR_BUDGET;
  if (c->state != ST_SESSION || M < 1 || M > std::min(32, c->max_nodes - 1) || iters < 1 || !out_ms)
    return fail(c, SS_ERR_INVALID, "time_pass args");
  // draft forward of M frontier nodes (slots 1..M, children of the root), repeated; tree metadata
  // is set up host-side first.  Writes tree KV scratch only.
  std::vector<int> tk(M + 1), par(M + 1), dep(M + 1), anc(size_t(M + 1) * c->anc_stride, 0);
  std::vector<float> sc(M + 1, 0.f);
  for (int i = 0; i <= M; ++i) {
    tk[i] = (i * 7919) % c->V;
    par[i] = i ? 0 : -1;
    dep[i] = i ? 1 : 0;
    anc[size_t(i) * c->anc_stride] = 0;
    if (i) anc[size_t(i) * c->anc_stride + 1] = i;
  }
  CK(cudaMemcpyAsync(c->tok, tk.data(), tk.size() * 4, cudaMemcpyHostToDevice, c->cs));
  CK(cudaMemcpyAsync(c->parent, par.data(), par.size() * 4, cudaMemcpyHostToDevice, c->cs));
  CK(cudaMemcpyAsync(c->depth, dep.data(), dep.size() * 4, cudaMemcpyHostToDevice, c->cs));
  CK(cudaMemcpyAsync(c->score, sc.data(), sc.size() * 4, cudaMemcpyHostToDevice, c->cs));
  CK(cudaMemcpyAsync(c->anc, anc.data(), anc.size() * 4, cudaMemcpyHostToDevice, c->cs));
  CK(cudaStreamSynchronize(c->cs));
  g_skip = skip;
  PassOut o;
  o.logits = true;
  auto one = [&]() { return forward_pass(c, false, M, 1, o); };
  ss_status s = one();   // warm-up
  if (s == SS_OK) {
    CK(cudaEventRecord(c->e0, c->cs));
    for (int i = 0; i < iters && s == SS_OK; ++i) s = one();
    CK(cudaEventRecord(c->e1, c->cs));
  }
  g_skip = 0;
  if (s != SS_OK) return s;
  CK(cudaEventSynchronize(c->e1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, c->e0, c->e1));
  *out_ms = ms / iters;
  return check_launch(c, "time_pass");
}

ss_status ss_debug_trace_pass(ss_ctx* c, int32_t M, int64_t* out, int32_t cap, int32_t* out_n) {
  GUARD(c);
  if (ensure_debug_bufs(c) != SS_OK) return SS_ERR_BUDGET;
  if (c->state != ST_SESSION || !out || cap < 1 || !out_n) return fail(c, SS_ERR_INVALID, "trace_pass args");
  // run one draft pass with %globaltimer events recorded in every dequant-GEMV launch
  float ms = 0.f;
  ss_status s = ss_debug_time_pass(c, M, 1, 0, &ms);   // sets up the frontier + warm-up
  if (s != SS_OK) return s;
  if (cap > 512) cap = 512;
  constexpr int E = kTraceEvents;
  std::vector<unsigned long long> init(size_t(cap) * E);
  for (int i = 0; i < cap; ++i)
    for (int j = 0; j < E; ++j) init[size_t(i) * E + j] = (j == 0) ? ~0ull : 0ull;
  unsigned long long* buf = c->tracebuf;
  CK(cudaMemcpyAsync(buf, init.data(), init.size() * 8, cudaMemcpyHostToDevice, c->cs));
  CK(cudaStreamSynchronize(c->cs));
  g_trace = buf;
  g_trace_n = 0;
  g_trace_cap = cap;
  PassOut o;
  o.logits = true;
  int n;
  s = forward_pass(c, false, M, 1, o);
  n = g_trace_n;
  g_trace = nullptr;
  if (s != SS_OK) return s;
  CK(cudaMemcpyAsync(init.data(), buf, size_t(n) * E * 8, cudaMemcpyDeviceToHost, c->cs));
  CK(cudaStreamSynchronize(c->cs));
  std::memcpy(out, init.data(), size_t(n) * E * 8);
  *out_n = n;
  return SS_OK;
}

ss_status ss_debug_step_timeline(ss_ctx* c, const ss_draft_params* dp, double* out, int32_t cap, int32_t* out_n,
                                 double* out_phases) {
  GUARD(c);
  if (!dp || !out || cap < 1 || !out_n || !out_phases) return fail(c, SS_ERR_INVALID, "step_timeline args");
  if (c->state != ST_SESSION || c->B != 1) return fail(c, SS_ERR_STRUCTURE, "step_timeline: one-request session");
  cudaEvent_t ev0, ev_d, ev_v, ev_a;
  for (cudaEvent_t* e : {&ev0, &ev_d, &ev_v, &ev_a}) CK(cudaEventCreate(e));
  for (auto& kv : c->tl_ev)
    for (cudaEvent_t e : kv.second)
      if (e) cudaEventDestroy(e);
  c->tl_ev.clear();
  c->tl_on = true;
  ss_status s = SS_OK;
  {   // a lead-in step with the events on: the copies that refill the ring during the measured step's
      // draft are issued while the lead-in step's verify releases ring regions
    int32_t toks[1024], n = 0;
    if ((s = draft_impl(c, -1, dp)) == SS_OK && (s = verify_impl(c)) == SS_OK)
      s = accept_impl(c, toks, &n, nullptr, c->cur_deff + 1);
    if (s != SS_OK) {
      c->tl_on = false;
      return s;
    }
  }
  const int64_t seq0 = c->next_consume;
  CK(cudaEventRecord(ev0, c->cs));
  s = draft_impl(c, -1, dp);
  if (s == SS_OK) {
    CK(cudaEventRecord(ev_d, c->cs));
    s = verify_impl(c);
  }
  if (s == SS_OK) {
    CK(cudaEventRecord(ev_v, c->cs));
    int32_t toks[1024], n = 0;
    s = accept_impl(c, toks, &n, nullptr, c->cur_deff + 1);
  }
  c->tl_on = false;
  if (s != SS_OK) return s;
  CK(cudaEventRecord(ev_a, c->cs));
  CK(cudaDeviceSynchronize());
  auto ms = [&](cudaEvent_t e) {
    float t = 0.f;
    if (!e || cudaEventElapsedTime(&t, ev0, e) != cudaSuccess) {
      cudaGetLastError();
      return -1e9;
    }
    return double(t);
  };
  out_phases[0] = ms(ev_d);
  out_phases[1] = ms(ev_v);
  out_phases[2] = ms(ev_a);
  // rows: seq - seq0, layer, group, bytes, copy start, copy end, compute start, ring release (ms from the
  // step start; copies of this verify's first groups were issued during the previous step: negative)
  int k = 0;
  const int n_items = int(c->cycle.size());
  for (auto& kv : c->tl_ev) {
    if (k >= cap) break;
    const int64_t seq = kv.first;
    if (seq < seq0) continue;   // consumed by the lead-in step's verify
    const auto lg = c->cycle[size_t(seq % n_items)];
    double* r = out + size_t(k) * 8;
    r[0] = double(seq - seq0);
    r[1] = lg.first;
    r[2] = lg.second;
    r[3] = double(c->lw[lg.first].host_used[lg.second]);
    for (int j = 0; j < 4; ++j) r[4 + j] = kv.second[j] ? ms(kv.second[j]) : -1e9;
    ++k;
  }
  *out_n = k;
  for (auto& kv : c->tl_ev)
    for (cudaEvent_t e : kv.second)
      if (e) cudaEventDestroy(e);
  c->tl_ev.clear();
  for (cudaEvent_t e : {ev0, ev_d, ev_v, ev_a}) cudaEventDestroy(e);
  return SS_OK;
}

ss_status ss_debug_cta_trace(ss_ctx* c, int32_t M, int32_t launch, int64_t* out, int32_t cap, int32_t* out_n) {
  GUARD(c);
  if (ensure_debug_bufs(c) != SS_OK) return SS_ERR_BUDGET;
  if (c->state != ST_SESSION || !out || cap < 1 || !out_n || launch < 0) return fail(c, SS_ERR_INVALID, "cta_trace args");
  float ms = 0.f;
  ss_status s = ss_debug_time_pass(c, M, 1, 0, &ms);   // frontier set-up + warm-up
  if (s != SS_OK) return s;
  const size_t n = size_t(cap) * 5;
  if (n * 8 > size_t(512) * kTraceEvents * 8) return fail(c, SS_ERR_INVALID, "cta_trace: cap too large");
  CK(cudaMemsetAsync(c->tracebuf, 0, n * 8, c->cs));
  g_cta_trace = c->tracebuf;
  g_cta_launch = launch;
  g_gemv_n = 0;
  PassOut o;
  o.logits = true;
  s = forward_pass(c, false, M, 1, o);
  g_cta_trace = nullptr;
  if (s != SS_OK) return s;
  std::vector<unsigned long long> h(n);
  CK(cudaMemcpyAsync(h.data(), c->tracebuf, n * 8, cudaMemcpyDeviceToHost, c->cs));
  CK(cudaStreamSynchronize(c->cs));
  int k = 0;
  for (int i = 0; i < cap; ++i)
    if (h[size_t(i) * 5 + 1]) k = i + 1;   // CTAs that ran
  std::memcpy(out, h.data(), size_t(k) * 5 * 8);
  *out_n = k;
  return SS_OK;
}

// FragX rows [0, rows) of an activation buffer (layout NT) -> host fp32 [rows x cols] (debug)
static ss_status read_fragx(ss_ctx* c, const uint16_t* buf, int rows, int cols, int NT, float* out) {
  std::vector<uint16_t> h(size_t(NT) * 8 * cols);
  CK(cudaMemcpyAsync(h.data(), buf, h.size() * 2, cudaMemcpyDeviceToHost, c->cs));
  CK(cudaStreamSynchronize(c->cs));
  for (int m = 0; m < rows; ++m)
    for (int k = 0; k < cols; ++k) {
      const uint32_t b = uint32_t(h[fragx_offset(m, k, NT)]) << 16;
      std::memcpy(out + int64_t(m) * cols + k, &b, 4);
    }
  return SS_OK;
}

ss_status ss_debug_forward(ss_ctx* c, int32_t which, const int32_t* tokens, const int32_t* parents, int32_t n,
                           float* out_logits, float* opt_hidden) {
  GUARD(c);
  if (ensure_debug_bufs(c) != SS_OK) return SS_ERR_BUDGET;
  if (c->state != ST_SESSION && c->state != ST_DRAFTED)
    return fail(c, SS_ERR_STRUCTURE, "debug_forward needs a session (or a drafted tree)");
  if (!tokens || !parents || n < 1 || n > c->max_nodes || !out_logits) return fail(c, SS_ERR_INVALID, "debug_forward args");
  if (which == 1 && c->state == ST_DRAFTED) return fail(c, SS_ERR_STRUCTURE, "target debug_forward inside a step");
  // batched requests: tokens/parents/outputs are [B][n] over the active slots, trees of one shape
  const int B = c->B;
  std::vector<int> dep0(n);
  for (int b = 0; b < B; ++b) {
    const int32_t* tb = tokens + int64_t(b) * n;
    const int32_t* pb = parents + int64_t(b) * n;
    std::vector<int> dep(n), anc(size_t(n) * c->anc_stride, 0), par(pb, pb + n), tk(tb, tb + n);
    for (int i = 0; i < n; ++i) {
      if (i == 0 ? pb[0] != -1 : (pb[i] < 0 || pb[i] >= i)) return fail(c, SS_ERR_STRUCTURE, "tree not depth-major");
      dep[i] = i == 0 ? 0 : dep[pb[i]] + 1;
      if (i > 0 && dep[i] < dep[i - 1]) return fail(c, SS_ERR_STRUCTURE, "tree not depth-major");
      if (dep[i] >= c->anc_stride) return fail(c, SS_ERR_CAPACITY, "tree too deep");
      if (tb[i] < 0 || tb[i] >= c->V) return fail(c, SS_ERR_INVALID, "token id");
      if (b > 0 && dep[i] != dep0[i]) return fail(c, SS_ERR_STRUCTURE, "batched debug_forward: trees of one shape");
      int a = i, dd = dep[i];
      while (a >= 0) {
        anc[size_t(i) * c->anc_stride + dd--] = a;
        a = pb[a];
      }
    }
    if (b == 0) dep0 = dep;
    if (c->Pb[b] + dep[n - 1] + 1 > c->C) return fail(c, SS_ERR_CAPACITY, "tree beyond max_context");
    std::vector<float> sc(n, 0.f);
    const int64_t no = int64_t(b) * c->max_nodes;
    CK(cudaMemcpyAsync(c->tok + no, tk.data(), size_t(n) * 4, cudaMemcpyHostToDevice, c->cs));
    CK(cudaMemcpyAsync(c->parent + no, par.data(), size_t(n) * 4, cudaMemcpyHostToDevice, c->cs));
    CK(cudaMemcpyAsync(c->depth + no, dep.data(), size_t(n) * 4, cudaMemcpyHostToDevice, c->cs));
    CK(cudaMemcpyAsync(c->score + no, sc.data(), size_t(n) * 4, cudaMemcpyHostToDevice, c->cs));
    CK(cudaMemcpyAsync(c->anc + no * c->anc_stride, anc.data(), anc.size() * 4, cudaMemcpyHostToDevice, c->cs));
    CK(cudaStreamSynchronize(c->cs));   // the host vectors die with this iteration
  }
  ss_status s;
  std::vector<float> hid;
  if (which == 0) {
    int i0 = 0;
    while (i0 < n) {
      int i1 = i0;
      while (i1 < n && dep0[i1] == dep0[i0]) ++i1;
      const int rows = i1 - i0, M = B * rows;
      if (M > 32) return fail(c, SS_ERR_INVALID, "draft debug forward: <= 32 rows per depth (all slots)");
      PassOut o;
      o.logits = true;
      c->cur_rq = batch_map(c, rows);
      s = forward_pass(c, false, M, i0, o);
      c->cur_rq = ReqMap{0, 0, 0, 0};
      if (s != SS_OK) return s;
      for (int b = 0; b < B; ++b)
        CK(cudaMemcpyAsync(out_logits + (int64_t(b) * n + i0) * c->V, c->logits + int64_t(b) * rows * c->V,
                           size_t(rows) * c->V * 4, cudaMemcpyDeviceToHost, c->cs));
      if (opt_hidden) {   // the final normed rows the head just read (FragX, NT of the pass; fp32: h32)
        hid.resize(size_t(M) * c->H);
        if (c->f32) CK(cudaMemcpyAsync(hid.data(), c->h32, hid.size() * 4, cudaMemcpyDeviceToHost, c->cs));
        else if ((s = read_fragx(c, c->hfrag, M, c->H, gemv_nt(M), hid.data())) != SS_OK) return s;
        CK(cudaStreamSynchronize(c->cs));
        for (int b = 0; b < B; ++b)
          std::memcpy(opt_hidden + (int64_t(b) * n + i0) * c->H, hid.data() + size_t(b) * rows * c->H,
                      size_t(rows) * c->H * 4);
      }
      CK(cudaStreamSynchronize(c->cs));
      i0 = i1;
    }
  } else {
    PassOut o;   // no head: we read logits via the GEMV head in 32-row groups below
    c->n_nodes = n;
    c->cur_rq = batch_map(c, n);   // rows request-major: request b's nodes at b * n
    s = forward_pass(c, true, B * n, 0, o);
    c->cur_rq = ReqMap{0, 0, 0, 0};
    if (s != SS_OK) return s;
    if (c->f32) {   // logits and the final normed rows of the fp32 pass
      CK(cudaMemcpyAsync(out_logits, c->logits32, size_t(n) * c->V * 4, cudaMemcpyDeviceToHost, c->cs));
      if (opt_hidden) CK(cudaMemcpyAsync(opt_hidden, c->h32, size_t(n) * c->H * 4, cudaMemcpyDeviceToHost, c->cs));
      CK(cudaStreamSynchronize(c->cs));
      return check_launch(c, "debug_forward");
    }
    for (int r0 = 0; r0 < B * n; r0 += 32) {
      const int m = std::min(32, B * n - r0);
      launch_rmsnorm(c->x + int64_t(r0) * c->H, m, c->H, c->final_norm, c->cfg.rms_eps, c->hfrag, c->hxs, gemv_nt(m), false, c->cs);
      GemvParams p{};
      p.W = c->head;
      p.X = c->hfrag;
      p.N = c->V;
      p.K = c->H;
      p.NT = gemv_nt(m);
      p.partials = c->gv_part;
      p.counters = c->gv_cnt;
      p.max_seg = gemv_max_segments(c->V, c->H, gemv_streamk_grid(false, c->V, c->H, c->gv_grid));
      p.epi = base_epi(c, m);
      p.epi.kind = EPI_LOGITS;
      p.epi.out = c->logits;
      p.epi.ldo = c->V;
      launch_gemv(false, p, c->gv_grid, false, c->cs);
      CK(cudaMemcpyAsync(out_logits + int64_t(r0) * c->V, c->logits, size_t(m) * c->V * 4, cudaMemcpyDeviceToHost, c->cs));
      if (opt_hidden && (s = read_fragx(c, c->hfrag, m, c->H, gemv_nt(m), opt_hidden + int64_t(r0) * c->H)) != SS_OK)
        return s;
      CK(cudaStreamSynchronize(c->cs));
    }
  }
  return check_launch(c, "debug_forward");
}

ss_status ss_debug_set_tree(ss_ctx* c, const int32_t* tokens, const int32_t* parents, int32_t n, int32_t top_k) {
  GUARD(c);
  if (c->state != ST_SESSION) return fail(c, SS_ERR_STRUCTURE, "set_tree needs a session");
  if (!tokens || !parents || n < 1 || top_k < 1 || (n - 1) % top_k || n > c->max_nodes)
    return fail(c, SS_ERR_INVALID, "set_tree args");
  const int D = (n - 1) / top_k;
  if (c->P + 1 + D > c->C) return fail(c, SS_ERR_CAPACITY, "tree beyond max_context");
  std::vector<int> dep(n), anc(size_t(n) * c->anc_stride, 0);
  for (int i = 0; i < n; ++i) {
    const int want = i == 0 ? 0 : 1 + (i - 1) / top_k;
    dep[i] = i == 0 ? 0 : dep[parents[i]] + 1;
    if ((i == 0 && parents[0] != -1) || (i > 0 && (parents[i] < 0 || parents[i] >= i)) || dep[i] != want)
      return fail(c, SS_ERR_STRUCTURE, "set_tree: not a depth-major k-ary tree");
    int a = i, dd = dep[i];
    while (a >= 0) {
      anc[size_t(i) * c->anc_stride + dd--] = a;
      a = parents[a];
    }
  }
  std::vector<float> sc(n, 0.f);
  CK(cudaMemcpyAsync(c->tok, tokens, size_t(n) * 4, cudaMemcpyHostToDevice, c->cs));
  CK(cudaMemcpyAsync(c->parent, parents, size_t(n) * 4, cudaMemcpyHostToDevice, c->cs));
  CK(cudaMemcpyAsync(c->depth, dep.data(), size_t(n) * 4, cudaMemcpyHostToDevice, c->cs));
  CK(cudaMemcpyAsync(c->score, sc.data(), size_t(n) * 4, cudaMemcpyHostToDevice, c->cs));
  CK(cudaMemcpyAsync(c->anc, anc.data(), anc.size() * 4, cudaMemcpyHostToDevice, c->cs));
  CK(cudaMemcpyAsync(c->root_tok, tokens, 4, cudaMemcpyHostToDevice, c->cs));
  CK(cudaStreamSynchronize(c->cs));
  c->n_nodes = n;
  c->cur_k = top_k;
  c->cur_deff = D;
  CK(cudaEventRecord(c->e0, c->cs));
  CK(cudaEventRecord(c->e1, c->cs));
  c->state = ST_DRAFTED;
  return SS_OK;
}

static ss_status read_kv_impl(ss_ctx* c, bool draft, int32_t layer, int32_t pos0, int32_t n, uint16_t* k, uint16_t* v) {
  // pos0 indexes the kv-head row space of all slots: slot b's committed rows start at b * max_context
  if (layer < 0 || layer >= c->L || pos0 < 0 || n < 1 || pos0 + n > c->kv_ctx || !k || !v)
    return fail(c, SS_ERR_INVALID, "read_kv args");
  if (draft && !c->kcd) return fail(c, SS_ERR_STRUCTURE, "read_draft_kv: the draft shares the target's cache");
  const uint16_t* kc = draft ? c->kcd : c->kc;
  const uint16_t* vc = draft ? c->vcd : c->vc;
  CK(cudaStreamSynchronize(c->cs));
  const int es = c->kv_es;   // SS_FP32: 4-byte elements (k, v hold fp32 values)
  for (int h = 0; h < c->nkv; ++h) {
    const int64_t src = (layer * c->kc_layer + (int64_t(h) * c->kv_ctx + pos0) * c->d) * es;
    CK(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(k) + int64_t(h) * n * c->d * es, reinterpret_cast<const uint8_t*>(kc) + src,
                       size_t(n) * c->d * es, cudaMemcpyDeviceToHost, c->cs));
    CK(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(v) + int64_t(h) * n * c->d * es, reinterpret_cast<const uint8_t*>(vc) + src,
                       size_t(n) * c->d * es, cudaMemcpyDeviceToHost, c->cs));
  }
  CK(cudaStreamSynchronize(c->cs));
  return SS_OK;
}

ss_status ss_debug_read_kv(ss_ctx* c, int32_t layer, int32_t pos0, int32_t n, uint16_t* k, uint16_t* v) {
  GUARD(c);
  return read_kv_impl(c, false, layer, pos0, n, k, v);
}

ss_status ss_debug_read_draft_kv(ss_ctx* c, int32_t layer, int32_t pos0, int32_t n, uint16_t* k, uint16_t* v) {
  GUARD(c);
  return read_kv_impl(c, true, layer, pos0, n, k, v);
}

}  // extern "C"
