// Internal launcher interface of libsubspec (not part of the C-ABI).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ss {

// Batched requests: row m of a pass belongs to request req0 + m / rows and is
// that request's local node node_base + m % rows.  Per-request state is strided: tree arrays and
// tree-KV rows by node_stride, committed-KV rows by ctx_stride, committed_len / root_tok by 1.
// The zero map (rows = 0) is the single-request case: request req0 for every row, no offsets.
struct ReqMap {
  int rows;         // rows per request in this pass (0: all rows belong to request req0)
  int req0;         // first request of the pass
  int node_stride;  // per-request node capacity NS
  int ctx_stride;   // per-request committed-KV rows C
};
__host__ __device__ inline int rq_req(const ReqMap& r, int m) { return r.rows > 0 ? r.req0 + m / r.rows : r.req0; }
__host__ __device__ inline int rq_loc(const ReqMap& r, int m) { return r.rows > 0 ? m % r.rows : m; }

enum EpiKind { EPI_QKV = 0, EPI_RESID = 1, EPI_SILU = 2, EPI_LOGITS = 3, EPI_ARGMAX = 4, EPI_STORE = 5, EPI_RESID_NORM = 7,
               EPI_TOPK = 8 };

// Epilogue parameters shared by the GEMV (draft, M <= 32) and GEMM (verify) kernels.
struct EpiParams {
  int kind;
  int M;                         // valid tokens (rows of X)
  // EPI_QKV
  const uint16_t* bias;          // fused [q|k|v] bias (bf16) or nullptr
  uint16_t* q_out;               // [M x q_dim] bf16 natural
  uint16_t* k_tree;              // this layer's tree scratch K [n_kv][max_nodes][d]
  uint16_t* v_tree;
  int max_nodes, node_base;      // max_nodes: tree-KV rows per kv head (all requests)
  const int* committed_len;      // device P (per request)
  const int* depth;              // per-node depth (request b, row m: b * rq.node_stride + node_base + local m)
  ReqMap rq;                     // batched requests (zero: one request)
  const float2* rope;            // [max_ctx][d/2] (cos, sin)
  int q_dim, kv_dim, head_dim;
  // EPI_RESID
  float* x;                      // [M x ldx] fp32 residual stream
  int ldx;
  // EPI_SILU
  uint16_t* act;                 // FragX [Mpad x F]
  float* act_xs;                 // group sums [F/64][Mpad] (sum of the bf16 activations)
  int act_nt, ffn;
  // EPI_LOGITS / EPI_STORE
  float* out;                    // [M x ldo]
  int ldo;
  // EPI_RESID_NORM: residual add + per-tile sums of squares of the new x rows (fused RMSNorm)
  float* sumsq;                  // [N/128][sumsq_ld]
  int sumsq_ld;                  // Mpad; 0 = the caller's tile stride
  // EPI_RESID_NORM (cluster GEMV only): + in-kernel barrier of the tile owners, then the owner of
  // tile r writes h = bf16(x * r_m * gain) for columns [128 r, 128 r + 128) in FragX + group sums
  const uint16_t* norm_gain;
  uint16_t* norm_out;
  float* norm_xs;
  unsigned long long* norm_ctr;  // monotonic arrival counter of the norm barrier (zero at creation)
  int n_tiles;
  float eps;
  // EPI_TOPK (draft head, K5 folded into the GEMV): per (token, 128-row vocab tile) the tile's max logit,
  // sum exp((l - max) / T) and its top tk_k logits (value desc, index asc) -> [token][tile] arrays
  float* tk_max;                 // [M][tk_tiles]
  float* tk_sum;
  float* tk_val;                 // [M][tk_tiles][tk_k]
  int* tk_idx;
  int tk_k, tk_tiles;
  float tk_inv_t;
  // EPI_ARGMAX: per (token, row tile) partial (max, idx, second max)
  float* am_val;                 // [M x n_tiles]
  int* am_idx;
  float* am_second;
  int am_tiles;
};

struct GemvParams {
  const uint8_t* W;              // tiled weights (Q4 or BF16)
  const uint16_t* X;             // FragX [Mpad x K]
  const float* XS;               // Q4 only: group sums of X, [K/64][Mpad] fp32 (sum of the bf16 values)
  int N, K, NT;                  // NT = Mpad / 8
  float* partials;               // [n_tiles][max_seg][128*Mpad]
  int* counters;                 // [n_tiles], zero on entry, restored to zero on exit
  int max_seg;
  int stages;                    // ring depth (set by the launcher)
  const uint8_t* pf;             // weights of the NEXT matrix: prefetched into L2 while this one runs
  int64_t pf_bytes;
  unsigned long long* trace;     // optional %globaltimer trace: [kTraceEvents] events of this launch (debug)
  unsigned long long* cta_trace; // optional per-CTA trace [grid][5]: smid, entry, first data, loop end, end
  unsigned long long* gtrace;    // optional per-group clock64 events of CTA 0 [64][8] (debug)
  int ctas_per_sm;               // cluster plan: resident CTAs per SM to plan for (0 = default 2)
  int qbits;                     // code bits of a quantised matrix: 4 (0 = 4) or 2 (NEXT-3)
  EpiParams epi;
};

int gemv_max_segments(int N, int K, int grid);   // grid: the Stream-K grid (gemv_streamk_grid)
int gemv_streamk_grid(bool q4, int N, int K, int sms);
bool gemv_tiles_all_resident(bool q4, int NT, int N, int K, int sms, int bits = 4);
void launch_gemv(bool q4, const GemvParams& p, int grid, bool pdl, cudaStream_t st);
void launch_gemv_q(const GemvParams& p, int sms, bool pdl, cudaStream_t st);   // substitutes (gemv_q.cu)
bool gemv_q_tiles_all_resident(int NT, int N, int K, int sms, int bits);

struct GemmParams {
  const uint8_t* W;              // tiled BF16 weights [N x K] (row tiles [tile0, tile0 + N/128) of the matrix)
  const uint16_t* X;             // FragX [Mpad x K], Mpad % 128 == 0
  int N, K, NT;                  // NT = Mpad/8; N = rows of this launch
  EpiParams epi;
  int tile0;                     // first row tile of the matrix this launch covers (epilogue row index)
  int split_n;                   // rows of the whole matrix (K-split plan; 0 = N): a matrix launched in
                                 // row blocks keeps its reduction order (batch invariance)
};
// variant: 0 tcgen05 whole-chunk stages (default), 1 legacy mma.sync, 2 tcgen05 half-chunk stages
void launch_gemm(const GemmParams& p, bool pdl, cudaStream_t st, int variant = 0);
int gemm_tc_split(int N, int K, int sms);

// K7 stream codec (zstream.cu): lossless exponent-coded bf16 blobs of the streamed layers
constexpr int kZChunk = 16384;                 // weights per chunk (one bf16 tile-chunk)
constexpr uint32_t kZMagic = 0x315A5353u;      // "SSZ1"
struct ZTable {
  uint8_t exp[8];                              // code -> exponent; code 7 = exception
};
struct ZHeader {                               // at the start of every blob (64 bytes)
  uint32_t magic, mode, nchunks, nexc;         // mode 0: raw bf16 at a0; 1: coded
  ZTable table;
  uint64_t n, a0, b0, e0, used;                // weights; plane A, planes B, exceptions offsets; bytes to stream
};
static_assert(sizeof(ZHeader) == 64, "ZHeader");
size_t zhdr_bytes(int64_t n);
size_t zblob_cap(int64_t n);
cudaError_t zencode(const uint16_t* x, int64_t n, uint8_t* blob, void* scratch, cudaStream_t st, ZHeader* out);
void launch_zdecode(const uint8_t* blob, uint16_t* out, int64_t n, cudaStream_t st);
void launch_zdecode_range(const uint8_t* blob, uint16_t* out, int chunk0, int nchunks, cudaStream_t st);
void zdecode_host(const uint8_t* blob, uint16_t* out);

// generator / quantizer / readback
void launch_gen_natural(uint16_t* dst, uint64_t key, uint64_t count, float c32, int gain, cudaStream_t st,
                        uint64_t first = 0);   // elements [first, first + count) of the tensor
void launch_gen_tiled(uint8_t* dst, uint64_t key, int64_t rows, int64_t K, float c32, int map, int64_t row_off,
                      cudaStream_t st);
void launch_tile_from_natural(uint8_t* dst, const uint16_t* src, int64_t rows, int64_t K, int map, int64_t row_off,
                              cudaStream_t st);
void launch_quantize(const uint8_t* src_bf16_tiled, uint8_t* dst_q, int64_t N, int64_t K, int bits, int hqq_iters,
                     cudaStream_t st);
void launch_q4_to_canonical(const uint8_t* q4, uint8_t* codes, uint16_t* s, uint16_t* z, int64_t N, int64_t K,
                            cudaStream_t st);
void launch_tiled_to_natural(const uint8_t* t, uint16_t* out, int64_t N, int64_t K, cudaStream_t st);

// small kernels (K4, K5, K8, K9)
void launch_embed_rmsnorm(const int* tokens_dev, int tok_offset, int M, const uint16_t* embed, float* x, int H,
                          const uint16_t* gain, float eps, uint16_t* h_fragx, float* h_xs, int nt, bool pdl,
                          cudaStream_t st, ReqMap rq = ReqMap{0, 0, 0, 0});
void launch_rmsnorm(const float* x, int M, int H, const uint16_t* gain, float eps, uint16_t* h_fragx, float* h_xs,
                    int nt, bool pdl, cudaStream_t st);

struct AttnParams {
  const uint16_t* q;             // [n_q x n_h*d] bf16
  const uint16_t* k_cache;       // committed [n_kv][max_ctx][d]
  const uint16_t* v_cache;
  const uint16_t* k_tree;        // [n_kv][max_nodes][d]
  const uint16_t* v_tree;
  const int* committed_len;
  const int* anc;                // [max_nodes][anc_stride] ancestor slots root..self
  const int* depth;              // [max_nodes]
  int anc_stride, max_ctx, max_nodes;   // max_ctx / max_nodes: rows per kv head (all requests)
  int n_q, node_base;            // query rows are nodes node_base .. node_base + n_q - 1
  ReqMap rq;                     // batched requests (zero: one request)
  int n_heads, n_kv, head_dim;
  int cluster;                   // CTAs per (kv head, node) cluster (set by the launcher)
  unsigned long long* trace;     // optional (debug): 0 entry min, 1 dep released max, 2 q loaded max,
                                 // 3 key loop done max, 4 CTA merge done max, 5 end max
  uint16_t* out_fragx;           // [Mpad x n_heads*d] FragX
  float* out_xs;                 // group sums [n_heads*d/64][Mpad]
  int out_nt;
};
void launch_attention(const AttnParams& p, bool pdl, cudaStream_t st);

struct TopkParams {
  const float* logits;           // [M x V]
  int M, V, k;
  float inv_t;                   // 1 / sharpen temperature
  int blocks_per_row;
  float* blk_max;                // [M][B]
  float* blk_sum;                // [M][B]  sum exp((l - blk_max) * inv_t)
  float* blk_val;                // [M][B][k]
  int* blk_idx;
  // tree state (device)
  int* tok;                      // [max_nodes]
  int* parent;
  int* depth;
  float* score;
  int* anc;                      // [max_nodes][anc_stride]
  int anc_stride;
  int node_base;                 // frontier nodes node_base .. node_base + M - 1
  int child_base;                // new nodes child_base .. child_base + k - 1
  int child_depth;
  int req_rows;                  // batched: frontier rows per request (0: all M rows, one request);
  int node_stride;               // one select CTA per request, tree arrays strided by node_stride
};
void launch_topk(const TopkParams& p, bool pdl, cudaStream_t st);
// the global selection only, over per-tile statistics the head GEMV's EPI_TOPK epilogue wrote
// (blocks_per_row = vocab tiles)
void launch_topk_select(const TopkParams& p, bool pdl, cudaStream_t st);

void launch_argmax_merge(const float* am_val, const int* am_idx, const float* am_second, int M, int tiles,
                         int* argmax, float* gap, bool pdl, cudaStream_t st);

struct AcceptParams {
  const int* argmax;             // [n_nodes]
  const int* tok;
  const int* parent;
  int* commit_meta;              // [2]: base position, rows committed
  int n_nodes, k, depth_max;
  int* committed_len;            // in/out
  int* root_tok;                 // out: bonus token = next root
  int* out_tokens;               // [depth_max + 1] emitted tokens
  int* out_n;                    // count
  int* out_path;                 // [depth_max + 1]: root + accepted slots
  // KV commit
  uint16_t* k_cache;             // base of committed K for layer 0; layer stride below
  uint16_t* v_cache;
  const uint16_t* k_tree;
  const uint16_t* v_tree;
  int64_t cache_layer_stride, tree_layer_stride;   // elements
  int n_layers, n_kv, head_dim, max_ctx, max_nodes;
  int chain;                     // 1: commit all nodes (prefill chunk), ignore argmax
  // batched requests: request b = req0 + blockIdx; argmax rows by n_nodes, tree arrays / tree-KV rows
  // by node_stride, committed-KV rows by ctx_stride, outputs by out_stride, meta by 2
  int n_req, req0, node_stride, ctx_stride, out_stride;
};
void launch_commit(const AcceptParams& p, bool pdl, cudaStream_t st);   // commit only (commit_meta from accept)
void launch_accept_commit(const AcceptParams& p, bool pdl, cudaStream_t st);

// SS_FP32 precision mode (f32.cu)
void launch_rmsnorm_f32(const int* tokens, int tok_offset, const uint16_t* embed, float* x, int M, int H,
                        const uint16_t* gain, float eps, float* h, cudaStream_t st);
void launch_linear_f32(const float* X, int M, int K, const uint8_t* W, int fmt, int N, float* Y, cudaStream_t st);
void launch_qkv_post_f32(const float* Y, int M, const uint16_t* bias, int qd, int kvd, int d, const float2* rope,
                         const int* committed_len, const int* depth, int node_base, float* q_out, float* k_tree,
                         float* v_tree, int max_nodes, cudaStream_t st);
void launch_attention_f32(const float* q, const float* k_cache, const float* v_cache, const float* k_tree,
                          const float* v_tree, const int* committed_len, const int* anc, const int* depth, int anc_stride,
                          int max_ctx, int max_nodes, int node_base, int M, int n_heads, int n_kv, int d, float* out,
                          cudaStream_t st);
void launch_add_f32(float* x, const float* y, int64_t n, cudaStream_t st);
void launch_silu_mul_f32(const float* Y, int M, int F, float* act, cudaStream_t st);
void launch_argmax_f32(const float* logits, int M, int V, int* argmax, float* gap, cudaStream_t st);

// tree init for a new step: root node (slot 0) with token *root_tok, depth 0
void launch_tree_init(const int* root_tok, int* tok, int* parent, int* depth, float* score, int* anc, bool pdl,
                      cudaStream_t st, int n_req = 1, int node_stride = 0, int anc_stride = 0);
// chain tree for prefill chunk: tokens copied from device buffer
void launch_chain_init(const int* tokens, int n, int* tok, int* parent, int* depth, float* score, int* anc,
                       int anc_stride, cudaStream_t st);

}  // namespace ss
