/*
 * subspec.h — C-ABI of libsubspec: one SubSpec tree-speculative decode step on a B200.
 *
 * Method: Substitute Speculative Decoding (arXiv 2509.18344, §4).  The draft model
 * reuses the target's GPU-resident layers ("GPU-Resident Layer Sharing"),
 * replaces every offloaded layer with a low-bit quantized substitute that stays on the GPU
 * ("Quantized Substitute Weights"; 4-bit, group 64) and shares
 * the target's KV-cache ("Shared KV-Cache").  It grows a context-aware dynamic
 * draft tree of depth D with top-k expansion over sharpened cumulative scores (
 * k = 6, D = 48, T = 0.2).  The target verifies all 1 + kD nodes in one pass
 * with its offloaded layers streamed from pinned host memory, and the
 * longest root path matching the target's greedy choices is accepted and committed (greedy
 * verification).  The committed output equals greedy AR decoding of the
 * target ("lossless").  Step order follows Eq. 2.
 *
 * Conventions:
 *  - Every function returns ss_status; on error ss_last_error(ctx) describes it.  After any CUDA
 *    error the context is poisoned: every later call returns SS_ERR_CUDA; only ss_destroy is valid.
 *  - Ownership: the library never retains a caller pointer after a call returns, except the
 *    device arena and streams given to ss_create, which the caller keeps alive until ss_destroy.
 *    Every device allocation of the context is carved from that arena, so arena_bytes is the
 *    emulated VRAM cap (CUDA context memory is excluded).  The context owns its
 *    pinned host store (cudaHostAlloc, portable) for offloaded layers.
 *  - Host pointers: all array arguments below are HOST pointers unless named dev_*; they are
 *    read/written only during the call.  Calls that return host data synchronise the compute
 *    stream before returning.
 *  - Call order: create -> load_weights -> build_substitutes -> prefill ->
 *    (draft_tree -> verify_tree -> accept_and_commit)*  [or ss_step / ss_generate].  Any other
 *    order returns SS_ERR_STRUCTURE.  One context per session; no concurrent calls on a context.
 *  - Capacity: before drafting, D is clamped to D_eff = min(D, floor((max_context - P - 1)/k));
 *    D_eff = 0 runs an AR step (tree = root only).  SS_ERR_CAPACITY only when P + 1 > max_context,
 *    detected before any write.
 *  - Layouts: token ids int32; all weights bf16 [out x in] row-major (bit patterns as uint16).
 */
#ifndef SUBSPEC_H
#define SUBSPEC_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SS_OK = 0,
  SS_ERR_INVALID = 1,   /* bad argument, non-finite input, unsupported config */
  SS_ERR_CAPACITY = 2,  /* context would exceed max_context (checked before any write) */
  SS_ERR_STRUCTURE = 3, /* call out of order, malformed tree */
  SS_ERR_BUDGET = 4,    /* arena (VRAM cap) below the minimum footprint */
  SS_ERR_CUDA = 5       /* CUDA failure; context poisoned */
} ss_status;

/* Arithmetic of the forward passes.  SS_BF16: the target is bf16 (BASELINE.json;
 * PAPER.md:361 "Original (fp16)", reading R20) with bf16 rounding at the named points of reading R3
 * (normed inputs, q/k/v, attention output, SiLU*mul) and fp32 accumulation; parity tolerance 2e-2 x
 * logit scale.  SS_FP32: the same weights (bf16 values, exact in fp32) with every activation kept in
 * fp32 (no rounding points, fp32 KV cache, fp32 CUDA-core arithmetic); parity tolerance 1e-4 x logit
 * scale.  SS_FP32 is a parity mode: it supports n_resident = n_layers (nothing streamed), batch 1. */
enum { SS_BF16 = 0, SS_FP32 = 1 };

/* Decoder-only model shape (Llama/Qwen family).  hidden, ffn, qkv rows and vocab
 * must be multiples of 128; head_dim is 64 or 128; n_heads % n_kv_heads == 0. */
typedef struct {
  int32_t n_layers, hidden, n_heads, n_kv_heads, head_dim, ffn, vocab, max_context;
  float rope_theta, rms_eps;
  int32_t qkv_bias;
  int32_t precision;    /* SS_BF16 (0) or SS_FP32 (1) */
} ss_model_config;

/* Sizes the context provisions buffers for (all >= the values later used). */
typedef struct {
  int32_t max_depth;    /* D_max (48) */
  int32_t max_top_k;    /* k_max (<= 32) */
  int32_t max_chunk;    /* prefill chunk (256) */
  int32_t max_batch;    /* request slots of one weight stream (0 or 1 = one
                           request, the paper's batch 1); max_batch * max_top_k <= 32.  Each
                           slot owns max_context rows of committed KV inside the arena. */
} ss_limits;

/* Per-context options (ss_create; NULL = the defaults below).  They replace process-wide
 * environment switches, so contexts in one process may differ. */
typedef struct {
  int32_t embed_on_host;  /* 1 (default): the embedding table lives in mapped pinned host memory and
                             a pass gathers its <= max_nodes rows over the host link (zero-copy); its
                             2*vocab*hidden bytes of the VRAM cap go to the streaming ring (reading
                             R24).  0: the embedding is GPU-resident in the arena, the
                             placement of PAPER.md:534 ("Embedding and head layers are default to be
                             GPU-resident").  The head is always GPU-resident. */
  int32_t async_stream;   /* 1 (default): layer copies overlap compute.  0: the
                             Table-2 "async transfer" ablation: a group is copied only after the
                             previous group's compute. */
  int32_t cuda_graphs;    /* 1 (default): the draft loop is replayed from a CUDA graph; 0: eager */
  int32_t fuse_norm;      /* 1 (default): RMSNorm fused into the o/down GEMV epilogues (draft) */
  int32_t separate_draft_kv; /* 0 (default): the draft attends over the target's committed KV (shared
                             KV-cache).  1: SURVEY §8(f) NEXT-4, Table 2's row
                             without "+ shared KV": the draft keeps its own
                             committed cache, filled with the draft's own K/V — by draft forwards of
                             every prefill chunk and, each step, by committing the draft's tree K/V of
                             the accepted path (one extra KV-only draft pass covers depth D).  Costs
                             2 x L x max_context x n_kv x head_dim x 2 bytes of the cap plus tree
                             scratch.  One request per context (max_batch <= 1), bf16 only. */
  int32_t compress_stream;  /* 1 (default, bf16): the host store holds each offloaded matrix as a
                             lossless exponent-coded blob (sign+mantissa bytes, 3-bit exponent codes,
                             exceptions; ~0.69 of the bf16 bytes for Gaussian-like weights), streamed
                             as is and decoded on the GPU before the verify GEMM: the same bf16
                             weights, fewer bytes over the host link (A4).  Costs
                             one decode buffer of the largest matrix group in the cap.  0: plain bf16.
                             Ignored in SS_FP32 mode. */
} ss_options;
void ss_default_options(ss_options* out);

/* Substitute quantization ("quantized to 4 bits with a group size 64 using HQQ"):
 * bits = 4 (or 3 / 2, see ss_set_substitute_bits), group_size = 64.  method: SS_QUANT_RTN (0, min/max
 * round-to-nearest, SPEC.md:125 — HQQ's initialisation, reading R1) or SS_QUANT_HQQ (1, the same scale
 * with HQQ's half-quadratic zero refinement: l_0.7 objective, beta0 = 10, kappa = 1.01, per 64-group
 * early stop keeping the zero of the lowest mean |x - x_hat|, fp64; reading R28 in DESIGN.md,
 * oracle/quant.py).  hqq_iters: maximum iterations (0 = 20, HQQ's default); ignored for RTN. */
enum { SS_QUANT_RTN = 0, SS_QUANT_HQQ = 1 };
typedef struct { int32_t bits, group_size, method, hqq_iters; } ss_quant_spec;

/* Draft tree parameters: depth D, top-k, sharpening temperature. */
typedef struct { int32_t depth, top_k; float sharpen_t; } ss_draft_params;

typedef struct {
  int64_t steps, tokens_emitted, prefill_tokens, gpu_launches;
  double draft_ms, verify_ms, accept_ms;      /* device time (CUDA events), cumulative */
  double stream_bytes, stream_busy_ms;        /* host->device layer streaming (copy stream) */
  int64_t arena_used, arena_cap, ring_bytes, host_pinned_bytes, substitute_bytes;
  int32_t n_resident, n_offloaded, committed_len, last_d_eff;
  double peer_bytes;                          /* NEXT-1: bytes this rank pushed to peers' rings */
  double stream_raw_bytes;                    /* bf16 bytes of the streamed groups delivered to the
                                                 verify (stream_bytes: what crossed the host link) */
} ss_stats;

typedef struct ss_ctx ss_ctx;

/* Create a context on `device`.  dev_arena/arena_bytes: caller-owned device block (torch), the
 * VRAM cap.  compute_stream/copy_stream: cudaStream_t handles (may be the same only if
 * streaming is never needed).  opt: NULL for ss_default_options.  Errors: INVALID (shape,
 * precision), BUDGET (arena too small for fixed parts). */
ss_status ss_create(const ss_model_config* cfg, const ss_limits* lim, const ss_options* opt, int device,
                    void* dev_arena, size_t arena_bytes, void* compute_stream, void* copy_stream, ss_ctx** out);

/* The target's weights as caller-owned HOST arrays: bf16 bit patterns, matrices [out x in]
 * row-major, read only during ss_load_weights (pageable or pinned memory).  Biases are NULL
 * unless cfg.qkv_bias.  The substitutes are derived from these ("data-free",
 * built from the target's own offloaded layers). */
typedef struct {
  const uint16_t* attn_norm;   /* [hidden] */
  const uint16_t* wq;          /* [n_heads*head_dim x hidden] */
  const uint16_t* bq;          /* [n_heads*head_dim] or NULL */
  const uint16_t* wk;          /* [n_kv_heads*head_dim x hidden] */
  const uint16_t* bk;          /* [n_kv_heads*head_dim] or NULL */
  const uint16_t* wv;          /* [n_kv_heads*head_dim x hidden] */
  const uint16_t* bv;          /* [n_kv_heads*head_dim] or NULL */
  const uint16_t* wo;          /* [hidden x n_heads*head_dim] */
  const uint16_t* mlp_norm;    /* [hidden] */
  const uint16_t* wg;          /* [ffn x hidden] */
  const uint16_t* wu;          /* [ffn x hidden] */
  const uint16_t* wd;          /* [hidden x ffn] */
} ss_host_layer;
typedef struct {
  const uint16_t* embed;        /* [vocab x hidden] */
  const ss_host_layer* layers;  /* [n_layers] */
  const uint16_t* final_norm;   /* [hidden] */
  const uint16_t* head;         /* [vocab x hidden] (untied) */
} ss_host_weights;

/* Load the target's bf16 weights from caller-owned host arrays and place them: layers
 * [0, n_resident) resident in the arena, the rest offloaded to the context's pinned host store in
 * device layout (App. H P:540 "All decoder layers ... offloaded" is n_resident = 0).
 * n_resident = -1: the planner's maximum resident prefix under the cap.  The
 * head and final norm are GPU-resident; the embedding as ss_options.embed_on_host says.  The
 * library keeps no pointer into `w` after returning.  Errors: INVALID (NULL tensor, bias presence
 * differs from cfg.qkv_bias), BUDGET (placement does not fit the cap), STRUCTURE (already loaded),
 * CUDA. */
ss_status ss_load_weights(ss_ctx* ctx, const ss_host_weights* w, int32_t n_resident);

/* As ss_load_weights, with the weights generated on the device by the counter-based synthetic
 * generator of SURVEY.md §8(c) O.1 (seed; the same values synth/weights.py produces on the host).
 * The benchmark workloads use it so that a 7B/32B-shape model need not be materialised on the host
 * first. */
ss_status ss_load_weights_synthetic(ss_ctx* ctx, uint64_t seed, int32_t n_resident);

/* Code width of the substitutes this context will build: 4 (default; "4 bits with a
 * group size 64"), 3 or 2 (the paper's "more aggressive" 2/3-bit direction,
 * PAPER.md:343; the same quantizer with 2^bits - 1 levels).  Fixes the substitutes' layout and
 * footprint (3-bit: 0.4375 B/weight, 2-bit: 0.3125, vs 0.5625), so it is only valid before loading
 * weights; the arena bytes it frees go to the streaming ring.  ss_build_substitutes must then pass
 * the same bits.  Errors: STRUCTURE (after load), INVALID (bits not 2, 3 or 4). */
ss_status ss_set_substitute_bits(ss_ctx* ctx, int32_t bits);

/* Bytes of the offloaded layers' host store for an explicit n_resident >= 0 (bf16, device layout).
 * Errors: INVALID. */
ss_status ss_host_store_bytes(ss_ctx* ctx, int32_t n_resident, size_t* out_bytes);

/* As ss_load_weights_synthetic, but the offloaded layers live in a CALLER-OWNED host store (e.g. one POSIX
 * shared-memory segment mapped by every rank of a multi-GPU job, so the node holds one copy —
 * SURVEY §8(e)).  host_store: >= ss_host_store_bytes(n_resident) bytes, page-aligned, owned by the
 * caller and kept alive until ss_destroy; the library page-locks it with cudaHostRegister (portable,
 * refcounted per process) and unregisters it at ss_destroy.  fill = 1: generate the offloaded
 * layers into the store (one context of the job); fill = 0: the store already holds them (the caller
 * orders the filling context's return before this call, e.g. with a barrier).  n_resident >= 0.
 * Errors: INVALID, BUDGET (store too small), CUDA (registration failed), as ss_load_weights. */
ss_status ss_load_weights_synthetic_shared(ss_ctx* ctx, uint64_t seed, int32_t n_resident, void* host_store,
                                           size_t host_bytes, int32_t fill);

/* Build the 4-bit (or, after ss_set_substitute_bits(3 / 2), 3- / 2-bit) group-64 substitute of every offloaded layer: stream it host->device through
 * the staging ring and quantize on the device (K1) with q->method.  Norms/biases are
 * shared.  Errors: INVALID (bits/group/method/hqq_iters), STRUCTURE (before load), CUDA. */
ss_status ss_build_substitutes(ss_ctx* ctx, const ss_quant_spec* q);

/* Start a new session (committed length 0) and prefill `prompt` (n tokens, host) through the
 * target in chunks of `chunk` tokens.  *out_first_token = greedy token at the
 * last prompt position, which becomes the root of the first draft tree. */
ss_status ss_prefill(ss_ctx* ctx, const int32_t* prompt, int32_t n, int32_t chunk, int32_t* out_first_token);

/* Draft pass loop (K2-K5): grow the tree from the current root (the last emitted token; or
 * root_token >= 0 to override).  Optional host outputs, each [1 + k*D_eff] (batched: [B][1 + k*D_eff]
 * over the active slots): tokens, parents, depths, cumulative log-scores (NULL to skip).
 * *opt_n_nodes receives 1 + k*D_eff. */
ss_status ss_draft_tree(ss_ctx* ctx, int32_t root_token, const ss_draft_params* p, int32_t* opt_tokens,
                        int32_t* opt_parents, int32_t* opt_depths, float* opt_scores, int32_t* opt_n_nodes);

/* Verification (K6-K8): one target pass over every node; offloaded layers streamed from the
 * pinned host store (K7).  Optional host outputs [n_nodes] (batched: [B][n_nodes]): target argmax
 * per node and the top-1/top-2 logit gap (near-tie flags). */
ss_status ss_verify_tree(ss_ctx* ctx, int32_t* opt_argmax, float* opt_gap);

/* Greedy acceptance + KV commit/compaction (K9).  out_tokens (capacity D+1) receives the
 * accepted draft tokens followed by the bonus token; *out_n in [1, D+1].  opt_path receives the
 * committed tree slots (root first, capacity D+1). */
ss_status ss_accept_and_commit(ss_ctx* ctx, int32_t* out_tokens, int32_t* out_n, int32_t* opt_path);

/* draft_tree + verify_tree + accept_and_commit without host round trips except the emitted tokens. */
ss_status ss_step(ss_ctx* ctx, const ss_draft_params* p, int32_t* out_tokens, int32_t* out_n);

/* Convenience loop: prefill then steps until max_new tokens (first token included) are emitted.
 * p->depth = 0 gives plain AR decoding through the same target path.  out_tokens capacity
 * max_new; opt_tau_hist capacity D+2 (histogram of tokens per step). */
ss_status ss_generate(ss_ctx* ctx, const int32_t* prompt, int32_t n, int32_t max_new, int32_t chunk,
                      const ss_draft_params* p, int32_t* out_tokens, int32_t* out_n, int32_t* opt_tau_hist);

/* ---- batched requests: one weight stream serves several trees ----------
 * The paper decodes one request at a time (batch 1) and avoids batching for latency;
 * every tree is still verified losslessly, so each request's output is its own greedy AR
 * output whatever the batch.  A context created with ss_limits.max_batch = Bmax has Bmax request
 * slots, each with its own tree arrays, committed KV (max_context rows) and committed length.  A
 * step drafts all B active trees together (B*k frontier rows per draft pass, one pass of the
 * substitute weights), verifies all B*(1+kD) nodes in ONE streamed target pass, and accepts and
 * commits each tree independently.  The trees share one shape per step: D_eff is clamped by the
 * longest request (O.10).  Ownership and synchronisation as for the one-request calls. */

/* Number of active slots n_req in [1, max_batch].  Changing it (or any n_req > 1) starts a new
 * batch session: every active slot must be prefilled again.  Errors: INVALID (range; the opt-in
 * persistent draft pass or legacy attention with n_req > 1), STRUCTURE (inside a step). */
ss_status ss_set_batch(ss_ctx* ctx, int32_t n_req);

/* ss_prefill for slot `slot` < n_req (ss_prefill == slot 0).  Drafting needs every active slot
 * prefilled.  Errors as ss_prefill, plus INVALID for a slot outside the active batch. */
ss_status ss_prefill_slot(ss_ctx* ctx, int32_t slot, const int32_t* prompt, int32_t n, int32_t chunk,
                          int32_t* out_first_token);

/* One batched step (draft + verify + accept/commit of every active slot).  out_tokens: host
 * [n_req][stride] (stride >= D + 1), out_n: host [n_req].  Synchronizes.  Errors as ss_step. */
ss_status ss_step_batch(ss_ctx* ctx, const ss_draft_params* p, int32_t stride, int32_t* out_tokens, int32_t* out_n);

/* Batched ss_generate: set_batch(n_req), prefill slot b with prompts[off_b .. off_b + lens[b])
 * (prompts concatenated on the host), then batched steps until every request has max_new tokens.
 * out_tokens: host [n_req][max_new]; out_n: [n_req]; opt_tau_hist as ss_generate (all requests). */
ss_status ss_generate_batch(ss_ctx* ctx, int32_t n_req, const int32_t* prompts, const int32_t* prompt_lens,
                            int32_t max_new, int32_t chunk, const ss_draft_params* p, int32_t* out_tokens,
                            int32_t* out_n, int32_t* opt_tau_hist);

ss_status ss_get_stats(ss_ctx* ctx, ss_stats* out);

/* cooperative weight streaming across the G GPUs of a node (PAPER.md:172-176
 * asynchronous transfer; P:382 faster interconnects).  Each rank's verify needs every offloaded layer;
 * instead of every rank pulling all of them over its own host link, rank r copies only slice r (1/G of
 * the bytes, 4 KiB aligned) of each streamed group from its host store into its ring and pushes that
 * slice over NVLink (copy engine, CUDA IPC mapping of the peers' arenas) into every peer's ring at the
 * same offset.  Completion and ring reuse are ordered by monotonic per-rank counters in device memory
 * (stream memory operations): "rank h's slice of item s has landed here" and "rank h has consumed items
 * < n".  Weights are bit-identical, so the output is unchanged.
 * Protocol: every rank calls ss_coop_export (outside a step, after ss_build_substitutes and prefill);
 * the caller exchanges the handles (e.g. all_gather); every rank calls ss_coop_enable(rank, world,
 * handles[world]), which drains this rank's stream and restarts its ring at offset 0; then the caller
 * BARRIERS before any rank continues.  From then on every rank must run the same sequence of target
 * passes (the same number of steps / prefill chunks: the GPUs verify in lockstep), and
 * no rank destroys its context before ss_coop_finish + a barrier.  export / enable / finish may be
 * repeated (one cooperative epoch each).  Errors: INVALID (handles, ranks differ in model/placement/ring), STRUCTURE (order, inside
 * a step, no streamed layers, fp32 mode, serial-stream ablation), CUDA (IPC or stream memory ops). */
typedef struct { uint8_t bytes[256]; } ss_coop_handle;
ss_status ss_coop_export(ss_ctx* ctx, ss_coop_handle* out);
ss_status ss_coop_enable(ss_ctx* ctx, int32_t rank, int32_t world, const ss_coop_handle* all);
/* End cooperative streaming on every rank (a common point after the last lockstep pass): releases
 * the peers' pending writes into this rank's ring, waits for this rank's pending pushes, and restarts
 * the stream alone.  The caller BARRIERS afterwards, before any rank destroys its context or decodes
 * alone.  Errors: STRUCTURE (not enabled, inside a step), CUDA. */
ss_status ss_coop_finish(ss_ctx* ctx);
ss_status ss_reset_stats(ss_ctx* ctx);
const char* ss_last_error(ss_ctx* ctx);
void ss_destroy(ss_ctx* ctx);

/* ---- debug / parity entry points (tests only) ------------------------------------------- */
/* The matmul / forward / pass-timing entry points write device outputs into a debug scratch buffer
 * allocated (cudaMalloc) on their first use, outside the context's arena: it is not a product
 * allocation and does not count against the emulated VRAM cap.  Errors: BUDGET if it cannot be
 * allocated. */
/* Device generator for one tensor id (natural row-major bf16 bits) -> host out[rows*cols]. */
ss_status ss_debug_gen_tensor(ss_ctx* ctx, uint64_t seed, int32_t tid, int64_t rows, int64_t cols,
                              int32_t kind /*0 mat, 1 gain, 2 bias*/, double sigma, uint16_t* out);
/* Target bf16 matrix of (layer, group) in fused natural row order -> host [N x K].
 * groups: 0 qkv [q;k;v], 1 o, 2 gate_up (rows interleaved per 64: gate 64, up 64, ...), 3 down. */
ss_status ss_debug_read_group(ss_ctx* ctx, int32_t layer, int32_t group, uint16_t* out);
/* Substitute of an offloaded (layer, group) in canonical form: codes [N x K] u8, s,z [N x K/64] bf16 bits. */
ss_status ss_debug_get_substitute(ss_ctx* ctx, int32_t layer, int32_t group, uint8_t* codes, uint16_t* s,
                                  uint16_t* z);
/* Run the draft GEMV (K2: substitute if offloaded, bf16 if resident) or the target GEMM (K6) of
 * (layer, group) on host activations x [M x K] (bf16 bits) -> host y [M x N] fp32 (fused row order). */
ss_status ss_debug_matmul(ss_ctx* ctx, int32_t which /*0 draft K2, 1 target K6*/, int32_t layer, int32_t group,
                          const uint16_t* x, int32_t M, float* y);
/* Teacher-forced forward of a depth-major tree (tokens/parents, n nodes) at the current committed
 * length: which = 0 draft (depth by depth, as the draft loop, the same kernels and batching), 1
 * target (one pass).  Writes the tree KV (draft or target values) but commits nothing.  With
 * B > 1 active slots the arrays are [B][n] (one tree per slot, all of one shape) and the passes
 * batch the slots as ss_step_batch does.  out_logits [B][n][V] fp32; opt_hidden (NULL to skip)
 * [B][n][hidden] fp32: the final RMSNorm output the head reads (bf16 values in SS_BF16). */
ss_status ss_debug_forward(ss_ctx* ctx, int32_t which, const int32_t* tokens, const int32_t* parents, int32_t n,
                           float* out_logits, float* opt_hidden);
/* Replace the device tree by a given depth-major tree (root first) for verify/accept tests. */
ss_status ss_debug_set_tree(ss_ctx* ctx, const int32_t* tokens, const int32_t* parents, int32_t n, int32_t top_k);
/* Committed K/V rows [pos0, pos0+n) of a layer -> host [n_kv x n x head_dim] bf16 bits each (batched
 * slots: slot b's position p is row b * max_context + p).  ss_debug_read_draft_kv: the same rows of
 * the draft's own cache (ss_options.separate_draft_kv = 1; STRUCTURE otherwise). */
ss_status ss_debug_read_kv(ss_ctx* ctx, int32_t layer, int32_t pos0, int32_t n, uint16_t* k, uint16_t* v);
ss_status ss_debug_read_draft_kv(ss_ctx* ctx, int32_t layer, int32_t pos0, int32_t n, uint16_t* k, uint16_t* v);
/* An offloaded group as the verify receives it: the host store's bytes copied to the device and
 * decoded by the stream codec's GPU kernel (ss_options.compress_stream), natural [N x K] bf16 bits ->
 * out.  out_mode: -1 plain bf16, 0 raw blob, 1 exponent-coded; out_stream_bytes: bytes streamed per
 * step for this group (either may be NULL).  Needs an idle ring (before the first prefill).
 * Errors: INVALID (resident group), STRUCTURE. */
ss_status ss_debug_decode_group(ss_ctx* ctx, int32_t layer, int32_t group, uint16_t* out, int32_t* out_mode,
                                uint64_t* out_stream_bytes);
/* Time launches of a matrix kernel with M tokens: average device ms per launch over `iters` rounds
 * (CUDA events on the compute stream).  which 0: the draft GEMV (K2 on substitutes, bf16 GEMV on
 * resident layers / the head), M <= 32; which 1: the target GEMM (K6) on resident layers or the head
 * (group -1, with the verify's per-tile argmax epilogue), M <= the verify rows.  layer -1: every
 * layer in turn; group -2: the four groups of each layer.  Errors: INVALID, STRUCTURE (which 1 on
 * an offloaded layer). */
ss_status ss_debug_time_matmul(ss_ctx* ctx, int32_t which, int32_t layer, int32_t group, int32_t M, int32_t iters,
                               float* out_ms);

/* Debug A/B switch of the kernels (tests and tools only): knob 2 = the K6 kernel variant (0 default:
 * tcgen05 with whole-chunk stages; 1: legacy mma.sync; 2: tcgen05 with half-chunk stages).  Captured
 * draft graphs are dropped.  Errors: INVALID (unknown knob or value). */
ss_status ss_debug_set_knob(ss_ctx* ctx, int32_t knob, int32_t value);
/* Time the draft forward of M frontier nodes (one draft pass incl. head, no top-k): average device ms
 * over `iters` eager launches.  skip: bit mask of kernel classes left out (1 attention, 2 RMSNorm,
 * 4 dequant-GEMVs, 8 head) — attribution only; results are not meaningful when skip != 0. */
ss_status ss_debug_time_pass(ss_ctx* ctx, int32_t M, int32_t iters, int32_t skip, float* out_ms);
/* One traced draft pass: each dequant-GEMV launch records 16 %globaltimer events (ns) into
 * out[16*i .. 16*i+15] (0 entry, 1/2 producer/consumer dependency release, 3 first data, 4 loop end,
 * 5 flush, 6 kernel end, 7 loop end max, 8 cluster reduction done, 9-12 residual / norm barrier /
 * norm scale / epilogue done; unused events 0); *out_n = number of launches traced (<= cap, <= 512). */
ss_status ss_debug_trace_pass(ss_ctx* ctx, int32_t M, int64_t* out, int32_t cap, int32_t* out_n);
/* Two SubSpec steps (draft + verify + accept, one request) with CUDA events around every streamed
 * layer group (A4 / K7, App. E); the second is reported: out[8*i .. 8*i+7] = (item -
 * first item consumed by the reported step, layer, group, host bytes, copy start, copy end, compute
 * start, ring release) in ms from that step's start (negative: during the lead-in step; -1e9 = not in
 * the window); out_phases[0..2] = draft end, verify end, accept end.  *out_n = rows (<= cap). */
ss_status ss_debug_step_timeline(ss_ctx* ctx, const ss_draft_params* p, double* out, int32_t cap, int32_t* out_n,
                                 double* out_phases);
/* One draft pass (non-fused) with a per-CTA trace of its `launch`-th dequant-GEMV launch (0 = layer
 * 0 qkv, 1 = layer 0 o, ...): out[5*i .. 5*i+4] = (SM id, entry, first data, main loop end, end) of
 * CTA i, %globaltimer ns; *out_n = CTAs recorded (<= cap <= 1638). */
ss_status ss_debug_cta_trace(ss_ctx* ctx, int32_t M, int32_t launch, int64_t* out, int32_t cap, int32_t* out_n);

#ifdef __cplusplus
}
#endif
#endif /* SUBSPEC_H */
