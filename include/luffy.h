/* luffy.h -- C ABI of libluffy: the token-condensed expert-parallel MoE layer of Luffy
 * (arXiv 2411.15419, "Communication-Efficient Sparsely-Activated Model Training via Sequence Migration
 * and Token Condensation"), forward and backward, hand-written CUDA for sm_100a (B200).
 *
 * Citations: P:n = PAPER.md line n (LaTeX source of the paper).  Readings Rn = DESIGN.md section 2.
 *
 * ---------------------------------------------------------------------------------------------------
 * General conventions
 *  - Every device pointer is caller-owned (e.g. allocated by PyTorch).  The library never allocates
 *    device memory after luffy_layer_create; all scratch lives in the caller's workspace.
 *  - Calls taking `stream` (a cudaStream_t passed as void*) are stream-ordered and asynchronous unless
 *    marked [sync].  Host pointers are marked (host); all other pointers are device pointers.
 *  - Row-major, rows 16-byte aligned: d_model % 8 == 0 and d_ffn % 8 == 0 (bf16) / % 4 (fp32).
 *    Element type of activations/weights = luffy_config.dtype (bf16 or fp32); gate weights, gate
 *    outputs and weight gradients are fp32.
 *  - Weights use the nn.Linear layout (out x in): W_g [E, d]; W1, W3 [E_l, f, d]; W2 [E_l, d, f],
 *    where E_l = E / world local experts on this rank (contiguous placement, R14: expert e lives on
 *    rank e / E_l).
 *  - ROW LAYOUT ("slot" space).  Per-row expert buffers are expert-major and every expert segment is
 *    padded to a multiple of LUFFY_ROW_ALIGN rows; padding rows are zero in every buffer the library
 *    writes.  On the source side a slot is the padded position of a representative in its send
 *    layout (expert asc, then token asc, R15).  On the expert side (recv / expert_out) the segment of
 *    local expert e holds source rank 0's rows, then rank 1's, ... then zero padding.  With world == 1
 *    the two layouts coincide: recv == send, expert_out == gathered.
 *  - world > 1 (expert parallel, one process per GPU): the exchange is device-initiated over NVLink.
 *    luffy_layer_create allocates the layer's peer-visible exchange region (recv x2, gathered, d_expert,
 *    d_send, counts, flags); the caller all-gathers the ranks' luffy_layer_ipc_handle blobs (e.g. with
 *    torch.distributed) and passes them to luffy_layer_ipc_open.  The pack kernel, the GEMM2 / dgrad1
 *    epilogues and the uncondense backward then store rows straight into the destination rank's buffer
 *    and publish per-step sequence flags (system-scope release); consumers wait on the device (acquire),
 *    so no host synchronisation is needed.  The step number the flags carry lives in device memory and is
 *    advanced by luffy_route's first launch, so a step (luffy_route .. luffy_route_bwd, no sequence
 *    migration) captured in a CUDA graph replays correctly; the receive buffers alternate by step
 *    parity, so capture two consecutive steps and replay them alternately.  With world > 1 the
 *    expert-side and gathered buffer arguments are NULL (the layer's exchange buffers are used;
 *    luffy_layer_exchange_buffers returns them).  All ranks must issue the same sequence of calls.
 *  - Errors: arguments are validated on the host before anything is enqueued; on failure a status is
 *    returned, nothing is launched and luffy_last_error() describes the problem.  CUDA failures map to
 *    LUFFY_E_CUDA.  Calling out of order returns LUFFY_E_STATE.  A rank that stops participating does not
 *    hang or kill the others: every cross-rank wait is bounded (luffy_layer_set_exchange_timeout, default
 *    20 s); on expiry the waiting kernel records the phase and step in the layer's error word and
 *    completes (that step's results are garbage), and every later luffy_* call on the layer returns
 *    LUFFY_E_STATE naming the phase -- the CUDA context stays usable.
 *  - Determinism: identical inputs give bitwise-identical outputs (no floating-point atomics).
 *  - Thread-compatibility: one thread at a time per luffy_ctx.
 * ------------------------------------------------------------------------------------------------- */
#ifndef LUFFY_H_
#define LUFFY_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define LUFFY_API __attribute__((visibility("default")))
#else
#define LUFFY_API
#endif

#define LUFFY_ROW_ALIGN 128
#define LUFFY_MAX_EXPERTS 256

typedef enum {
  LUFFY_OK = 0,
  LUFFY_E_INVALID = 1,      /* bad argument (shape, alignment, null pointer, range) */
  LUFFY_E_CUDA = 2,         /* a CUDA runtime call failed */
  LUFFY_E_NCCL = 3,         /* reserved (the exchange does not use NCCL) */
  LUFFY_E_CAPACITY = 4,     /* a receive / migration capacity would be exceeded (checked before any transfer) */
  LUFFY_E_UNSUPPORTED = 5,  /* configuration not supported by this build (e.g. no sm_100a device) */
  LUFFY_E_STATE = 6         /* call order violated (e.g. combine before dispatch) */
} luffy_status;

typedef enum { LUFFY_FP32 = 0, LUFFY_BF16 = 1 } luffy_dtype;
typedef enum { LUFFY_GELU = 0, LUFFY_SWIGLU = 1 } luffy_act;

typedef struct {
  int32_t world;          /* ranks of the expert-parallel group (1 = single GPU) */
  int32_t rank;           /* this rank, 0 <= rank < world */
  int32_t num_experts;    /* E, E % world == 0, E <= LUFFY_MAX_EXPERTS */
  int32_t top_k;          /* k, 1 <= k <= E ("top-2 gating") */
  int32_t d_model;        /* d */
  int32_t d_ffn;          /* f */
  int32_t dtype;          /* luffy_dtype of activations and expert weights */
  int32_t act;            /* luffy_act of the expert FFN (R12) */
  int32_t renormalize;    /* 1: gate weights renormalized over the k selected experts; 0: raw softmax
                             probability; -1: default (top_k > 1), R1 */
  int32_t max_tokens;     /* T capacity per rank */
  int32_t max_recv_rows;  /* expert-side row capacity incl. padding; 0: world*max_tokens*top_k + E_l*LUFFY_ROW_ALIGN */
  int32_t max_seqs;       /* sequences per rank for sequence migration (world > 1); 0: 256 */
  int32_t fast_measure;   /* 1: keep the state of the fast similarity measurement with history shortcuts
                             (luffy_layer_set_history; bf16 only); 0: off */
} luffy_config;

typedef struct luffy_ctx luffy_ctx;     /* per rank: config and device */
typedef struct luffy_layer luffy_layer; /* per MoE layer call chain: saved routing/condensation/layout */

typedef struct {
  int64_t copies;                 /* T * k token copies */
  int64_t reps;                   /* representatives R (rows that are dispatched and run by experts) */
  int64_t ambiguous_pairs;        /* pairs i < j of a group with |s_ij - h| <= 1e-5 (R18), from the fp32 Gram */
  int64_t near_tie_tokens;        /* tokens whose k+1 largest logits have an adjacent gap <= 1e-5 max(1,|l_1|) (R2) */
  int64_t decided_pairs;          /* fast measurement: pairs i < j decided by the previous block (not measured) */
  int64_t skipped_tiles;          /* fast measurement: 256x256 Gram tiles skipped (every pair decided) */
  int32_t rounds;                 /* parallel selection rounds used */
  int32_t reps_per_expert[LUFFY_MAX_EXPERTS];
  int32_t copies_per_expert[LUFFY_MAX_EXPERTS];
} luffy_condense_stats;

/* ---- lifetime ---------------------------------------------------------------------------------- */

/* Validates cfg and binds the context to the current CUDA device (must be sm_100).  [sync] */
LUFFY_API luffy_status luffy_create(const luffy_config* cfg, luffy_ctx** out);
LUFFY_API void luffy_destroy(luffy_ctx* ctx);

/* Bytes of device workspace one layer needs (saved state + scratch), a function of cfg only. */
LUFFY_API size_t luffy_layer_workspace_bytes(const luffy_config* cfg);

/* Binds a layer to `dev_workspace` (device, >= luffy_layer_workspace_bytes, 256-byte aligned).  With
 * world > 1 it also allocates the layer's exchange region (cudaMalloc; freed by luffy_layer_destroy).
 * [sync] */
LUFFY_API luffy_status luffy_layer_create(luffy_ctx* ctx, void* dev_workspace, size_t bytes, luffy_layer** out);
LUFFY_API void luffy_layer_destroy(luffy_layer* layer);

/* world > 1: size of one IPC handle blob; this rank's blob (host out[luffy_ipc_handle_bytes()]); and the
 * mapping of every rank's region from the all-gathered blobs (host [world][bytes], rank order).  [sync] */
LUFFY_API size_t luffy_ipc_handle_bytes(void);
LUFFY_API luffy_status luffy_layer_ipc_handle(const luffy_layer* layer, uint8_t* out);
LUFFY_API luffy_status luffy_layer_ipc_open(luffy_layer* layer, const uint8_t* all_handles);

/* world > 1: the layer's exchange buffers for the current step (any pointer argument may be NULL):
 * recv / d_expert_out [max_recv_rows, d] expert layout, gathered / d_send [send rows, d] send layout. */
LUFFY_API luffy_status luffy_layer_exchange_buffers(const luffy_layer* layer, void** recv, void** gathered,
                                                    void** d_expert_out, void** d_send);

/* Thread-local description of the last failure. */
LUFFY_API const char* luffy_last_error(void);

/* Number of CUDA kernels this library has launched in this process (for the bench's gpu_launches). */
LUFFY_API int64_t luffy_launch_count(void);

/* Programmatic dependent launch for every following launch of the process (default on, or off with
 * LUFFY_PDL=0).  Off: each kernel's device duration excludes the wait for its predecessor, which is what a
 * per-kernel timing table needs; results are identical either way. */
LUFFY_API void luffy_debug_set_pdl(int32_t on);

/* Padded row counts after the forward calls (host, valid after luffy_dispatch returned):
 * send_rows = padded rows of this rank's send layout; recv_rows = padded rows of its expert layout. */
LUFFY_API luffy_status luffy_layer_rows(const luffy_layer* layer, int64_t* send_rows, int64_t* recv_rows);

/* ---- forward (P:256-259 workflow: gate -> condensation -> dispatch -> experts -> combine) -------- */

/* Top-k gate, P:152/P:434 and R1/R2.  x [T, d] (dtype), w_gate [E, d] fp32.
 * logits = x W_g^T in fp32 with a fixed summation order; experts ordered by (logit desc, id asc);
 * topk_w = renormalized softmax over the k selected logits, or the softmax probability (R1).
 * Outputs topk_idx [T, k] int32 and topk_w [T, k] fp32 (device); the layer keeps copies for backward.
 * Starts a new forward on the layer.  0 < T <= max_tokens. */
LUFFY_API luffy_status luffy_route(luffy_layer* layer, const void* x, const float* w_gate, int32_t T,
                         int32_t* topk_idx, float* topk_w, void* stream);

/* Token condensation, P:358 (group = tokens routed to the same expert), P:373 (cosine similarity of the
 * remaining pairs), P:378 (threshold, then keep the highest-degree token and condense its neighbours,
 * repeat), P:405 (token_to_token map).  Normalized cosine s = (1 + cos)/2 (R4); edge iff s >= h;
 * zero vectors have no edges (R7); greedy on the dynamic residual degree with ties to the lowest token
 * (R8), computed exactly by parallel 2-hop rounds.  h > 1 disables condensation (identity map).
 * Output rep [T, k] int32: the token whose copy represents copy (t, j) in expert topk_idx[t, j]
 * (rep[rep] == rep).  `stats` (host, nullable) is filled synchronously when non-NULL ([sync] then); the
 * near-tie report recomputes candidate logits from x and the w_gate passed to this step's luffy_route,
 * which must still be valid. */
LUFFY_API luffy_status luffy_condense(luffy_layer* layer, const void* x, float h, int32_t* rep,
                            luffy_condense_stats* stats, void* stream);

/* Fast similarity measurement, P:359-373 (needs luffy_config.fast_measure = 1, bf16).  Step 2:
 * in this layer's following luffy_condense calls, a pair of tokens of one expert group whose finalized
 * weight in `prev`'s last condensation (the previous block) was > S1 gets weight 1, < S2 weight 0, without
 * measuring it (reading R20: history exists for pairs that shared an expert in prev; the first shared
 * expert in the row token's top-k order is read); the rest are measured (step 3).  Every condense
 * of a fast_measure layer records its own finalized weights' classification (> S1, < S2; shortcut values
 * included, reading R21) for the next block.  Gram tiles whose pairs are all decided are skipped.
 * prev: NULL (first block: classification only) or a fast_measure layer condensed earlier in the same
 * step on the SAME tokens in the same order (its T must equal this layer's T).  0 <= S2 < S1 <= 1. */
LUFFY_API luffy_status luffy_layer_set_history(luffy_layer* layer, const luffy_layer* prev, float S1, float S2);

/* Dispatch phase: packs only the representatives.  world == 1: into `recv` (the send
 * layout is the expert layout).  world > 1 (recv = NULL): the representative counts are pushed to every
 * rank, every rank derives all layouts on the device, and one fused kernel copies each representative
 * row from x straight into its expert's rank's receive buffer over NVLink; the call then waits (on the
 * device) for every rank's rows.  recv_rows (host, nullable): padded expert-layout rows ([sync]).
 * Capacity: max_recv_rows defaults to the worst case (every copy of every rank to this rank). */
LUFFY_API luffy_status luffy_dispatch(luffy_layer* layer, const void* x, void* recv, int64_t* recv_rows, void* stream);

/* Expert FFN ("expert networks that are essentially FFNs"; R12):
 * GELU:   pre = recv W1_e^T, act = GeLU_erf(pre), out = act W2_e^T;
 * SWIGLU: pre = [recv W1_e^T | recv W3_e^T] (saved_pre is [rows, 2f]), act = silu(pre1) * pre3.
 * bf16: tcgen05 grouped GEMMs, fp32 accumulation, bf16 outputs.  fp32: SIMT FFMA.
 * saved_pre [rows, f or 2f] and saved_act [rows, f] are written for the backward: for GELU saved_pre holds
 * GeLU'(pre) (the only function of pre the backward needs; computed with the same erf as the forward),
 * for SWIGLU the pre-activations [pre1 | pre3].  w3 NULL for GELU. */
LUFFY_API luffy_status luffy_expert_ffn(luffy_layer* layer, const void* recv, const void* w1, const void* w2,
                              const void* w3, void* out, void* saved_pre, void* saved_act, void* stream);

/* Combine phase: expert outputs in this rank's send layout (`gathered`).  world == 1: gathered
 * may alias expert_out (no-op) or is a copy.  world > 1: luffy_expert_ffn's GEMM2 epilogue already
 * stored every row into its source rank's gathered buffer over NVLink (fused combine); this call waits
 * for every rank's rows (expert_out and gathered may be NULL). */
LUFFY_API luffy_status luffy_combine(luffy_layer* layer, const void* expert_out, void* gathered, void* stream);

/* Output reuse, "use the expert output of token j to replace it" (R10):
 * y[t] = sum_j topk_w[t, j] * gathered[slot of rep(t, j)], fp32 accumulation, y [T, d] (dtype). */
LUFFY_API luffy_status luffy_uncondense(luffy_layer* layer, const void* gathered, void* y, void* stream);

/* Residual block (a transformer block's MoE sub-layer, y = x + MoE(x)): luffy_uncondense with the residual
 * branch added in the same pass, y[t] = x[t] + sum_j topk_w[t, j] * gathered[slot of rep(t, j)].  x is the
 * layer input of luffy_route ([T, d], this rank's tokens).  With sequence migration the x rows of every
 * token are pushed to the rank hosting its sequence (device-initiated, like the combine) and y holds the
 * hosted tokens (luffy_migration_out_tokens order).  The backward counterpart is
 * luffy_dispatch_bwd_residual. */
LUFFY_API luffy_status luffy_uncondense_residual(luffy_layer* layer, const void* gathered, const void* x, void* y,
                                                 void* stream);

/* ---- backward: exact autograd of the forward with routing and rep as constants (R11) ------------- */

/* d_gathered[slot] = sum over copies (t, j) represented by the slot (token order) of w[t,j] * dy[t];
 * padding slots are zeroed.  d_topk_w [T, k] fp32 = <dy[t], gathered[slot(t, j)]>. */
LUFFY_API luffy_status luffy_uncondense_bwd(luffy_layer* layer, const void* dy, const void* gathered,
                                  void* d_gathered, float* d_topk_w, void* stream);

/* Mirror of luffy_combine: d_expert_out (expert layout) <- d_gathered (send layout). */
LUFFY_API luffy_status luffy_combine_bwd(luffy_layer* layer, const void* d_gathered, void* d_expert_out, void* stream);

/* FFN backward: d_act = d_out W2; d_pre = d_act * act'(pre); d_recv = d_pre W1 (+ d_pre3 W3);
 * dw2 = d_out^T act; dw1 = d_pre^T recv (dw3 = d_pre3^T recv).  dw* fp32, overwritten.
 * `scratch_dpre` [rows, f or 2f] (dtype) receives d_pre.  dw3 / w3 NULL for GELU. */
LUFFY_API luffy_status luffy_expert_ffn_bwd(luffy_layer* layer, const void* d_out, const void* recv, const void* w1,
                                  const void* w2, const void* w3, const void* saved_pre,
                                  const void* saved_act, void* scratch_dpre, void* d_recv,
                                  float* dw1, float* dw2, float* dw3, void* stream);

/* Mirror of luffy_dispatch: d_send (send layout, internal for world > 1) <- d_recv (expert layout),
 * then dx[t] = sum over j with rep(t, j) == t of d_send[slot(t, j)] (dx overwritten, dtype). */
LUFFY_API luffy_status luffy_dispatch_bwd(luffy_layer* layer, const void* d_recv, void* dx, void* stream);

/* luffy_dispatch_bwd for a residual block: dx[t] = dy[t] + (expert-path gradient of x[t]).  dy: the dY
 * given to luffy_uncondense_bwd (home order [T, d]); with sequence migration pass NULL (the dY rows the
 * hosts returned to this rank are used).  Follow with luffy_route_bwd as usual (it accumulates). */
LUFFY_API luffy_status luffy_dispatch_bwd_residual(luffy_layer* layer, const void* d_recv, const void* dy, void* dx,
                                                   void* stream);

/* Gate backward: renormalized: dl_j = w_j (dw_j - sum_i w_i dw_i) on the top-k; raw softmax:
 * dl = p * (g - <p, g>); dw_gate [E, d] fp32 = dl^T x (overwritten); dx += dl W_g (accumulated). */
LUFFY_API luffy_status luffy_route_bwd(luffy_layer* layer, const void* x, const float* w_gate, const float* d_topk_w,
                             void* dx, float* dw_gate, void* stream);

/* Host export of the dispatch/combine plan (P:143 dispatch, P:144 combine; R14/R15).  The device count
 * exchange inside luffy_dispatch (world > 1) derives its layout with the SAME code (csrc/xplan.h, one
 * __host__ __device__ definition), so this call returns exactly the plan the kernels use.
 * counts_all [P][E] (host): representatives each source rank sends to each expert.  Outputs (host):
 * send_off [E+1]  padded send layout of `rank` (expert asc, each segment rounded up to LUFFY_ROW_ALIGN);
 * recv_off [E_l+1] padded expert layout of `rank` (local expert asc; within a segment source rank asc);
 * dst_base [E] (nullable): first row, in expert e's owner's layout, of the rows `rank` sends to e (the
 *   dispatch push writes send slot s of expert e to row dst_base[e] + s - send_off[e] there);
 * rank_of / slot_of [row_capacity] (nullable, together): for every expert-layout row r < recv_off[E_l] of
 *   `rank`, the source rank and its send slot (the combine returns row r there); -1 for padding rows;
 *   LUFFY_E_CAPACITY if recv_off[E_l] > row_capacity;
 * send_rows_to [P] / recv_rows_from [P] (nullable): rows exchanged with each peer (self included). */
LUFFY_API luffy_status luffy_exchange_plan(int32_t world, int32_t rank, int32_t num_experts, const int32_t* counts_all,
                                           int32_t* send_off, int32_t* recv_off, int32_t* dst_base, int32_t* rank_of,
                                           int32_t* slot_of, int64_t row_capacity, int64_t* send_rows_to,
                                           int64_t* recv_rows_from);

/* world > 1: bound (milliseconds, > 0) of every cross-rank wait of the layer's exchange; default 20000 or
 * the environment variable LUFFY_EXCHANGE_TIMEOUT_MS read at luffy_layer_create. */
LUFFY_API luffy_status luffy_layer_set_exchange_timeout(luffy_layer* layer, int64_t ms);

/* ---- debug export (tests) ----------------------------------------------------------------------- */

typedef enum {
  LUFFY_DBG_GCNT = 0,      /* int32 [E]     copies per expert group */
  LUFFY_DBG_GOFF = 1,      /* int32 [E+1]   padded group-row offsets */
  LUFFY_DBG_GTOK = 2,      /* int32 [goff[E]] token of each group row (-1 padding) */
  LUFFY_DBG_ADJOFF = 3,    /* int64 [E+1]   word offsets of the group adjacency bit matrices */
  LUFFY_DBG_ADJ = 4,       /* uint32 [adjoff[E]] adjacency bits (row r of group e: adjoff[e] + r * npad_e/32) */
  LUFFY_DBG_REP_LOCAL = 5, /* int32 [goff[E]] group row of each row's representative */
  LUFFY_DBG_SOFF = 6,      /* int32 [E+1]   padded send offsets */
  LUFFY_DBG_PERM = 7,      /* int32 [soff[E]] slot -> token (-1 padding) */
  LUFFY_DBG_POS = 8,       /* int32 [T, k]  slot of the representative of copy (t, j) */
  LUFFY_DBG_NREP = 9,      /* int32 [E]     representatives per expert */
  LUFFY_DBG_ROUNDS = 10,   /* uint32 [1]    greedy rounds of the last condense */
  LUFFY_DBG_GREEDY_TIMES = 11, /* uint32 [64] greedy control block: [3] = #stamps, [8+2i..9+2i] = %globaltimer ns at barrier i */
  LUFFY_DBG_HONE = 12,     /* uint32 [adjoff[E]] fast measurement: this block's finalized weight > S1 (adj layout) */
  LUFFY_DBG_HZERO = 13,    /* uint32 [adjoff[E]] finalized weight < S2 */
  LUFFY_DBG_DEC1 = 14,     /* uint32 [adjoff[E]] pairs decided by the previous block with weight 1 */
  LUFFY_DBG_DEC0 = 15,     /* uint32 [adjoff[E]] pairs decided by the previous block with weight 0 */
  LUFFY_DBG_TSKIP = 16     /* uint8 [tiles] skipped Gram tiles (pair tiles in upper-triangle order per group) */
} luffy_debug_item;

/* Synchronously copies an internal array of the layer's current forward to host memory `dst` (host).
 * *bytes (in: capacity of dst, out: bytes of the item).  [sync] */
LUFFY_API luffy_status luffy_debug_copy(luffy_layer* layer, int32_t item, void* dst, size_t* bytes, void* stream);

/* Registers a device buffer (16-byte aligned, capacity in floats; NULL unregisters) that every following
 * luffy_condense fills with the fp32 similarity Gram the threshold is applied to (tests: A18's
 * max |s_gpu - s_ref| check): group e occupies floats [adjoff[e] * 32, + npad_e^2) as a dense row-major
 * [npad_e][npad_e] matrix (npad_e = goff[e+1] - goff[e]); only 32x32 blocks with column block >= row
 * block are written (the matrix is symmetric); blocks beyond the capacity are skipped. */
LUFFY_API luffy_status luffy_debug_gram_dump(luffy_layer* layer, float* dst, size_t capacity_floats);

/* Grouped GEMM used by the expert FFN, exposed for unit tests.  kind 0 ("rows"): D[r, :N] over the
 * row segments off[0..G] (device, multiples of LUFFY_ROW_ALIGN) = A[r, :K] B_g^T with the epilogue `epi`
 * (0 store, 1 GeLU: aux = pre, 2 SwiGLU, 3 GeLU', 4 SwiGLU'); b_kmajor: B_g is [N, K], else [K, N].
 * kind 1 ("wgrad"): D_g[M, N] (fp32) = sum over segment rows of A[r, :M]^T B[r, :N]; here K is the leading
 * dimension of A (lda) and rows m >= Msplit go to D3.  dtype selects tcgen05 (bf16) or SIMT (fp32). */
LUFFY_API luffy_status luffy_debug_gemm(int32_t kind, int32_t dtype, int32_t epi, const void* A, const void* B,
                                        const void* B3, void* D, void* aux, float* D3, int32_t Msplit,
                                        const int32_t* off, int32_t G, int64_t max_rows, int32_t M, int32_t N,
                                        int32_t K, int32_t b_kmajor, void* stream);

/* ---- sequence migration in the layer (world > 1), P:264-299 -------------------------------------- */

/* K9: after luffy_condense and before luffy_dispatch.  seq_len (host, [num_seqs], sums to T) splits this
 * rank's tokens into sequences; num_seqs_all (host, [world], nullable = every rank has num_seqs) gives every
 * rank's sequence count.  Returns rows_at_all (host, [sum of num_seqs_all][world], every rank's sequences in
 * rank order): the number of DISTINCT representative rows each sequence uses on each rank (reading R16;
 * Alg. 1 line 1 input).  Every rank gets the same table (device exchange).  [sync] */
LUFFY_API luffy_status luffy_sequence_rows(luffy_layer* layer, const int32_t* seq_len, int32_t num_seqs,
                                           const int32_t* num_seqs_all, int64_t* rows_at_all, void* stream);

/* Registers the placement of this step (e.g. from luffy_plan_migration, run identically on every rank):
 * seq_len_all / seq_dest (host, [sum of num_seqs_all], rank order as in luffy_sequence_rows).  The combine then delivers each expert-output row to
 * every rank hosting a sequence that uses it (GEMM2 epilogue over NVLink); luffy_uncondense writes the
 * tokens this rank hosts (*out_rows of them, host) in (home rank, sequence, token) order -- see
 * luffy_migration_out_tokens; luffy_uncondense_bwd takes dY in that order and returns dY / d(gate weight)
 * to the home ranks.  Before luffy_dispatch.  Stream-ordered: the per-sequence tables are copied from the
 * layer's pinned staging buffer without a stream synchronisation (the call only waits, if at all, for the
 * previous call's copy to have left that buffer). */
LUFFY_API luffy_status luffy_set_migration(luffy_layer* layer, const int32_t* seq_len_all, const int32_t* seq_dest,
                                           int64_t* out_rows, void* stream);

/* (home rank, home token index) of each output row of this rank (host [out_rows]; either may be NULL).
 * After luffy_combine; synchronize the stream first.  [sync] */
LUFFY_API luffy_status luffy_migration_out_tokens(const luffy_layer* layer, int32_t* home_rank, int32_t* home_token);

/* ---- sequence migration placement (CPU, host memory, synchronous, reentrant, deterministic) ------ */

typedef struct {
  int32_t num_seqs;          /* S */
  int32_t num_ranks;         /* P */
  int32_t q;                 /* candidate-set size, Alg. 1 line 2 */
  int32_t objective;         /* 0: minimum cost growth (default, R16); 1: maximum as printed */
  const int32_t* seq_len;    /* [S] sequence lengths l_i */
  const int64_t* rows_at;    /* [S][P] expert-output rows of sequence i located on rank j */
  int64_t row_bytes;         /* bytes per row (d * sizeof(dtype)) */
  int64_t capacity_tokens;   /* per-rank token capacity; <= 0: max(ceil(1.5*sum(l)/P), max l) */
  int64_t d_model;           /* d of Eq. (1) */
} luffy_migration_problem;

/* Alg. 1 with Eq. (1) in exact int64 arithmetic (P := 1, R16): f_ij = row_bytes *
 * (rows_i - rows_at[i][j]); H_i = q ranks of least f (ties -> lower rank); sequences by length desc
 * (ties -> id asc) go to the capacity-feasible j in H_i of least s_ij = T_att(B_j+1, max(L_j, l_i)) -
 * T_att(B_j, L_j) (ties -> smaller f, then lower rank), else to any feasible rank by the same key,
 * else LUFFY_E_CAPACITY.  seq_dest [S] (host) receives the ranks; combine_bytes [P][P] (host, nullable)
 * the predicted combine traffic from rank r to rank dest. */
LUFFY_API luffy_status luffy_plan_migration(const luffy_migration_problem* prob, int32_t* seq_dest, int64_t* combine_bytes);

/* Eq. (1): 3*B*L*d^2 + 2*B*L^2*d (P := 1), exact int64. */
LUFFY_API int64_t luffy_attention_cost(int64_t B, int64_t L, int64_t d);

/* Adaptive condensation threshold, Eq. (2), P:384-387 (the step before the hot path; the layer takes h as
 * an argument): h_t = c / (1 + exp(l_norm)), l_norm = max(0, (l_ini - l_prev) / l_ini), with c = 1 as
 * printed (h in (0.269, 0.5]) or, reading R17b, c = 2 (h in [0.538, 1], the range the paper's narrative and
 * Table IV imply).  scale2 selects c = 2.  Host, pure; LUFFY_E_INVALID for l_ini <= 0 or non-finite inputs. */
LUFFY_API luffy_status luffy_adaptive_threshold(double l_ini, double l_prev, int32_t scale2, float* h_out);

#ifdef __cplusplus
}
#endif
#endif /* LUFFY_H_ */
