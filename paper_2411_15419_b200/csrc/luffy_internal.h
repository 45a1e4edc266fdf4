// Internal declarations of libluffy (not part of the C ABI).
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>

#include "luffy.h"

namespace luffy {

luffy_status fail(luffy_status st, const std::string& msg);
void note_launch(int n = 1);

constexpr int kRowAlign = LUFFY_ROW_ALIGN;
constexpr int kGreedyMaxRounds = 1 << 14;
// token slices of the deterministic dW_g reduction: enough CTAs to stream X once, bounded scratch
inline int wg_parts(int E, int d) {
  int p = (1 << 22) / (E * d);
  return p < 16 ? 16 : (p > 128 ? 128 : p);
}

inline int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

}  // namespace luffy

#ifdef __CUDACC__
#include <cuda_runtime.h>
#endif

// Layer state: pointers into the caller's workspace (device) plus host-side bookkeeping.
struct luffy_layer {
  struct luffy_ctx* ctx;
  // ---- config copies
  int P, rank, E, El, k, d, f, dtype, act, renorm, Tmax;
  int64_t C_max, Cpad_max, Rpad_max, recv_max, adj_words_max;
  // ---- routing (saved for backward)
  float* probs;       // [Tmax, E]
  int32_t* idx;       // [Tmax, k]
  float* w;           // [Tmax, k]
  // ---- groups (one per expert; source rank = this rank)
  int32_t* gcnt;      // [E] copies per expert
  int32_t* goff;      // [E+1] padded group-row offsets
  int32_t* gtok;      // [Cpad_max] token of each group row (-1 = padding)
  int32_t* gloc;      // [Tmax, k] group row (global, padded space) of copy (t, j)
  int32_t* gcopy;     // [Cpad_max] copy t * k + j of each group row (-1 = padding)
  float* gw;          // [Cpad_max] gate weight of each group row (0 for padding)
  int32_t* gchunk;    // [ceil(Tmax / 128)][E] per-chunk copies per expert -> chunk prefixes (grouping)
  uint32_t* gticket;  // [1] last-CTA ticket of the grouping count (zero between launches)
  void* xg;           // [Cpad_max, d] gathered group rows (dtype)
  double* gnorm;      // [Cpad_max] |x| in fp64
  int64_t* adjoff;    // [E+1] word offsets of each group's bit adjacency
  uint32_t* adj;      // adjacency bits, group e: rows of W_e = goff-span/32 words
  int32_t* rep_local; // [Cpad_max] group row of the representative
  uint64_t* key;      // [Cpad_max] greedy priorities
  uint64_t* m1;       // [Cpad_max]
  uint64_t* m2;       // [Cpad_max]
  uint32_t* alive;    // [Cpad_max/32]
  uint32_t* win;      // [Cpad_max/32]
  uint32_t* ctrl;     // [64 + kGreedyMaxRounds] grid barrier + per-round counters
  // ---- fast similarity measurement (config fast_measure, readings R20/R21), adj layout
  bool fast_measure;
  uint32_t* hone;     // this block's finalized weight > S1 (history for the next block)
  uint32_t* hzero;    // this block's finalized weight < S2
  uint32_t* dec1;     // pairs decided by the previous block: weight 1
  uint32_t* dec0;     //                                        weight 0
  uint8_t* tskip;     // [tiles] Gram tiles whose pairs are all decided
  const luffy_layer* hist_prev;  // previous block (luffy_layer_set_history), nullable
  float hist_S1, hist_S2;
  bool hist_valid;    // hone / hzero hold this step's classification
  // ---- pack / layout
  int32_t* nrep;      // [E] representatives per expert
  int32_t* gnrep;     // [E] representatives per group, published by representative selection
  bool gnrep_valid;   // set when the selection kernel of this step published gnrep
  int32_t* mrank;     // [Cpad_max] rank of each row in its representative's member list (token order)
  int32_t* mcnt_row;  // [Cpad_max] member-list length of each representative row
  bool mrank_valid;   // set when the selection kernel of this step published mrank / mcnt_row
  int32_t* soff;      // [E+1] padded send offsets
  int32_t* lslot;     // [Cpad_max] slot of a group row that is a representative (-1 otherwise)
  int32_t* perm;      // [Rpad_max] slot -> token (-1 = padding)
  int32_t* slot_gl;   // [Rpad_max] slot -> group row (-1 = padding)
  int32_t* pos;       // [Tmax, k] slot of the representative of copy (t, j)
  int32_t* rep;       // [Tmax, k] representative token of copy (t, j)
  int32_t* mstart;    // [Rpad_max] first member (group-row space) of each slot's member list
  int32_t* mcnt;      // [Rpad_max] members per slot
  int32_t* mcur;      // [Rpad_max] placement cursor
  int32_t* marr;      // [Rpad_max] arrivals of the window partials of a slot (uncondense backward)
  int32_t* members;   // [Cpad_max] member group rows, slot-major, token order within a slot
  int32_t* mslot;     // [Cpad_max] slot of each member entry (-1 = padding)
  float* mpart;       // [Cpad_max / 16 * 2, d] fp32 partial sums of slots crossing member windows
  int32_t* roff;      // [El+1] padded expert-side row offsets (device)
  int32_t* cnt_all;   // [P, E] all-gathered representative counts (device)
  void* send;         // [Rpad_max, d] send buffer (world > 1); reused as d_send in backward
  // ---- backward scratch
  float* dl;          // [Tmax, E] gate logit gradients
  float* rpart;       // [ceil(d / 1024), Tmax, E] split partial logits of the register-W_g gate (8 < E <= 32)
  float* wg_part;     // [kWgParts, E, d]
  const float* wg_route;  // w_gate of this step's luffy_route (the stats' near-tie report reads it)
  uint64_t* stat64;   // [4] device stats of the last condense: [0] near-threshold pairs, [1] near-tie tokens
  // ---- debug export
  float* dbg_gram;    // caller's device buffer for the fp32 Gram (luffy_debug_gram_dump), nullable
  size_t dbg_gram_cap;  // its capacity in floats
  // ---- host-side state
  int T;
  float h;
  bool has_adj;
  int stage;          // 0 none, 1 routed, 2 condensed, 3 dispatched, 4 ffn, 5 combined, 6 uncondensed
  int64_t send_rows_h, recv_rows_h;
  // ---- device-initiated exchange (world > 1), see exchange.cuh
  uint32_t seq;        // step sequence number (incremented by luffy_route)
  char* x_region;      // own peer-visible region (cudaMalloc, CUDA IPC)
  size_t x_region_bytes;
  uint8_t x_handle[64];
  void* x_peer_base_h[64];  // host: mapped base of every rank's region (own at [rank])
  bool x_open;
  uint32_t* x_err_h;     // [2] mapped pinned host memory: first timed-out exchange wait (phase + 1, seq)
  uint32_t* x_err_d;     // its device alias
  uint32_t* x_errw;      // [2] device copy polled by the waits (workspace)
  uint32_t* gdone;       // [E] Gram pair tiles finished per group (x2: both CTAs of a pair), zeroed by grouping
  bool gdone_live;       // the tensor-core Gram of this condense counts into gdone (the greedy waits on it)
  uint32_t* dseq;        // [1] device step sequence number (world > 1: bumped by luffy_route's first launch;
                         //     every exchange flag carries it, so a captured step replays correctly)
  uint64_t x_timeout_ns; // bound of every cross-rank wait (LUFFY_EXCHANGE_TIMEOUT_MS, luffy_layer_set_exchange_timeout)
  void* x_recv[2];     // own buffers inside the region
  void* x_gathered;
  void* x_dexp;
  void* x_dsend;
  int32_t* x_cnt_inbox;  // [P][E]
  uint32_t* x_flags;     // [XP_NUM][P]
  uint32_t* x_counters;  // [XP_NUM]
  // device tables (workspace)
  void** x_peer_recv;      // [2][P]
  void** x_peer_gathered;  // [P]
  void** x_peer_dexp;      // [P]
  void** x_peer_dsend;     // [P]
  int32_t** x_peer_cnt;    // [P]
  uint32_t** x_flagptr;    // [XP_NUM][P] -> (phase, my rank) slot in each rank's flags
  int32_t* x_dst_base;     // [E] destination row base of my rows of expert e in its owner's layout
  int32_t* x_src_soff;     // [P][E+1] padded send offsets of every rank
  int32_t* x_rank_of;      // [recv_max] source rank of each expert-layout row (-1 padding)
  int32_t* x_slot_of;      // [recv_max] its slot in the source's send layout
  // ---- sequence migration (world > 1), Alg. 1 decides seq_dest; migration.cu
  int Smax;                // sequence capacity per rank
  int S;                   // sequences of the current step (0 = not registered)
  int32_t Sq[64];          // sequences of every rank this step (luffy_sequence_rows)
  int32_t* mig_stage_h;    // pinned host staging [2 * Smax] (seq_dest, out_start) of luffy_set_migration
  void* mig_stage_ev;      // cudaEvent_t: the staging copy of the previous call has completed
  bool mig;                // seq_dest set for the current step
  int64_t n_out;           // output rows of this rank (tokens of the sequences it hosts)
  int32_t* seq_start;      // [Smax+1] token range of each of my sequences
  int32_t* seq_dest_l;     // [Smax] destination rank of each of my sequences
  int32_t* out_start;      // [Smax] first output row of each of my sequences at its destination
  uint32_t* seq_bits;      // [Smax][Rpad/32] distinct representative slots of each sequence (K9)
  int32_t* rows_local;     // [Smax][P]
  unsigned long long* dmask;  // [Rpad] destination ranks of each of my send slots
  unsigned long long* x_rowmask;  // region [recv_max]: destination mask of each expert row
  int32_t* x_mig_inbox;    // region [P][Smax][P] rows_at of every rank
  int32_t* x_meta;         // region [P*Tmax][2 + k] (home rank, home token, pos[k]) of my output rows
  float* x_meta_w;         // region [P*Tmax][k]
  void* x_dy_in;           // region [Tmax][d] dY of my tokens returned by their destinations
  void* x_res;             // region [P*Tmax][d] residual rows x of the tokens this rank hosts
  void** x_peer_res;       // [P]
  float* x_dw_in;          // region [Tmax][k]
  unsigned long long** x_peer_rowmask;  // [P]
  int32_t** x_peer_mig;    // [P]
  int32_t** x_peer_meta;   // [P]
  float** x_peer_meta_w;   // [P]
  void** x_peer_dy_in;     // [P]
  float** x_peer_dw_in;    // [P]
};

// ---- kernel launchers (defined in the .cu files); all enqueue on `s` and return cudaError_t as int
namespace luffy {
struct Ctx;
int launch_route(const luffy_layer* L, const void* x, const float* wg, int32_t* idx_out, float* w_out, void* s);
int launch_group_build(luffy_layer* L, const void* x, void* s);
int launch_identity_rep(luffy_layer* L, void* s);
int launch_gram_simt(luffy_layer* L, float h, unsigned long long* band, void* s);
int launch_gram_tc(luffy_layer* L, float h, unsigned long long* band, void* s);
int launch_near_tie(const luffy_layer* L, const void* x, const float* wg, unsigned long long* out, void* s);
int launch_greedy(luffy_layer* L, void* s);
int launch_pack(luffy_layer* L, const void* x, void* dst_rows, int32_t* rep_out, void* s);
int launch_uncondense(const luffy_layer* L, const void* gathered, const void* res, void* y, void* s);
int launch_uncondense_bwd(const luffy_layer* L, const void* dy, const void* gathered, void* dg, float* dw, void* s);
int launch_unpack_bwd(const luffy_layer* L, const void* dsend, const void* res, void* dx, void* s);
int launch_route_bwd(const luffy_layer* L, const void* x, const float* wg, const float* dw, void* dx, float* dwg, void* s);
int launch_xdispatch(luffy_layer* L, const void* x, void* s);
int launch_xwait(const luffy_layer* L, int phase, void* s);
int launch_xstep(const luffy_layer* L, void* s);
int launch_seq_rows(luffy_layer* L, void* s);
int launch_set_migration(luffy_layer* L, void* s);
int launch_mig_meta_push(luffy_layer* L, void* s);
int launch_uncondense_mig(const luffy_layer* L, const void* x_res, void* y, void* s);
int launch_mig_bwd_push(const luffy_layer* L, const void* dy, void* s);

// Grouped GEMM epilogues (gemm_simt.cu / gemm_tc.cu).  EPI_GELU stores GeLU(acc) and aux = GeLU'(acc);
// EPI_DGELU multiplies by that aux.
enum Epi { EPI_STORE = 0, EPI_GELU = 1, EPI_SWIGLU = 2, EPI_DGELU = 3, EPI_DSWIGLU = 4 };
}  // namespace luffy
