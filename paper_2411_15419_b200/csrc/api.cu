// C ABI of libluffy (include/luffy.h): context, workspace layout, argument validation, call order and
// the expert-parallel exchange (NCCL over NVLink) between the kernels.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "nccl_shim.h"

struct luffy_ctx {
  luffy_config cfg;
  int device;
  luffy::nccl::CommPtr comm;
};

namespace luffy {

static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};

luffy_status fail(luffy_status st, const std::string& msg) {
  g_err = msg;
  return st;
}
void note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int gemm_rows_simt(int dtype, int epi, const void* A, const void* B, const void* B3, void* D, void* aux0,
                   const int32_t* off, int G, int64_t max_rows, int N, int K, int b_kmajor, void* s);
int gemm_wgrad_simt(int dtype, const void* A, const void* B, float* D, float* D3, int Msplit, const int32_t* off, int G,
                    int M, int N, int lda, int ldb, void* s);
int gemm_rows_tc(int epi, const void* A, const void* B, const void* B3, void* D, void* aux0, const int32_t* off, int G,
                 int64_t max_rows, int N, int K, int b_kmajor, void* s);
int gemm_wgrad_tc(const void* A, const void* B, float* D, float* D3, int Msplit, const int32_t* off, int G, int M, int N,
                  int lda, int ldb, int64_t max_rows, void* s);
int launch_pack_rows(luffy_layer* L, const void* x, void* dst_rows, void* s);

namespace {

luffy_status cuda_fail(int err, const char* where) {
  if (err == 0) return LUFFY_OK;
  return fail(LUFFY_E_CUDA, std::string(where) + ": " + cudaGetErrorString((cudaError_t)err));
}
#define LUFFY_CHECK(expr, where)                           \
  do {                                                     \
    int _r = (expr);                                       \
    if (_r != 0) return cuda_fail(_r, where);              \
  } while (0)

luffy_status nccl_fail(nccl::Result r, const char* where) {
  const nccl::Api* a = nccl::api();
  return fail(LUFFY_E_NCCL, std::string(where) + ": " + (a ? a->GetErrorString(r) : "NCCL unavailable"));
}
#define LUFFY_NCCL(expr, where)                            \
  do {                                                     \
    nccl::Result _r = (expr);                              \
    if (_r != 0) return nccl_fail(_r, where);              \
  } while (0)

size_t elem_size(int dtype) { return dtype == LUFFY_BF16 ? 2 : 4; }

// Workspace carve: identical walk for sizing (base == nullptr) and binding.
struct Carver {
  char* base;
  size_t off = 0;
  template <typename T>
  T* take(size_t count) {
    off = (off + 255) / 256 * 256;
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += count * sizeof(T);
    return p;
  }
};

struct Dims {
  int P, E, El, k, d, f, Tmax;
  int64_t C, Cpad, Rpad, recv, adjw;
};

Dims dims_of(const luffy_config* c) {
  Dims m;
  m.P = c->world;
  m.E = c->num_experts;
  m.El = c->num_experts / c->world;
  m.k = c->top_k;
  m.d = c->d_model;
  m.f = c->d_ffn;
  m.Tmax = c->max_tokens;
  m.C = (int64_t)m.Tmax * m.k;
  m.Cpad = m.C + (int64_t)m.E * kRowAlign;
  m.Rpad = m.Cpad;
  m.recv = c->max_recv_rows > 0 ? c->max_recv_rows : (int64_t)m.P * m.C + (int64_t)m.El * kRowAlign;
  m.adjw = m.Cpad * m.Cpad / 32;  // sum over groups of npad^2/32 <= (sum npad)^2/32
  return m;
}

void carve(const luffy_config* c, Carver& cv, luffy_layer* L) {
  const Dims m = dims_of(c);
  const size_t es = elem_size(c->dtype);
  luffy_layer tmp;
  luffy_layer* o = L ? L : &tmp;
  o->probs = cv.take<float>((size_t)m.Tmax * m.E);
  o->idx = cv.take<int32_t>(m.C);
  o->w = cv.take<float>(m.C);
  o->gcnt = cv.take<int32_t>(m.E);
  o->goff = cv.take<int32_t>(m.E + 1);
  o->gtok = cv.take<int32_t>(m.Cpad);
  o->gloc = cv.take<int32_t>(m.C);
  o->gw = cv.take<float>(m.Cpad);
  o->xg = cv.take<char>(m.Cpad * m.d * es);
  o->gnorm = cv.take<double>(m.Cpad);
  o->adjoff = cv.take<int64_t>(m.E + 1);
  o->adj = cv.take<uint32_t>(m.adjw);
  o->rep_local = cv.take<int32_t>(m.Cpad);
  o->key = cv.take<uint64_t>(m.Cpad);
  o->m1 = cv.take<uint64_t>(m.Cpad);
  o->alive = cv.take<uint32_t>(m.Cpad / 32 + 1);
  o->win = cv.take<uint32_t>(m.Cpad / 32 + 1);
  o->ctrl = cv.take<uint32_t>(64 + kGreedyMaxRounds);
  o->nrep = cv.take<int32_t>(m.E);
  o->soff = cv.take<int32_t>(m.E + 1);
  o->lslot = cv.take<int32_t>(m.Cpad);
  o->perm = cv.take<int32_t>(m.Rpad);
  o->slot_gl = cv.take<int32_t>(m.Rpad);
  o->pos = cv.take<int32_t>(m.C);
  o->rep = cv.take<int32_t>(m.C);
  o->mstart = cv.take<int32_t>(m.Rpad);
  o->mcnt = cv.take<int32_t>(m.Rpad);
  o->mcur = cv.take<int32_t>(m.Rpad);
  o->members = cv.take<int32_t>(m.Cpad);
  o->mslot = cv.take<int32_t>(m.Cpad);
  o->mpart = cv.take<float>((size_t)(m.Cpad / 16) * 2 * m.d);
  o->roff = cv.take<int32_t>(m.El + 1);
  o->cnt_all = cv.take<int32_t>((size_t)m.P * m.E);
  o->send = m.P > 1 ? cv.take<char>(m.Rpad * m.d * es) : nullptr;
  o->dl = cv.take<float>((size_t)m.Tmax * m.E);
  o->wg_part = cv.take<float>((size_t)std::max(wg_parts(m.E, m.d), (m.Tmax + 63) / 64) * m.E * m.d);
}

luffy_status validate(const luffy_config* c) {
  if (!c) return fail(LUFFY_E_INVALID, "config is NULL");
  if (c->world < 1 || c->rank < 0 || c->rank >= c->world) return fail(LUFFY_E_INVALID, "need 0 <= rank < world");
  if (c->num_experts < 1 || c->num_experts > LUFFY_MAX_EXPERTS) return fail(LUFFY_E_INVALID, "num_experts out of range");
  if (c->num_experts % c->world) return fail(LUFFY_E_INVALID, "num_experts % world != 0");
  if (c->top_k < 1 || c->top_k > c->num_experts || c->top_k > 8) return fail(LUFFY_E_INVALID, "need 1 <= top_k <= min(E, 8)");
  if (c->d_model < 64 || c->d_model % 64) return fail(LUFFY_E_INVALID, "d_model must be a positive multiple of 64");
  if (c->d_ffn < 64 || c->d_ffn % 64) return fail(LUFFY_E_INVALID, "d_ffn must be a positive multiple of 64");
  if (c->dtype != LUFFY_BF16 && c->dtype != LUFFY_FP32) return fail(LUFFY_E_INVALID, "dtype must be LUFFY_BF16 or LUFFY_FP32");
  if (c->act != LUFFY_GELU && c->act != LUFFY_SWIGLU) return fail(LUFFY_E_INVALID, "act must be LUFFY_GELU or LUFFY_SWIGLU");
  if (c->renormalize < -1 || c->renormalize > 1) return fail(LUFFY_E_INVALID, "renormalize must be -1, 0 or 1");
  if (c->max_tokens < 1) return fail(LUFFY_E_INVALID, "max_tokens must be >= 1");
  if (c->dtype == LUFFY_BF16 && (c->d_model % 256 || c->d_ffn % 256))
    return fail(LUFFY_E_UNSUPPORTED, "bf16 (tcgen05) path needs d_model and d_ffn multiples of 256");
  const Dims m = dims_of(c);
  if (m.Cpad >= (int64_t)1 << 30) return fail(LUFFY_E_INVALID, "max_tokens * top_k too large");
  if (c->world == 1 && c->max_recv_rows > 0 && c->max_recv_rows < m.Rpad)
    return fail(LUFFY_E_INVALID, "world == 1 needs max_recv_rows >= max_tokens*top_k + E*LUFFY_ROW_ALIGN (or 0)");
  return LUFFY_OK;
}

// bf16: tcgen05 tensor cores; fp32: exact SIMT FFMA (tf32 would break the fp32 tolerance).
int gemm_rows(int dtype, int epi, const void* A, const void* B, const void* B3, void* D, void* aux0, const int32_t* off,
              int G, int64_t max_rows, int N, int K, int b_kmajor, void* s) {
  if (dtype == LUFFY_BF16) return gemm_rows_tc(epi, A, B, B3, D, aux0, off, G, max_rows, N, K, b_kmajor, s);
  return gemm_rows_simt(dtype, epi, A, B, B3, D, aux0, off, G, max_rows, N, K, b_kmajor, s);
}
int gemm_wgrad(int dtype, const void* A, const void* B, float* D, float* D3, int Msplit, const int32_t* off, int G, int M,
               int N, int lda, int ldb, int64_t max_rows, void* s) {
  if (dtype == LUFFY_BF16) return gemm_wgrad_tc(A, B, D, D3, Msplit, off, G, M, N, lda, ldb, max_rows, s);
  return gemm_wgrad_simt(dtype, A, B, D, D3, Msplit, off, G, M, N, lda, ldb, s);
}

luffy_status need(const void* p, const char* name) {
  if (!p) return fail(LUFFY_E_INVALID, std::string(name) + " is NULL");
  return LUFFY_OK;
}
#define LUFFY_NEED(p)                                   \
  do {                                                  \
    luffy_status _s = need((p), #p);                    \
    if (_s != LUFFY_OK) return _s;                      \
  } while (0)
#define LUFFY_ALIGNED(p)                                                                   \
  do {                                                                                     \
    if (reinterpret_cast<uintptr_t>(p) % 16)                                               \
      return fail(LUFFY_E_INVALID, std::string(#p) + " must be 16-byte aligned");          \
  } while (0)
#define LUFFY_STAGE(L, s, name)                                                                         \
  do {                                                                                                  \
    if ((L)->stage < (s)) return fail(LUFFY_E_STATE, std::string(name) + ": called out of order");      \
  } while (0)

// Expert-side row offsets for the GEMMs: with one rank the send layout is the expert layout.
const int32_t* expert_off(const luffy_layer* L) { return L->P == 1 ? L->soff : L->roff; }
int64_t expert_rows_bound(const luffy_layer* L) { return L->P == 1 ? L->Rpad_max : L->recv_rows_h; }

// One grouped exchange.  dir 0: source->expert (dispatch / combine_bwd): src rows at send offsets
// `soff_h` (this rank's counts), dst rows in the expert layout.  dir 1: the reverse.
luffy_status exchange(luffy_layer* L, int dir, const void* src, void* dst, cudaStream_t st) {
  const nccl::Api* a = nccl::api();
  if (!a) return fail(LUFFY_E_NCCL, "NCCL could not be loaded (libnccl.so.2)");
  const size_t rb = (size_t)L->d * elem_size(L->dtype);
  const int P = L->P, E = L->E, El = L->El, me = L->rank;
  const int32_t* cnt = L->cnt_all_h;
  auto expert_row = [&](int e, int srcrank) {  // row of (srcrank's block of expert e) at its owner
    const int el = e % El;
    int64_t r = L->roff_h[el];
    for (int q = 0; q < srcrank; ++q) r += cnt[(size_t)q * E + e];
    return r;
  };
  const char* s = static_cast<const char*>(src);
  char* d = static_cast<char*>(dst);
  LUFFY_NCCL(a->GroupStart(), "ncclGroupStart");
  for (int p = 0; p < P; ++p) {
    for (int el = 0; el < El; ++el) {
      if (dir == 0) {
        // I send my rows for expert e = p*El + el to p; I receive p's rows for my expert me*El + el.
        const int e_out = p * El + el, e_in = me * El + el;
        const size_t n_out = cnt[(size_t)me * E + e_out], n_in = cnt[(size_t)p * E + e_in];
        const char* sp = s + (size_t)L->soff_h[e_out] * rb;
        char* dp = d + (size_t)expert_row(e_in, p) * rb;
        if (p == me) {
          if (n_out) {
            cudaError_t ce = cudaMemcpyAsync(d + (size_t)expert_row(e_out, me) * rb, sp, n_out * rb, cudaMemcpyDeviceToDevice, st);
            if (ce != cudaSuccess) { a->GroupEnd(); return cuda_fail(ce, "exchange self copy"); }
          }
          continue;
        }
        if (n_out) LUFFY_NCCL(a->Send(sp, n_out * rb, nccl::kUint8, p, L->ctx->comm, st), "ncclSend");
        if (n_in) LUFFY_NCCL(a->Recv(dp, n_in * rb, nccl::kUint8, p, L->ctx->comm, st), "ncclRecv");
      } else {
        // I send p's rows of my expert me*El + el back to p; I receive my rows of expert p*El + el.
        const int e_out = me * El + el, e_in = p * El + el;
        const size_t n_out = cnt[(size_t)p * E + e_out], n_in = cnt[(size_t)me * E + e_in];
        const char* sp = s + (size_t)expert_row(e_out, p) * rb;
        char* dp = d + (size_t)L->soff_h[e_in] * rb;
        if (p == me) {
          if (n_in) {
            cudaError_t ce = cudaMemcpyAsync(dp, s + (size_t)expert_row(e_in, me) * rb, n_in * rb, cudaMemcpyDeviceToDevice, st);
            if (ce != cudaSuccess) { a->GroupEnd(); return cuda_fail(ce, "exchange self copy"); }
          }
          continue;
        }
        if (n_out) LUFFY_NCCL(a->Send(sp, n_out * rb, nccl::kUint8, p, L->ctx->comm, st), "ncclSend");
        if (n_in) LUFFY_NCCL(a->Recv(dp, n_in * rb, nccl::kUint8, p, L->ctx->comm, st), "ncclRecv");
      }
    }
  }
  LUFFY_NCCL(a->GroupEnd(), "ncclGroupEnd");
  return LUFFY_OK;
}

// Zero the padding rows of an expert-layout buffer (host-known layout, world > 1).
luffy_status zero_expert_padding(luffy_layer* L, void* buf, cudaStream_t st) {
  const size_t rb = (size_t)L->d * elem_size(L->dtype);
  for (int el = 0; el < L->El; ++el) {
    const int e = L->rank * L->El + el;
    int64_t used = 0;
    for (int q = 0; q < L->P; ++q) used += L->cnt_all_h[(size_t)q * L->E + e];
    const int64_t r0 = L->roff_h[el] + used, r1 = L->roff_h[el + 1];
    if (r1 > r0) LUFFY_CHECK(cudaMemsetAsync(static_cast<char*>(buf) + r0 * rb, 0, (r1 - r0) * rb, st), "memset padding");
  }
  return LUFFY_OK;
}

}  // namespace
}  // namespace luffy

using namespace luffy;

extern "C" {

const char* luffy_last_error(void) { return g_err.c_str(); }

luffy_status luffy_exchange_plan(int32_t world, int32_t rank, int32_t num_experts, const int32_t* counts_all,
                                 int32_t* send_off, int32_t* recv_off, int64_t* send_rows_to, int64_t* recv_rows_from) {
  if (world < 1 || rank < 0 || rank >= world || num_experts < 1 || num_experts % world)
    return fail(LUFFY_E_INVALID, "exchange_plan: bad world/rank/num_experts");
  LUFFY_NEED(counts_all);
  LUFFY_NEED(send_off);
  LUFFY_NEED(recv_off);
  const int P = world, E = num_experts, El = E / world;
  send_off[0] = 0;
  for (int e = 0; e < E; ++e) {
    const int32_t c = counts_all[(size_t)rank * E + e];
    if (c < 0) return fail(LUFFY_E_INVALID, "exchange_plan: negative count");
    send_off[e + 1] = send_off[e] + (int32_t)round_up(c, kRowAlign);
  }
  recv_off[0] = 0;
  for (int el = 0; el < El; ++el) {
    const int e = rank * El + el;
    int64_t rows = 0;
    for (int q = 0; q < P; ++q) rows += counts_all[(size_t)q * E + e];
    recv_off[el + 1] = recv_off[el] + (int32_t)round_up(rows, kRowAlign);
  }
  for (int p = 0; p < P; ++p) {
    int64_t so = 0, ri = 0;
    for (int el = 0; el < El; ++el) {
      so += counts_all[(size_t)rank * E + p * El + el];
      ri += counts_all[(size_t)p * E + rank * El + el];
    }
    if (send_rows_to) send_rows_to[p] = so;
    if (recv_rows_from) recv_rows_from[p] = ri;
  }
  return LUFFY_OK;
}
int64_t luffy_launch_count(void) { return g_launches.load(); }

luffy_status luffy_get_unique_id(uint8_t id[128]) {
  if (!id) return fail(LUFFY_E_INVALID, "id is NULL");
  const nccl::Api* a = nccl::api();
  if (!a) return fail(LUFFY_E_NCCL, "NCCL could not be loaded (libnccl.so.2)");
  nccl::UniqueId u;
  LUFFY_NCCL(a->GetUniqueId(&u), "ncclGetUniqueId");
  std::memcpy(id, u.internal, 128);
  return LUFFY_OK;
}

luffy_status luffy_create(const luffy_config* cfg, const uint8_t* nccl_id, luffy_ctx** out) {
  luffy_status st = validate(cfg);
  if (st != LUFFY_OK) return st;
  LUFFY_NEED(out);
  int dev = 0;
  LUFFY_CHECK(cudaGetDevice(&dev), "cudaGetDevice");
  cudaDeviceProp prop;
  LUFFY_CHECK(cudaGetDeviceProperties(&prop, dev), "cudaGetDeviceProperties");
  if (prop.major != 10 || prop.minor != 0)
    return fail(LUFFY_E_UNSUPPORTED, "libluffy is built for sm_100a (B200); found sm_" + std::to_string(prop.major) +
                                         std::to_string(prop.minor));
  luffy_ctx* c = new luffy_ctx();
  c->cfg = *cfg;
  if (c->cfg.renormalize < 0) c->cfg.renormalize = cfg->top_k > 1 ? 1 : 0;
  c->device = dev;
  c->comm = nullptr;
  if (cfg->world > 1) {
    if (!nccl_id) {
      delete c;
      return fail(LUFFY_E_INVALID, "world > 1 needs an NCCL unique id");
    }
    const nccl::Api* a = nccl::api();
    if (!a) {
      delete c;
      return fail(LUFFY_E_NCCL, "NCCL could not be loaded (libnccl.so.2)");
    }
    nccl::UniqueId u;
    std::memcpy(u.internal, nccl_id, 128);
    nccl::Result r = a->CommInitRank(&c->comm, cfg->world, u, cfg->rank);
    if (r != 0) {
      delete c;
      return nccl_fail(r, "ncclCommInitRank");
    }
  }
  *out = c;
  return LUFFY_OK;
}

void luffy_destroy(luffy_ctx* ctx) {
  if (!ctx) return;
  if (ctx->comm) {
    const nccl::Api* a = nccl::api();
    if (a) a->CommDestroy(ctx->comm);
  }
  delete ctx;
}

size_t luffy_layer_workspace_bytes(const luffy_config* cfg) {
  if (validate(cfg) != LUFFY_OK) return 0;
  Carver cv{nullptr};
  carve(cfg, cv, nullptr);
  return (cv.off + 255) / 256 * 256;
}

luffy_status luffy_layer_create(luffy_ctx* ctx, void* ws, size_t bytes, luffy_layer** out) {
  LUFFY_NEED(ctx);
  LUFFY_NEED(ws);
  LUFFY_NEED(out);
  if (reinterpret_cast<uintptr_t>(ws) % 256) return fail(LUFFY_E_INVALID, "workspace must be 256-byte aligned");
  const size_t need_b = luffy_layer_workspace_bytes(&ctx->cfg);
  if (bytes < need_b) return fail(LUFFY_E_INVALID, "workspace too small: need " + std::to_string(need_b) + " bytes");
  luffy_layer* L = new luffy_layer();
  std::memset(L, 0, sizeof(*L));
  Carver cv{static_cast<char*>(ws)};
  carve(&ctx->cfg, cv, L);
  const Dims m = dims_of(&ctx->cfg);
  L->ctx = ctx;
  L->P = m.P;
  L->rank = ctx->cfg.rank;
  L->E = m.E;
  L->El = m.El;
  L->k = m.k;
  L->d = m.d;
  L->f = m.f;
  L->dtype = ctx->cfg.dtype;
  L->act = ctx->cfg.act;
  L->renorm = ctx->cfg.renormalize;
  L->Tmax = m.Tmax;
  L->C_max = m.C;
  L->Cpad_max = m.Cpad;
  L->Rpad_max = m.Rpad;
  L->recv_max = m.recv;
  L->adj_words_max = m.adjw;
  cudaError_t e1 = cudaMallocHost(&L->cnt_all_h, sizeof(int32_t) * m.P * m.E);
  cudaError_t e2 = cudaMallocHost(&L->roff_h, sizeof(int32_t) * (m.El + 1));
  cudaError_t e3 = cudaMallocHost(&L->soff_h, sizeof(int32_t) * (m.E + 1));
  if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess) {
    luffy_layer_destroy(L);
    return fail(LUFFY_E_CUDA, "cudaMallocHost failed");
  }
  *out = L;
  return LUFFY_OK;
}

void luffy_layer_destroy(luffy_layer* L) {
  if (!L) return;
  if (L->cnt_all_h) cudaFreeHost(L->cnt_all_h);
  if (L->roff_h) cudaFreeHost(L->roff_h);
  if (L->soff_h) cudaFreeHost(L->soff_h);
  delete L;
}

luffy_status luffy_layer_rows(const luffy_layer* L, int64_t* send_rows, int64_t* recv_rows) {
  LUFFY_NEED(L);
  LUFFY_STAGE(L, 3, "luffy_layer_rows");
  if (send_rows) *send_rows = L->send_rows_h;
  if (recv_rows) *recv_rows = L->recv_rows_h;
  return LUFFY_OK;
}

// ------------------------------------------------------------------------------------------ forward

luffy_status luffy_route(luffy_layer* L, const void* x, const float* w_gate, int32_t T, int32_t* topk_idx,
                         float* topk_w, void* stream) {
  LUFFY_NEED(L);
  LUFFY_NEED(x);
  LUFFY_NEED(w_gate);
  LUFFY_NEED(topk_idx);
  LUFFY_NEED(topk_w);
  LUFFY_ALIGNED(x);
  LUFFY_ALIGNED(w_gate);
  if (T < 1 || T > L->Tmax) return fail(LUFFY_E_INVALID, "need 0 < T <= max_tokens");
  L->T = T;
  L->stage = 0;
  LUFFY_CHECK(launch_route(L, x, w_gate, topk_idx, topk_w, stream), "luffy_route");
  L->stage = 1;
  return LUFFY_OK;
}

luffy_status luffy_condense(luffy_layer* L, const void* x, float h, int32_t* rep, luffy_condense_stats* stats,
                            void* stream) {
  LUFFY_NEED(L);
  LUFFY_NEED(x);
  LUFFY_NEED(rep);
  LUFFY_ALIGNED(x);
  LUFFY_STAGE(L, 1, "luffy_condense");
  if (!(h == h)) return fail(LUFFY_E_INVALID, "h is NaN");
  L->h = h;
  LUFFY_CHECK(launch_group_build(L, x, stream), "luffy_condense/group_build");
  if (h > 1.0f) {
    L->has_adj = false;
    LUFFY_CHECK(launch_identity_rep(L, stream), "luffy_condense/identity");
  } else {
    L->has_adj = true;
    // bf16: tcgen05 Gram; fp32: exact SIMT FFMA Gram
    if (L->dtype == LUFFY_BF16) LUFFY_CHECK(launch_gram_tc(L, h, stream), "luffy_condense/gram");
    else LUFFY_CHECK(launch_gram_simt(L, h, stream), "luffy_condense/gram");
    LUFFY_CHECK(launch_greedy(L, stream), "luffy_condense/greedy");
  }
  LUFFY_CHECK(launch_pack(L, x, nullptr, rep, stream), "luffy_condense/layout");
  L->stage = 2;
  if (stats) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::vector<int32_t> gc(L->E), nr(L->E);
    uint32_t rounds = 0;
    LUFFY_CHECK(cudaMemcpyAsync(gc.data(), L->gcnt, sizeof(int32_t) * L->E, cudaMemcpyDeviceToHost, st), "stats");
    LUFFY_CHECK(cudaMemcpyAsync(nr.data(), L->nrep, sizeof(int32_t) * L->E, cudaMemcpyDeviceToHost, st), "stats");
    LUFFY_CHECK(cudaMemcpyAsync(&rounds, L->ctrl + 2, sizeof(uint32_t), cudaMemcpyDeviceToHost, st), "stats");
    LUFFY_CHECK(cudaStreamSynchronize(st), "stats sync");
    std::memset(stats, 0, sizeof(*stats));
    for (int e = 0; e < L->E; ++e) {
      stats->copies += gc[e];
      stats->reps += nr[e];
      stats->copies_per_expert[e] = gc[e];
      stats->reps_per_expert[e] = nr[e];
    }
    stats->rounds = (int32_t)rounds;
  }
  return LUFFY_OK;
}

luffy_status luffy_dispatch(luffy_layer* L, const void* x, void* recv, int64_t* recv_rows, void* stream) {
  LUFFY_NEED(L);
  LUFFY_NEED(x);
  LUFFY_NEED(recv);
  LUFFY_ALIGNED(x);
  LUFFY_ALIGNED(recv);
  LUFFY_STAGE(L, 2, "luffy_dispatch");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (L->P == 1) {
    LUFFY_CHECK(launch_pack_rows(L, x, recv, stream), "luffy_dispatch/pack");
    if (recv_rows) {
      int32_t r = 0;
      LUFFY_CHECK(cudaMemcpyAsync(&r, L->soff + L->E, sizeof(int32_t), cudaMemcpyDeviceToHost, st), "rows");
      LUFFY_CHECK(cudaStreamSynchronize(st), "rows sync");
      L->send_rows_h = L->recv_rows_h = r;
      *recv_rows = r;
    } else {
      L->send_rows_h = L->recv_rows_h = L->Rpad_max;  // upper bound (no host sync at world == 1)
    }
    L->stage = 3;
    return LUFFY_OK;
  }
  const nccl::Api* a = nccl::api();
  if (!a) return fail(LUFFY_E_NCCL, "NCCL could not be loaded (libnccl.so.2)");
  LUFFY_CHECK(launch_pack_rows(L, x, L->send, stream), "luffy_dispatch/pack");
  // counts of representatives per expert from every rank (1 KiB), then the host posts the receives
  LUFFY_NCCL(a->AllGather(L->nrep, L->cnt_all, L->E, nccl::kInt32, L->ctx->comm, st), "ncclAllGather(counts)");
  LUFFY_CHECK(cudaMemcpyAsync(L->cnt_all_h, L->cnt_all, sizeof(int32_t) * L->P * L->E, cudaMemcpyDeviceToHost, st), "counts D2H");
  LUFFY_CHECK(cudaStreamSynchronize(st), "counts sync");
  luffy_status sp = luffy_exchange_plan(L->P, L->rank, L->E, L->cnt_all_h, L->soff_h, L->roff_h, nullptr, nullptr);
  if (sp != LUFFY_OK) return sp;
  if (L->roff_h[L->El] > L->recv_max)
    return fail(LUFFY_E_CAPACITY, "dispatch: " + std::to_string(L->roff_h[L->El]) + " expert rows exceed max_recv_rows " +
                                      std::to_string(L->recv_max));
  L->send_rows_h = L->soff_h[L->E];
  L->recv_rows_h = L->roff_h[L->El];
  LUFFY_CHECK(cudaMemcpyAsync(L->roff, L->roff_h, sizeof(int32_t) * (L->El + 1), cudaMemcpyHostToDevice, st), "roff H2D");
  luffy_status s2 = zero_expert_padding(L, recv, st);
  if (s2 != LUFFY_OK) return s2;
  s2 = exchange(L, 0, L->send, recv, st);
  if (s2 != LUFFY_OK) return s2;
  if (recv_rows) *recv_rows = L->recv_rows_h;
  L->stage = 3;
  return LUFFY_OK;
}

luffy_status luffy_expert_ffn(luffy_layer* L, const void* recv, const void* w1, const void* w2, const void* w3, void* out,
                              void* saved_pre, void* saved_act, void* stream) {
  LUFFY_NEED(L);
  LUFFY_NEED(recv);
  LUFFY_NEED(w1);
  LUFFY_NEED(w2);
  LUFFY_NEED(out);
  LUFFY_NEED(saved_pre);
  LUFFY_NEED(saved_act);
  LUFFY_STAGE(L, 3, "luffy_expert_ffn");
  if (L->act == LUFFY_SWIGLU && !w3) return fail(LUFFY_E_INVALID, "SWIGLU needs w3");
  const int32_t* off = expert_off(L);
  const int64_t rows = expert_rows_bound(L);
  if (L->act == LUFFY_GELU) {
    LUFFY_CHECK(gemm_rows(L->dtype, EPI_GELU, recv, w1, nullptr, saved_act, saved_pre, off, L->El, rows, L->f, L->d, 1, stream),
                "expert_ffn/gemm1");
  } else {
    LUFFY_CHECK(gemm_rows(L->dtype, EPI_SWIGLU, recv, w1, w3, saved_act, saved_pre, off, L->El, rows, 2 * L->f, L->d, 1, stream),
                "expert_ffn/gemm1");
  }
  LUFFY_CHECK(gemm_rows(L->dtype, EPI_STORE, saved_act, w2, nullptr, out, nullptr, off, L->El, rows, L->d, L->f, 1, stream),
              "expert_ffn/gemm2");
  if (L->stage < 4) L->stage = 4;
  return LUFFY_OK;
}

luffy_status luffy_combine(luffy_layer* L, const void* expert_out, void* gathered, void* stream) {
  LUFFY_NEED(L);
  LUFFY_NEED(expert_out);
  LUFFY_NEED(gathered);
  LUFFY_STAGE(L, 4, "luffy_combine");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (L->P == 1) {
    if (gathered != expert_out)
      LUFFY_CHECK(cudaMemcpyAsync(gathered, expert_out, (size_t)L->send_rows_h * L->d * elem_size(L->dtype),
                                  cudaMemcpyDeviceToDevice, st), "combine copy");
  } else {
    luffy_status s2 = exchange(L, 1, expert_out, gathered, st);
    if (s2 != LUFFY_OK) return s2;
  }
  L->stage = 5;
  return LUFFY_OK;
}

luffy_status luffy_uncondense(luffy_layer* L, const void* gathered, void* y, void* stream) {
  LUFFY_NEED(L);
  LUFFY_NEED(gathered);
  LUFFY_NEED(y);
  LUFFY_ALIGNED(y);
  LUFFY_STAGE(L, 5, "luffy_uncondense");
  LUFFY_CHECK(launch_uncondense(L, gathered, y, stream), "luffy_uncondense");
  L->stage = 6;
  return LUFFY_OK;
}

// ------------------------------------------------------------------------------------------ backward

luffy_status luffy_uncondense_bwd(luffy_layer* L, const void* dy, const void* gathered, void* d_gathered, float* d_topk_w,
                                  void* stream) {
  LUFFY_NEED(L);
  LUFFY_NEED(dy);
  LUFFY_NEED(gathered);
  LUFFY_NEED(d_gathered);
  LUFFY_NEED(d_topk_w);
  LUFFY_ALIGNED(dy);
  LUFFY_STAGE(L, 6, "luffy_uncondense_bwd");
  LUFFY_CHECK(launch_uncondense_bwd(L, dy, gathered, d_gathered, d_topk_w, stream), "luffy_uncondense_bwd");
  return LUFFY_OK;
}

luffy_status luffy_combine_bwd(luffy_layer* L, const void* d_gathered, void* d_expert_out, void* stream) {
  LUFFY_NEED(L);
  LUFFY_NEED(d_gathered);
  LUFFY_NEED(d_expert_out);
  LUFFY_STAGE(L, 6, "luffy_combine_bwd");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (L->P == 1) {
    if (d_gathered != d_expert_out)
      LUFFY_CHECK(cudaMemcpyAsync(d_expert_out, d_gathered, (size_t)L->send_rows_h * L->d * elem_size(L->dtype),
                                  cudaMemcpyDeviceToDevice, st), "combine_bwd copy");
    return LUFFY_OK;
  }
  luffy_status s2 = zero_expert_padding(L, d_expert_out, st);
  if (s2 != LUFFY_OK) return s2;
  return exchange(L, 0, d_gathered, d_expert_out, st);
}

luffy_status luffy_expert_ffn_bwd(luffy_layer* L, const void* d_out, const void* recv, const void* w1, const void* w2,
                                  const void* w3, const void* saved_pre, const void* saved_act, void* scratch_dpre,
                                  void* d_recv, float* dw1, float* dw2, float* dw3, void* stream) {
  LUFFY_NEED(L);
  LUFFY_NEED(d_out);
  LUFFY_NEED(recv);
  LUFFY_NEED(w1);
  LUFFY_NEED(w2);
  LUFFY_NEED(saved_pre);
  LUFFY_NEED(saved_act);
  LUFFY_NEED(scratch_dpre);
  LUFFY_NEED(d_recv);
  LUFFY_NEED(dw1);
  LUFFY_NEED(dw2);
  LUFFY_STAGE(L, 6, "luffy_expert_ffn_bwd");
  if (L->act == LUFFY_SWIGLU && (!w3 || !dw3)) return fail(LUFFY_E_INVALID, "SWIGLU needs w3 and dw3");
  const int32_t* off = expert_off(L);
  const int64_t rows = expert_rows_bound(L);
  const int d = L->d, f = L->f, G = L->El;
  if (L->act == LUFFY_GELU) {
    LUFFY_CHECK(gemm_rows(L->dtype, EPI_DGELU, d_out, w2, nullptr, scratch_dpre, const_cast<void*>(saved_pre), off, G, rows,
                          f, d, 0, stream), "ffn_bwd/dgrad2");
    LUFFY_CHECK(gemm_rows(L->dtype, EPI_STORE, scratch_dpre, w1, nullptr, d_recv, nullptr, off, G, rows, d, f, 0, stream),
                "ffn_bwd/dgrad1");
    LUFFY_CHECK(gemm_wgrad(L->dtype, d_out, saved_act, dw2, nullptr, d, off, G, d, f, d, f, rows, stream), "ffn_bwd/wgrad2");
    LUFFY_CHECK(gemm_wgrad(L->dtype, scratch_dpre, recv, dw1, nullptr, f, off, G, f, d, f, d, rows, stream), "ffn_bwd/wgrad1");
  } else {
    LUFFY_CHECK(gemm_rows(L->dtype, EPI_DSWIGLU, d_out, w2, nullptr, scratch_dpre, const_cast<void*>(saved_pre), off, G,
                          rows, f, d, 0, stream), "ffn_bwd/dgrad2");
    LUFFY_CHECK(gemm_rows(L->dtype, EPI_STORE, scratch_dpre, w1, w3, d_recv, nullptr, off, G, rows, d, 2 * f, 0, stream),
                "ffn_bwd/dgrad1");
    LUFFY_CHECK(gemm_wgrad(L->dtype, d_out, saved_act, dw2, nullptr, d, off, G, d, f, d, f, rows, stream), "ffn_bwd/wgrad2");
    LUFFY_CHECK(gemm_wgrad(L->dtype, scratch_dpre, recv, dw1, dw3, f, off, G, 2 * f, d, 2 * f, d, rows, stream), "ffn_bwd/wgrad1");
  }
  return LUFFY_OK;
}

luffy_status luffy_dispatch_bwd(luffy_layer* L, const void* d_recv, void* dx, void* stream) {
  LUFFY_NEED(L);
  LUFFY_NEED(d_recv);
  LUFFY_NEED(dx);
  LUFFY_ALIGNED(dx);
  LUFFY_STAGE(L, 6, "luffy_dispatch_bwd");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const void* dsend = d_recv;
  if (L->P > 1) {
    luffy_status s2 = exchange(L, 1, d_recv, L->send, st);
    if (s2 != LUFFY_OK) return s2;
    dsend = L->send;
  }
  LUFFY_CHECK(launch_unpack_bwd(L, dsend, dx, stream), "luffy_dispatch_bwd");
  return LUFFY_OK;
}

luffy_status luffy_route_bwd(luffy_layer* L, const void* x, const float* w_gate, const float* d_topk_w, void* dx,
                             float* dw_gate, void* stream) {
  LUFFY_NEED(L);
  LUFFY_NEED(x);
  LUFFY_NEED(w_gate);
  LUFFY_NEED(d_topk_w);
  LUFFY_NEED(dx);
  LUFFY_NEED(dw_gate);
  LUFFY_STAGE(L, 6, "luffy_route_bwd");
  LUFFY_CHECK(launch_route_bwd(L, x, w_gate, d_topk_w, dx, dw_gate, stream), "luffy_route_bwd");
  return LUFFY_OK;
}

luffy_status luffy_debug_gemm(int32_t kind, int32_t dtype, int32_t epi, const void* A, const void* B, const void* B3,
                              void* D, void* aux, float* D3, int32_t Msplit, const int32_t* off, int32_t G,
                              int64_t max_rows, int32_t M, int32_t N, int32_t K, int32_t b_kmajor, void* stream) {
  LUFFY_NEED(A);
  LUFFY_NEED(B);
  LUFFY_NEED(D);
  LUFFY_NEED(off);
  if (kind == 0) {
    LUFFY_CHECK(gemm_rows(dtype, epi, A, B, B3, D, aux, off, G, max_rows, N, K, b_kmajor, stream), "luffy_debug_gemm");
  } else {
    LUFFY_CHECK(gemm_wgrad(dtype, A, B, static_cast<float*>(D), D3, Msplit, off, G, M, N, K, N, max_rows, stream),
                "luffy_debug_gemm");
  }
  return LUFFY_OK;
}

luffy_status luffy_debug_copy(luffy_layer* L, int32_t item, void* dst, size_t* bytes, void* stream) {
  LUFFY_NEED(L);
  LUFFY_NEED(bytes);
  LUFFY_STAGE(L, 2, "luffy_debug_copy");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int32_t goffE = 0, soffE = 0;
  int64_t adjE = 0;
  LUFFY_CHECK(cudaMemcpyAsync(&goffE, L->goff + L->E, sizeof(int32_t), cudaMemcpyDeviceToHost, st), "debug");
  LUFFY_CHECK(cudaMemcpyAsync(&soffE, L->soff + L->E, sizeof(int32_t), cudaMemcpyDeviceToHost, st), "debug");
  if (L->has_adj)
    LUFFY_CHECK(cudaMemcpyAsync(&adjE, L->adjoff + L->E, sizeof(int64_t), cudaMemcpyDeviceToHost, st), "debug");
  LUFFY_CHECK(cudaStreamSynchronize(st), "debug sync");
  const void* src = nullptr;
  size_t n = 0;
  switch (item) {
    case LUFFY_DBG_GCNT: src = L->gcnt; n = sizeof(int32_t) * L->E; break;
    case LUFFY_DBG_GOFF: src = L->goff; n = sizeof(int32_t) * (L->E + 1); break;
    case LUFFY_DBG_GTOK: src = L->gtok; n = sizeof(int32_t) * goffE; break;
    case LUFFY_DBG_ADJOFF: src = L->adjoff; n = L->has_adj ? sizeof(int64_t) * (L->E + 1) : 0; break;
    case LUFFY_DBG_ADJ: src = L->adj; n = sizeof(uint32_t) * adjE; break;
    case LUFFY_DBG_REP_LOCAL: src = L->rep_local; n = sizeof(int32_t) * goffE; break;
    case LUFFY_DBG_SOFF: src = L->soff; n = sizeof(int32_t) * (L->E + 1); break;
    case LUFFY_DBG_PERM: src = L->perm; n = sizeof(int32_t) * soffE; break;
    case LUFFY_DBG_POS: src = L->pos; n = sizeof(int32_t) * L->T * L->k; break;
    case LUFFY_DBG_NREP: src = L->nrep; n = sizeof(int32_t) * L->E; break;
    case LUFFY_DBG_ROUNDS: src = L->ctrl + 2; n = sizeof(uint32_t); break;
    case LUFFY_DBG_GREEDY_TIMES: src = L->ctrl; n = sizeof(uint32_t) * 64; break;
    default: return fail(LUFFY_E_INVALID, "luffy_debug_copy: unknown item");
  }
  if (dst == nullptr || *bytes < n) {
    *bytes = n;
    return dst == nullptr ? LUFFY_OK : fail(LUFFY_E_INVALID, "luffy_debug_copy: destination too small");
  }
  *bytes = n;
  if (n) {
    LUFFY_CHECK(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, st), "debug copy");
    LUFFY_CHECK(cudaStreamSynchronize(st), "debug sync");
  }
  return LUFFY_OK;
}

}  // extern "C"
