// C ABI of libluffy (include/luffy.h): context, workspace layout, argument validation, call order and
// the device-initiated expert-parallel exchange over NVLink (CUDA IPC) between the kernels.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "exchange.cuh"

struct luffy_ctx {
  luffy_config cfg;
  int device;
};

namespace luffy {

static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};

luffy_status fail(luffy_status st, const std::string& msg) {
  g_err = msg;
  return st;
}
void note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

namespace {
std::mutex g_cache_mu;
std::map<std::tuple<const void*, int, int64_t>, int> g_cache;
int cur_dev() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}
}  // namespace
bool dev_cache_get(const void* key, int64_t extra, int* value) {
  std::lock_guard<std::mutex> g(g_cache_mu);
  auto it = g_cache.find(std::make_tuple(key, cur_dev(), extra));
  if (it == g_cache.end()) return false;
  *value = it->second;
  return true;
}
void dev_cache_put(const void* key, int64_t extra, int value) {
  std::lock_guard<std::mutex> g(g_cache_mu);
  g_cache[std::make_tuple(key, cur_dev(), extra)] = value;
}
int device_sms() {
  static const char tag = 0;
  int n = 0;
  if (dev_cache_get(&tag, 0, &n)) return n;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, cur_dev());
  dev_cache_put(&tag, 0, n);
  return n;
}
// The attribute is an upper bound, so it only ever grows: the largest size set so far on this device is
// cached (key extra = -2) and smaller requests are no-ops.
int smem_optin(const void* kernel, int bytes) {
  int v = 0;
  if (dev_cache_get(kernel, -2, &v) && v >= bytes) return 0;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) dev_cache_put(kernel, -2, bytes);
  return (int)e;
}
// Programmatic dependent launch on/off: LUFFY_PDL=0 in the environment, or luffy_debug_set_pdl at run time
// (bench.py's per-kernel pass turns it off so a kernel's measured duration excludes its dependency wait).
static std::atomic<int> g_pdl{-1};
bool pdl_enabled() {
  int v = g_pdl.load(std::memory_order_relaxed);
  if (v < 0) {
    const char* e = std::getenv("LUFFY_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
    g_pdl.store(v, std::memory_order_relaxed);
  }
  return v != 0;
}

int gemm_rows_simt(int dtype, int epi, const void* A, const void* B, const void* B3, void* D, void* aux0,
                   const int32_t* off, int G, int64_t max_rows, int N, int K, int b_kmajor, const XRedirect* rd,
                   const XSignal* sig, void* s);
int gemm_wgrad_simt(int dtype, const void* A, const void* B, float* D, float* D3, int Msplit, const int32_t* off, int G,
                    int M, int N, int lda, int ldb, void* s);
int gemm_rows_tc(int epi, const void* A, const void* B, const void* B3, void* D, void* aux0, const int32_t* off, int G,
                 int64_t max_rows, int N, int K, int b_kmajor, const XRedirect* rd, const XSignal* sig, void* s,
                 const XWaitRows* wr = nullptr);
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
  int P, E, El, k, d, f, Tmax, Smax;
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
  m.Smax = c->max_seqs > 0 ? c->max_seqs : 256;
  m.C = (int64_t)m.Tmax * m.k;
  m.Cpad = m.C + (int64_t)m.E * kRowAlign;
  m.Rpad = m.Cpad;
  m.recv = c->max_recv_rows > 0 ? c->max_recv_rows : (int64_t)m.P * m.C + (int64_t)m.El * kRowAlign;
  m.adjw = m.Cpad * m.Cpad / 32;  // sum over groups of npad^2/32 <= (sum npad)^2/32
  return m;
}

// Upper bound of the 256x256 pair tiles over any split of the padded group rows into E groups.
int64_t max_pair_tiles(const Dims& m) {
  const int64_t nt = m.Cpad / 256 + m.E;
  return nt * (nt + 1) / 2;
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
  o->gcopy = cv.take<int32_t>(m.Cpad);
  o->gw = cv.take<float>(m.Cpad);
  o->gchunk = cv.take<int32_t>((size_t)((m.Tmax + 127) / 128) * m.E);
  o->gticket = cv.take<uint32_t>(1);
  o->xg = cv.take<char>(m.Cpad * m.d * es);
  o->gnorm = cv.take<double>(m.Cpad);
  o->adjoff = cv.take<int64_t>(m.E + 1);
  o->adj = cv.take<uint32_t>(m.adjw);
  o->rep_local = cv.take<int32_t>(m.Cpad);
  o->key = cv.take<uint64_t>(m.Cpad);
  o->m1 = cv.take<uint64_t>(m.Cpad);
  o->m2 = cv.take<uint64_t>(m.Cpad);
  o->alive = cv.take<uint32_t>(m.Cpad / 32 + 1);
  o->win = cv.take<uint32_t>(m.Cpad / 32 + 1);
  o->ctrl = cv.take<uint32_t>(64 + kGreedyMaxRounds);
  o->stat64 = cv.take<uint64_t>(4);
  o->x_errw = cv.take<uint32_t>(2);
  o->dseq = cv.take<uint32_t>(1);
  o->gdone = cv.take<uint32_t>(LUFFY_MAX_EXPERTS);
  if (c->fast_measure) {
    o->hone = cv.take<uint32_t>(m.adjw);
    o->hzero = cv.take<uint32_t>(m.adjw);
    o->dec1 = cv.take<uint32_t>(m.adjw);
    o->dec0 = cv.take<uint32_t>(m.adjw);
    o->tskip = cv.take<uint8_t>(max_pair_tiles(m));
  }
  o->nrep = cv.take<int32_t>(m.E);
  o->gnrep = cv.take<int32_t>(m.E);
  o->mrank = cv.take<int32_t>(m.Cpad);
  o->mcnt_row = cv.take<int32_t>(m.Cpad);
  o->soff = cv.take<int32_t>(m.E + 1);
  o->lslot = cv.take<int32_t>(m.Cpad);
  o->perm = cv.take<int32_t>(m.Rpad);
  o->slot_gl = cv.take<int32_t>(m.Rpad);
  o->pos = cv.take<int32_t>(m.C);
  o->rep = cv.take<int32_t>(m.C);
  o->mstart = cv.take<int32_t>(m.Rpad);
  o->mcnt = cv.take<int32_t>(m.Rpad);
  o->mcur = cv.take<int32_t>(m.Rpad);
  o->marr = cv.take<int32_t>(m.Rpad);
  o->members = cv.take<int32_t>(m.Cpad);
  o->mslot = cv.take<int32_t>(m.Cpad);
  o->mpart = cv.take<float>((size_t)(m.Cpad / 16) * 2 * m.d);
  o->roff = cv.take<int32_t>(m.El + 1);
  o->cnt_all = cv.take<int32_t>((size_t)m.P * m.E);
  o->send = m.P > 1 ? cv.take<char>(m.Rpad * m.d * es) : nullptr;
  if (m.P > 1) {
    o->x_peer_recv = cv.take<void*>(2 * m.P);
    o->x_peer_gathered = cv.take<void*>(m.P);
    o->x_peer_dexp = cv.take<void*>(m.P);
    o->x_peer_dsend = cv.take<void*>(m.P);
    o->x_peer_cnt = cv.take<int32_t*>(m.P);
    o->x_flagptr = cv.take<uint32_t*>((size_t)XP_NUM * m.P);
    o->x_dst_base = cv.take<int32_t>(m.E);
    o->x_src_soff = cv.take<int32_t>((size_t)m.P * (m.E + 1));
    o->x_rank_of = cv.take<int32_t>(m.recv);
    o->x_slot_of = cv.take<int32_t>(m.recv);
    o->seq_start = cv.take<int32_t>(m.Smax + 1);
    o->seq_dest_l = cv.take<int32_t>(m.Smax);
    o->out_start = cv.take<int32_t>(m.Smax);
    o->seq_bits = cv.take<uint32_t>((size_t)m.Smax * (m.Rpad / 32));
    o->dmask = cv.take<unsigned long long>(m.Rpad);
    o->x_peer_rowmask = cv.take<unsigned long long*>(m.P);
    o->x_peer_mig = cv.take<int32_t*>(m.P);
    o->x_peer_meta = cv.take<int32_t*>(m.P);
    o->x_peer_meta_w = cv.take<float*>(m.P);
    o->x_peer_dy_in = cv.take<void*>(m.P);
    o->x_peer_dw_in = cv.take<float*>(m.P);
    o->x_peer_res = cv.take<void*>(m.P);
  }
  o->dl = cv.take<float>((size_t)m.Tmax * m.E);
  o->rpart = cv.take<float>((size_t)((m.d + 1023) / 1024) * m.Tmax * m.E);
  o->wg_part = cv.take<float>((size_t)std::max(wg_parts(m.E, m.d), (m.Tmax + 31) / 32) * m.E * m.d);
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
  if (c->max_seqs < 0) return fail(LUFFY_E_INVALID, "max_seqs must be >= 0");
  if (c->fast_measure != 0 && c->fast_measure != 1) return fail(LUFFY_E_INVALID, "fast_measure must be 0 or 1");
  if (c->fast_measure && c->dtype != LUFFY_BF16)
    return fail(LUFFY_E_UNSUPPORTED, "fast_measure (history shortcuts) needs the bf16 tcgen05 Gram");
  if (c->dtype == LUFFY_BF16 && (c->d_model % 256 || c->d_ffn % 256))
    return fail(LUFFY_E_UNSUPPORTED, "bf16 (tcgen05) path needs d_model and d_ffn multiples of 256");
  const Dims m = dims_of(c);
  if (m.Cpad >= (int64_t)1 << 30) return fail(LUFFY_E_INVALID, "max_tokens * top_k too large");
  if (c->world > kMaxWorld) return fail(LUFFY_E_INVALID, "world > 64 is not supported");
  if (c->world == 1 && c->max_recv_rows > 0 && c->max_recv_rows < m.Rpad)
    return fail(LUFFY_E_INVALID, "world == 1 needs max_recv_rows >= max_tokens*top_k + E*LUFFY_ROW_ALIGN (or 0)");
  return LUFFY_OK;
}

// bf16: tcgen05 tensor cores; fp32: exact SIMT FFMA (tf32 would break the fp32 tolerance).
int gemm_rows(int dtype, int epi, const void* A, const void* B, const void* B3, void* D, void* aux0, const int32_t* off,
              int G, int64_t max_rows, int N, int K, int b_kmajor, void* s, const XRedirect* rd = nullptr,
              const XSignal* sig = nullptr, const XWaitRows* wr = nullptr) {
  if (dtype == LUFFY_BF16) return gemm_rows_tc(epi, A, B, B3, D, aux0, off, G, max_rows, N, K, b_kmajor, rd, sig, s, wr);
  return gemm_rows_simt(dtype, epi, A, B, B3, D, aux0, off, G, max_rows, N, K, b_kmajor, rd, sig, s);
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
int64_t expert_rows_bound(const luffy_layer* L) { return L->P == 1 ? L->Rpad_max : L->recv_max; }

// Exchange region layout (identical offsets on every rank).
struct XLayout {
  size_t recv[2], gathered, dexp, dsend, cnt, flags, counters, rowmask, mig, meta, meta_w, dy_in, dw_in, res, total;
};
XLayout xlayout(const luffy_layer* L) {
  const size_t rb = (size_t)L->d * elem_size(L->dtype);
  XLayout x;
  size_t o = 0;
  auto take = [&](size_t n) { o = (o + 255) / 256 * 256; size_t r = o; o += n; return r; };
  x.recv[0] = take((size_t)L->recv_max * rb);
  x.recv[1] = take((size_t)L->recv_max * rb);
  x.gathered = take((size_t)L->P * L->Rpad_max * rb);  // [source rank][slot]
  x.dexp = take((size_t)L->recv_max * rb);
  x.dsend = take((size_t)L->Rpad_max * rb);
  x.cnt = take(sizeof(int32_t) * L->P * L->E);
  x.flags = take(sizeof(uint32_t) * XP_NUM * L->P);
  x.counters = take(sizeof(uint32_t) * XP_NUM);
  x.rowmask = take(sizeof(unsigned long long) * L->recv_max);
  x.mig = take(sizeof(int32_t) * L->P * L->Smax * L->P);
  x.meta = take(sizeof(int32_t) * (size_t)L->P * L->Tmax * (2 + L->k));
  x.meta_w = take(sizeof(float) * (size_t)L->P * L->Tmax * L->k);
  x.dy_in = take((size_t)L->Tmax * rb);
  x.dw_in = take(sizeof(float) * (size_t)L->Tmax * L->k);
  x.res = take((size_t)L->P * L->Tmax * rb);
  x.total = (o + 4095) / 4096 * 4096;
  return x;
}

// This rank's own rows inside the [source rank][slot] gathered buffer.
void* home_gathered(const luffy_layer* L) {
  return static_cast<char*>(L->x_gathered) + (size_t)L->rank * L->Rpad_max * L->d * elem_size(L->dtype);
}

luffy_status need_open(const luffy_layer* L, const char* where) {
  if (L->P > 1 && !L->x_open)
    return fail(LUFFY_E_STATE, std::string(where) + ": world > 1 needs luffy_layer_ipc_open first");
  return LUFFY_OK;
}
#define LUFFY_OPEN(L, where)                             \
  do {                                                   \
    luffy_status _s = need_open((L), (where));           \
    if (_s != LUFFY_OK) return _s;                       \
  } while (0)

// A cross-rank wait of an earlier call timed out (exchange.cuh xwait_flag): the layer is unusable.
luffy_status exchange_health(const luffy_layer* L, const char* where) {
  if (L->P > 1 && L->x_err_h) {
    const uint32_t ph = *reinterpret_cast<volatile const uint32_t*>(L->x_err_h);
    if (ph != 0u) {
      static const char* names[] = {"counts", "dispatch", "combine", "combine_bwd", "dispatch_bwd", "migration rows",
                                    "migration meta", "migration bwd"};
      const uint32_t sq = reinterpret_cast<volatile const uint32_t*>(L->x_err_h)[1];
      return fail(LUFFY_E_STATE, std::string(where) + ": an exchange wait timed out (phase " +
                                     (ph - 1 < XP_NUM ? names[ph - 1] : "?") + ", step " + std::to_string(sq) +
                                     "): a peer rank stopped participating; the layer must be recreated");
    }
  }
  return LUFFY_OK;
}
#define LUFFY_HEALTHY(L, where)                          \
  do {                                                   \
    luffy_status _s = exchange_health((L), (where));     \
    if (_s != LUFFY_OK) return _s;                       \
  } while (0)

}  // namespace
}  // namespace luffy

using namespace luffy;

extern "C" {

const char* luffy_last_error(void) { return g_err.c_str(); }

luffy_status luffy_exchange_plan(int32_t world, int32_t rank, int32_t num_experts, const int32_t* counts_all,
                                 int32_t* send_off, int32_t* recv_off, int32_t* dst_base, int32_t* rank_of,
                                 int32_t* slot_of, int64_t row_capacity, int64_t* send_rows_to, int64_t* recv_rows_from) {
  if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world || num_experts < 1 ||
      num_experts > LUFFY_MAX_EXPERTS || num_experts % world)
    return fail(LUFFY_E_INVALID, "exchange_plan: bad world/rank/num_experts");
  LUFFY_NEED(counts_all);
  LUFFY_NEED(send_off);
  LUFFY_NEED(recv_off);
  const int P = world, E = num_experts, El = E / world;
  for (int i = 0; i < P * E; ++i)
    if (counts_all[i] < 0) return fail(LUFFY_E_INVALID, "exchange_plan: negative count");
  // the same code the device count-exchange kernel runs (xplan.h), on one host thread
  std::vector<int32_t> soff_all((size_t)P * (E + 1)), base(E);
  xplan_body(counts_all, P, E, rank, nullptr, recv_off, base.data(), soff_all.data(), 0, 1);
  std::memcpy(send_off, soff_all.data() + (size_t)rank * (E + 1), sizeof(int32_t) * (E + 1));
  if (dst_base) std::memcpy(dst_base, base.data(), sizeof(int32_t) * E);
  if (rank_of || slot_of) {
    if (!rank_of || !slot_of) return fail(LUFFY_E_INVALID, "exchange_plan: rank_of and slot_of go together");
    if (recv_off[El] > row_capacity) return fail(LUFFY_E_CAPACITY, "exchange_plan: row_capacity < recv_off[E_l]");
    for (int64_t r = 0; r < recv_off[El]; ++r) xplan_row(r, counts_all, recv_off, soff_all.data(), P, E, rank, rank_of + r, slot_of + r);
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
void luffy_debug_set_pdl(int32_t on) { g_pdl.store(on ? 1 : 0, std::memory_order_relaxed); }

luffy_status luffy_create(const luffy_config* cfg, luffy_ctx** out) {
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
  *out = c;
  return LUFFY_OK;
}

void luffy_destroy(luffy_ctx* ctx) { delete ctx; }

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
  {  // the grouping's last-CTA ticket starts at zero (every launch leaves it at zero)
    cudaError_t e = cudaMemset(L->gticket, 0, sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMemset(L->x_errw, 0, 2 * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMemset(L->dseq, 0, sizeof(uint32_t));
    if (e != cudaSuccess) {
      delete L;
      return cuda_fail(e, "luffy_layer_create (workspace init)");
    }
  }
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
  L->Smax = m.Smax;
  L->fast_measure = ctx->cfg.fast_measure != 0;
  L->hist_S1 = 0.8f;   // SPEC S:394 defaults (Fig. 7 probes 0.8 / 0.2); luffy_layer_set_history sets them
  L->hist_S2 = 0.2f;
  if (L->P > 1) {
    // the peer-visible exchange region: allocated once here, mapped by the peers via CUDA IPC
    const XLayout xl = xlayout(L);
    L->x_region_bytes = xl.total;
    cudaError_t e = cudaMalloc(&L->x_region, xl.total);
    if (e == cudaSuccess) e = cudaMemset(L->x_region, 0, xl.total);
    cudaIpcMemHandle_t h;
    if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, L->x_region);
    if (e != cudaSuccess) {
      luffy_layer_destroy(L);
      return cuda_fail(e, "exchange region (cudaMalloc / cudaIpcGetMemHandle)");
    }
    std::memcpy(L->x_handle, &h, sizeof(h));
    // the exchange error word: pinned host memory mapped into the device (read without a sync)
    e = cudaHostAlloc(reinterpret_cast<void**>(&L->x_err_h), 2 * sizeof(uint32_t), cudaHostAllocMapped);
    if (e == cudaSuccess) e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&L->x_err_d), L->x_err_h, 0);
    if (e != cudaSuccess) {
      luffy_layer_destroy(L);
      return cuda_fail(e, "exchange error word (cudaHostAlloc mapped)");
    }
    L->x_err_h[0] = L->x_err_h[1] = 0u;
    {
      const char* v = std::getenv("LUFFY_EXCHANGE_TIMEOUT_MS");
      const long long ms = v ? std::atoll(v) : 20000;
      L->x_timeout_ns = (uint64_t)(ms > 0 ? ms : 20000) * 1000000ull;
    }
    L->x_recv[0] = L->x_region + xl.recv[0];
    L->x_recv[1] = L->x_region + xl.recv[1];
    L->x_gathered = L->x_region + xl.gathered;
    L->x_dexp = L->x_region + xl.dexp;
    L->x_dsend = L->x_region + xl.dsend;
    L->x_cnt_inbox = reinterpret_cast<int32_t*>(L->x_region + xl.cnt);
    L->x_flags = reinterpret_cast<uint32_t*>(L->x_region + xl.flags);
    L->x_counters = reinterpret_cast<uint32_t*>(L->x_region + xl.counters);
    L->x_rowmask = reinterpret_cast<unsigned long long*>(L->x_region + xl.rowmask);
    L->x_mig_inbox = reinterpret_cast<int32_t*>(L->x_region + xl.mig);
    L->x_meta = reinterpret_cast<int32_t*>(L->x_region + xl.meta);
    L->x_meta_w = reinterpret_cast<float*>(L->x_region + xl.meta_w);
    L->x_dy_in = L->x_region + xl.dy_in;
    L->x_dw_in = reinterpret_cast<float*>(L->x_region + xl.dw_in);
    L->x_res = L->x_region + xl.res;
  }
  *out = L;
  return LUFFY_OK;
}

void luffy_layer_destroy(luffy_layer* L) {
  if (!L) return;
  if (L->x_open)
    for (int p = 0; p < L->P; ++p)
      if (p != L->rank && L->x_peer_base_h[p]) cudaIpcCloseMemHandle(L->x_peer_base_h[p]);
  if (L->x_region) cudaFree(L->x_region);
  if (L->x_err_h) cudaFreeHost(L->x_err_h);
  if (L->mig_stage_h) cudaFreeHost(L->mig_stage_h);
  if (L->mig_stage_ev) cudaEventDestroy(static_cast<cudaEvent_t>(L->mig_stage_ev));
  delete L;
}

luffy_status luffy_layer_set_exchange_timeout(luffy_layer* L, int64_t ms) {
  LUFFY_NEED(L);
  if (ms <= 0) return fail(LUFFY_E_INVALID, "luffy_layer_set_exchange_timeout: ms must be > 0");
  L->x_timeout_ns = (uint64_t)ms * 1000000ull;
  return LUFFY_OK;
}

size_t luffy_ipc_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

luffy_status luffy_layer_ipc_handle(const luffy_layer* L, uint8_t* out) {
  LUFFY_NEED(L);
  LUFFY_NEED(out);
  if (L->P == 1) return fail(LUFFY_E_STATE, "luffy_layer_ipc_handle: world == 1 has no exchange region");
  std::memcpy(out, L->x_handle, sizeof(cudaIpcMemHandle_t));
  return LUFFY_OK;
}

luffy_status luffy_layer_ipc_open(luffy_layer* L, const uint8_t* all_handles) {
  LUFFY_NEED(L);
  LUFFY_NEED(all_handles);
  if (L->P == 1) return LUFFY_OK;
  if (L->x_open) return fail(LUFFY_E_STATE, "luffy_layer_ipc_open: already open");
  const XLayout xl = xlayout(L);
  const size_t hb = sizeof(cudaIpcMemHandle_t);
  for (int p = 0; p < L->P; ++p) {
    if (p == L->rank) {
      if (std::memcmp(all_handles + p * hb, L->x_handle, hb) != 0)
        return fail(LUFFY_E_INVALID, "luffy_layer_ipc_open: entry of this rank is not its own handle");
      L->x_peer_base_h[p] = L->x_region;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, all_handles + p * hb, hb);
    void* base = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
    L->x_peer_base_h[p] = base;
  }
  // device tables of peer addresses
  const int P = L->P;
  std::vector<void*> recv(2 * P), gath(P), dexp(P), dsend(P);
  std::vector<int32_t*> cnt(P), mig(P), meta(P);
  std::vector<uint32_t*> flag((size_t)XP_NUM * P);
  std::vector<unsigned long long*> rowmask(P);
  std::vector<float*> meta_w(P), dw_in(P);
  std::vector<void*> dy_in(P), res(P);
  for (int p = 0; p < P; ++p) {
    char* b = static_cast<char*>(L->x_peer_base_h[p]);
    recv[p] = b + xl.recv[0];
    recv[P + p] = b + xl.recv[1];
    gath[p] = b + xl.gathered;
    dexp[p] = b + xl.dexp;
    dsend[p] = b + xl.dsend;
    cnt[p] = reinterpret_cast<int32_t*>(b + xl.cnt);
    mig[p] = reinterpret_cast<int32_t*>(b + xl.mig);
    meta[p] = reinterpret_cast<int32_t*>(b + xl.meta);
    meta_w[p] = reinterpret_cast<float*>(b + xl.meta_w);
    rowmask[p] = reinterpret_cast<unsigned long long*>(b + xl.rowmask);
    dy_in[p] = b + xl.dy_in;
    dw_in[p] = reinterpret_cast<float*>(b + xl.dw_in);
    res[p] = b + xl.res;
    for (int ph = 0; ph < XP_NUM; ++ph)
      flag[(size_t)ph * P + p] = reinterpret_cast<uint32_t*>(b + xl.flags) + ph * P + L->rank;
  }
  LUFFY_CHECK(cudaMemcpy(L->x_peer_recv, recv.data(), sizeof(void*) * 2 * P, cudaMemcpyHostToDevice), "ipc tables");
  LUFFY_CHECK(cudaMemcpy(L->x_peer_gathered, gath.data(), sizeof(void*) * P, cudaMemcpyHostToDevice), "ipc tables");
  LUFFY_CHECK(cudaMemcpy(L->x_peer_dexp, dexp.data(), sizeof(void*) * P, cudaMemcpyHostToDevice), "ipc tables");
  LUFFY_CHECK(cudaMemcpy(L->x_peer_dsend, dsend.data(), sizeof(void*) * P, cudaMemcpyHostToDevice), "ipc tables");
  LUFFY_CHECK(cudaMemcpy(L->x_peer_cnt, cnt.data(), sizeof(int32_t*) * P, cudaMemcpyHostToDevice), "ipc tables");
  LUFFY_CHECK(cudaMemcpy(L->x_flagptr, flag.data(), sizeof(uint32_t*) * XP_NUM * P, cudaMemcpyHostToDevice), "ipc tables");
  LUFFY_CHECK(cudaMemcpy(L->x_peer_rowmask, rowmask.data(), sizeof(void*) * P, cudaMemcpyHostToDevice), "ipc tables");
  LUFFY_CHECK(cudaMemcpy(L->x_peer_mig, mig.data(), sizeof(void*) * P, cudaMemcpyHostToDevice), "ipc tables");
  LUFFY_CHECK(cudaMemcpy(L->x_peer_meta, meta.data(), sizeof(void*) * P, cudaMemcpyHostToDevice), "ipc tables");
  LUFFY_CHECK(cudaMemcpy(L->x_peer_meta_w, meta_w.data(), sizeof(void*) * P, cudaMemcpyHostToDevice), "ipc tables");
  LUFFY_CHECK(cudaMemcpy(L->x_peer_dy_in, dy_in.data(), sizeof(void*) * P, cudaMemcpyHostToDevice), "ipc tables");
  LUFFY_CHECK(cudaMemcpy(L->x_peer_dw_in, dw_in.data(), sizeof(void*) * P, cudaMemcpyHostToDevice), "ipc tables");
  LUFFY_CHECK(cudaMemcpy(L->x_peer_res, res.data(), sizeof(void*) * P, cudaMemcpyHostToDevice), "ipc tables");
  L->x_open = true;
  return LUFFY_OK;
}

luffy_status luffy_layer_rows(const luffy_layer* L, int64_t* send_rows, int64_t* recv_rows) {
  LUFFY_NEED(L);
  LUFFY_STAGE(L, 3, "luffy_layer_rows");
  int32_t so = 0, ro = 0;
  LUFFY_CHECK(cudaMemcpy(&so, L->soff + L->E, sizeof(int32_t), cudaMemcpyDeviceToHost), "rows");
  LUFFY_CHECK(cudaMemcpy(&ro, (L->P == 1 ? L->soff + L->E : L->roff + L->El), sizeof(int32_t), cudaMemcpyDeviceToHost),
              "rows");
  if (send_rows) *send_rows = so;
  if (recv_rows) *recv_rows = ro;
  return LUFFY_OK;
}

// ------------------------------------------------------------------------------------------ forward

luffy_status luffy_route(luffy_layer* L, const void* x, const float* w_gate, int32_t T, int32_t* topk_idx,
                         float* topk_w, void* stream) {
  LUFFY_NEED(L);
  LUFFY_HEALTHY(L, "luffy_route");
  LUFFY_NEED(x);
  LUFFY_NEED(w_gate);
  LUFFY_NEED(topk_idx);
  LUFFY_NEED(topk_w);
  LUFFY_ALIGNED(x);
  LUFFY_ALIGNED(w_gate);
  if (T < 1 || T > L->Tmax) return fail(LUFFY_E_INVALID, "need 0 < T <= max_tokens");
  L->T = T;
  L->wg_route = w_gate;
  L->stage = 0;
  L->seq += 1;  // a new forward step (every rank calls in lockstep)
  L->S = 0;
  L->mig = false;
  if (L->P > 1) LUFFY_CHECK(launch_xstep(L, stream), "luffy_route/step");
  LUFFY_CHECK(launch_route(L, x, w_gate, topk_idx, topk_w, stream), "luffy_route");
  L->stage = 1;
  return LUFFY_OK;
}

luffy_status luffy_condense(luffy_layer* L, const void* x, float h, int32_t* rep, luffy_condense_stats* stats,
                            void* stream) {
  LUFFY_NEED(L);
  LUFFY_HEALTHY(L, "luffy_condense");
  LUFFY_NEED(x);
  LUFFY_NEED(rep);
  LUFFY_ALIGNED(x);
  LUFFY_STAGE(L, 1, "luffy_condense");
  if (!(h == h)) return fail(LUFFY_E_INVALID, "h is NaN");
  L->h = h;
  unsigned long long* band = nullptr;  // stats: near-threshold pair count from the Gram epilogue
  if (stats) {
    LUFFY_CHECK(cudaMemsetAsync(L->stat64, 0, 4 * sizeof(uint64_t), static_cast<cudaStream_t>(stream)), "stats");
    band = reinterpret_cast<unsigned long long*>(L->stat64);
    LUFFY_CHECK(launch_near_tie(L, x, L->wg_route, reinterpret_cast<unsigned long long*>(L->stat64) + 1, stream),
                "luffy_condense/near_tie");
  }
  LUFFY_CHECK(launch_group_build(L, x, stream), "luffy_condense/group_build");
  if (L->hist_prev) {
    const luffy_layer* P = L->hist_prev;
    if (P->T != L->T || P->stage < 2)
      return fail(LUFFY_E_STATE, "luffy_condense: the history layer must be condensed earlier in this step on the same T tokens");
  }
  L->hist_valid = false;
  if (h > 1.0f) {
    L->has_adj = false;
    LUFFY_CHECK(launch_identity_rep(L, stream), "luffy_condense/identity");
  } else {
    L->has_adj = true;
    // bf16: tcgen05 Gram; fp32: exact SIMT FFMA Gram
    L->gdone_live = L->dtype == LUFFY_BF16;
    if (L->dtype == LUFFY_BF16) LUFFY_CHECK(launch_gram_tc(L, h, band, stream), "luffy_condense/gram");
    else LUFFY_CHECK(launch_gram_simt(L, h, band, stream), "luffy_condense/gram");
    LUFFY_CHECK(launch_greedy(L, stream), "luffy_condense/greedy");
    L->hist_valid = L->fast_measure;
  }
  LUFFY_CHECK(launch_pack(L, x, nullptr, rep, stream), "luffy_condense/layout");
  L->stage = 2;
  if (stats) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::vector<int32_t> gc(L->E), nr(L->E);
    uint32_t rounds = 0;
    uint64_t s64[4] = {0, 0, 0, 0};
    LUFFY_CHECK(cudaMemcpyAsync(s64, L->stat64, sizeof(s64), cudaMemcpyDeviceToHost, st), "stats");
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
    stats->ambiguous_pairs = (int64_t)s64[0];
    stats->near_tie_tokens = (int64_t)s64[1];
    stats->decided_pairs = (int64_t)s64[2];
    stats->skipped_tiles = (int64_t)s64[3];
  }
  return LUFFY_OK;
}

// world > 1: the layer's own exchange buffers are the only valid expert-side / gathered buffers; the
// caller passes NULL (or the same pointer, from luffy_layer_exchange_buffers).
static luffy_status own_or_null(const void* given, const void* own, const char* name) {
  if (given != nullptr && given != own)
    return fail(LUFFY_E_INVALID, std::string(name) + ": with world > 1 pass NULL (the layer's exchange buffer is used)");
  return LUFFY_OK;
}
#define LUFFY_OWN(given, own, name)                               \
  do {                                                            \
    luffy_status _s = own_or_null((given), (own), (name));        \
    if (_s != LUFFY_OK) return _s;                                \
  } while (0)

luffy_status luffy_layer_exchange_buffers(const luffy_layer* L, void** recv, void** gathered, void** d_expert_out,
                                          void** d_send) {
  LUFFY_NEED(L);
  if (L->P == 1) return fail(LUFFY_E_STATE, "luffy_layer_exchange_buffers: world == 1 uses caller buffers");
  if (recv) *recv = L->x_recv[L->seq & 1];
  if (gathered) *gathered = home_gathered(L);
  if (d_expert_out) *d_expert_out = L->x_dexp;
  if (d_send) *d_send = L->x_dsend;
  return LUFFY_OK;
}

luffy_status luffy_dispatch(luffy_layer* L, const void* x, void* recv, int64_t* recv_rows, void* stream) {
  LUFFY_NEED(L);
  LUFFY_HEALTHY(L, "luffy_dispatch");
  LUFFY_NEED(x);
  LUFFY_ALIGNED(x);
  LUFFY_STAGE(L, 2, "luffy_dispatch");
  LUFFY_OPEN(L, "luffy_dispatch");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (L->P == 1) {
    LUFFY_NEED(recv);
    LUFFY_ALIGNED(recv);
    LUFFY_CHECK(launch_pack_rows(L, x, recv, stream), "luffy_dispatch/pack");
  } else {
    LUFFY_OWN(recv, L->x_recv[L->seq & 1], "luffy_dispatch recv");
    LUFFY_CHECK(launch_xdispatch(L, x, stream), "luffy_dispatch/exchange");
  }
  L->stage = 3;
  if (recv_rows) {
    int32_t r = 0;
    LUFFY_CHECK(cudaMemcpyAsync(&r, L->P == 1 ? L->soff + L->E : L->roff + L->El, sizeof(int32_t),
                                cudaMemcpyDeviceToHost, st), "rows");
    LUFFY_CHECK(cudaStreamSynchronize(st), "rows sync");
    *recv_rows = r;
  }
  return LUFFY_OK;
}

luffy_status luffy_expert_ffn(luffy_layer* L, const void* recv, const void* w1, const void* w2, const void* w3, void* out,
                              void* saved_pre, void* saved_act, void* stream) {
  LUFFY_NEED(L);
  LUFFY_HEALTHY(L, "luffy_expert_ffn");
  LUFFY_NEED(w1);
  LUFFY_NEED(w2);
  LUFFY_NEED(saved_pre);
  LUFFY_NEED(saved_act);
  LUFFY_STAGE(L, 3, "luffy_expert_ffn");
  if (L->act == LUFFY_SWIGLU && !w3) return fail(LUFFY_E_INVALID, "SWIGLU needs w3");
  const int32_t* off = expert_off(L);
  const int64_t rows = expert_rows_bound(L);
  XRedirect rd{};
  XSignal sig{};
  if (L->P == 1) {
    LUFFY_NEED(recv);
    LUFFY_NEED(out);
  } else {
    LUFFY_OWN(recv, L->x_recv[L->seq & 1], "luffy_expert_ffn recv");
    recv = L->x_recv[L->seq & 1];
    rd.rank_of = L->x_rank_of;  // fused combine: GEMM2 rows go to the gathered buffer of every rank in the
    rd.slot_of = L->x_slot_of;  // row's destination mask (the source, or the hosts of migrated sequences)
    rd.peer_base = L->x_peer_gathered;
    rd.mask = L->x_rowmask;
    rd.stride = L->Rpad_max;
    sig = make_signal(L, XP_COMB);
  }
  // fused dispatch (bf16): GEMM1 waits per tile for the source ranks of its rows (see launch_xdispatch)
  XWaitRows wr{};
  const bool tile_wait = L->P > 1 && L->dtype == LUFFY_BF16;
  if (tile_wait) {
    wr.flags = L->x_flags + XP_DISP * L->P;
    wr.seqp = L->dseq;
    wr.P = L->P;
    wr.E = L->E;
    wr.El = L->El;
    wr.me = L->rank;
    wr.cnt_all = L->cnt_all;
    wr.roff = L->roff;
    wr.err = make_xerr(L);
  }
  if (L->act == LUFFY_GELU) {
    LUFFY_CHECK(gemm_rows(L->dtype, EPI_GELU, recv, w1, nullptr, saved_act, saved_pre, off, L->El, rows, L->f, L->d, 1, stream,
                          nullptr, nullptr, tile_wait ? &wr : nullptr),
                "expert_ffn/gemm1");
  } else {
    LUFFY_CHECK(gemm_rows(L->dtype, EPI_SWIGLU, recv, w1, w3, saved_act, saved_pre, off, L->El, rows, 2 * L->f, L->d, 1, stream,
                          nullptr, nullptr, tile_wait ? &wr : nullptr),
                "expert_ffn/gemm1");
  }
  LUFFY_CHECK(gemm_rows(L->dtype, EPI_STORE, saved_act, w2, nullptr, out, nullptr, off, L->El, rows, L->d, L->f, 1, stream,
                        L->P > 1 ? &rd : nullptr, L->P > 1 ? &sig : nullptr),
              "expert_ffn/gemm2");
  if (L->stage < 4) L->stage = 4;
  return LUFFY_OK;
}

luffy_status luffy_combine(luffy_layer* L, const void* expert_out, void* gathered, void* stream) {
  LUFFY_NEED(L);
  LUFFY_HEALTHY(L, "luffy_combine");
  LUFFY_STAGE(L, 4, "luffy_combine");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (L->P == 1) {
    LUFFY_NEED(expert_out);
    LUFFY_NEED(gathered);
    if (gathered != expert_out)
      LUFFY_CHECK(cudaMemcpyAsync(gathered, expert_out, (size_t)L->Rpad_max * L->d * elem_size(L->dtype),
                                  cudaMemcpyDeviceToDevice, st), "combine copy");
  } else {
    // the rows were pushed by the experts' GEMM2 epilogues; wait until every rank has published them
    LUFFY_OWN(gathered, home_gathered(L), "luffy_combine gathered");
    if (L->mig) {  // tokens of migrated sequences: their slots and gate weights go to the hosting rank
      LUFFY_CHECK(launch_mig_meta_push(L, stream), "luffy_combine/meta");
      LUFFY_CHECK(launch_xwait(L, XP_META, stream), "luffy_combine/meta wait");
    }
    LUFFY_CHECK(launch_xwait(L, XP_COMB, stream), "luffy_combine/wait");
  }
  L->stage = 5;
  return LUFFY_OK;
}

static luffy_status uncondense_impl(luffy_layer* L, const void* gathered, const void* res, void* y, void* stream,
                                    const char* name) {
  LUFFY_NEED(L);
  LUFFY_HEALTHY(L, name);
  LUFFY_NEED(y);
  LUFFY_ALIGNED(y);
  LUFFY_STAGE(L, 5, name);
  if (res) LUFFY_ALIGNED(res);
  if (L->P == 1) {
    LUFFY_NEED(gathered);
  } else {
    LUFFY_OWN(gathered, home_gathered(L), name);
    gathered = home_gathered(L);
    if (L->mig) {  // y holds the tokens of the sequences this rank hosts (luffy_migration_out_tokens)
      LUFFY_CHECK(launch_uncondense_mig(L, res, y, stream), name);
      L->stage = 6;
      return LUFFY_OK;
    }
  }
  LUFFY_CHECK(launch_uncondense(L, gathered, res, y, stream), name);
  L->stage = 6;
  return LUFFY_OK;
}

luffy_status luffy_uncondense(luffy_layer* L, const void* gathered, void* y, void* stream) {
  return uncondense_impl(L, gathered, nullptr, y, stream, "luffy_uncondense");
}

luffy_status luffy_uncondense_residual(luffy_layer* L, const void* gathered, const void* x, void* y, void* stream) {
  LUFFY_NEED(x);
  return uncondense_impl(L, gathered, x, y, stream, "luffy_uncondense_residual");
}

// ------------------------------------------------------------------------------------------ backward

luffy_status luffy_uncondense_bwd(luffy_layer* L, const void* dy, const void* gathered, void* d_gathered, float* d_topk_w,
                                  void* stream) {
  LUFFY_NEED(L);
  LUFFY_HEALTHY(L, "luffy_uncondense_bwd");
  LUFFY_NEED(dy);
  LUFFY_NEED(d_topk_w);
  LUFFY_ALIGNED(dy);
  LUFFY_STAGE(L, 6, "luffy_uncondense_bwd");
  if (L->P == 1) {
    LUFFY_NEED(gathered);
    LUFFY_NEED(d_gathered);
  } else {
    LUFFY_OWN(gathered, home_gathered(L), "luffy_uncondense_bwd gathered");
    if (d_gathered) return fail(LUFFY_E_INVALID, "luffy_uncondense_bwd: with world > 1 pass d_gathered = NULL");
    gathered = home_gathered(L);  // (the rows go straight to the experts' ranks: fused combine backward)
    if (L->mig) {
      // dy holds the hosted tokens: d(gate weight) and dY go back to each token's home rank, where the
      // condensed backward then runs on this rank's own tokens
      LUFFY_CHECK(launch_mig_bwd_push(L, dy, stream), "luffy_uncondense_bwd/migration");
      LUFFY_CHECK(cudaMemcpyAsync(d_topk_w, L->x_dw_in, sizeof(float) * L->T * L->k, cudaMemcpyDeviceToDevice,
                                  static_cast<cudaStream_t>(stream)), "dw copy");
      LUFFY_CHECK(launch_uncondense_bwd(L, L->x_dy_in, gathered, nullptr, nullptr, stream), "luffy_uncondense_bwd");
      return LUFFY_OK;
    }
  }
  LUFFY_CHECK(launch_uncondense_bwd(L, dy, gathered, d_gathered, d_topk_w, stream), "luffy_uncondense_bwd");
  return LUFFY_OK;
}

luffy_status luffy_combine_bwd(luffy_layer* L, const void* d_gathered, void* d_expert_out, void* stream) {
  LUFFY_NEED(L);
  LUFFY_HEALTHY(L, "luffy_combine_bwd");
  LUFFY_STAGE(L, 6, "luffy_combine_bwd");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (L->P == 1) {
    LUFFY_NEED(d_gathered);
    LUFFY_NEED(d_expert_out);
    if (d_gathered != d_expert_out)
      LUFFY_CHECK(cudaMemcpyAsync(d_expert_out, d_gathered, (size_t)L->Rpad_max * L->d * elem_size(L->dtype),
                                  cudaMemcpyDeviceToDevice, st), "combine_bwd copy");
    return LUFFY_OK;
  }
  LUFFY_OWN(d_expert_out, L->x_dexp, "luffy_combine_bwd d_expert_out");
  return launch_xwait(L, XP_CBWD, stream) ? fail(LUFFY_E_CUDA, "luffy_combine_bwd/wait") : LUFFY_OK;
}

luffy_status luffy_expert_ffn_bwd(luffy_layer* L, const void* d_out, const void* recv, const void* w1, const void* w2,
                                  const void* w3, const void* saved_pre, const void* saved_act, void* scratch_dpre,
                                  void* d_recv, float* dw1, float* dw2, float* dw3, void* stream) {
  LUFFY_NEED(L);
  LUFFY_HEALTHY(L, "luffy_expert_ffn_bwd");
  LUFFY_NEED(w1);
  LUFFY_NEED(w2);
  LUFFY_NEED(saved_pre);
  LUFFY_NEED(saved_act);
  LUFFY_NEED(scratch_dpre);
  LUFFY_NEED(dw1);
  LUFFY_NEED(dw2);
  LUFFY_STAGE(L, 6, "luffy_expert_ffn_bwd");
  if (L->act == LUFFY_SWIGLU && (!w3 || !dw3)) return fail(LUFFY_E_INVALID, "SWIGLU needs w3 and dw3");
  const int32_t* off = expert_off(L);
  const int64_t rows = expert_rows_bound(L);
  const int d = L->d, f = L->f, G = L->El;
  XRedirect rd{};
  XSignal sig{};
  if (L->P == 1) {
    LUFFY_NEED(d_out);
    LUFFY_NEED(recv);
    LUFFY_NEED(d_recv);
  } else {
    LUFFY_OWN(d_out, L->x_dexp, "luffy_expert_ffn_bwd d_out");
    LUFFY_OWN(recv, L->x_recv[L->seq & 1], "luffy_expert_ffn_bwd recv");
    if (d_recv) return fail(LUFFY_E_INVALID, "luffy_expert_ffn_bwd: with world > 1 pass d_recv = NULL");
    d_out = L->x_dexp;
    recv = L->x_recv[L->seq & 1];
    rd.rank_of = L->x_rank_of;  // fused dispatch backward: dX rows go to their source rank's d_send
    rd.slot_of = L->x_slot_of;
    rd.peer_base = L->x_peer_dsend;
    sig = make_signal(L, XP_DBWD);
  }
  const XRedirect* rdp = L->P > 1 ? &rd : nullptr;
  const XSignal* sgp = L->P > 1 ? &sig : nullptr;
  if (L->act == LUFFY_GELU) {
    LUFFY_CHECK(gemm_rows(L->dtype, EPI_DGELU, d_out, w2, nullptr, scratch_dpre, const_cast<void*>(saved_pre), off, G, rows,
                          f, d, 0, stream), "ffn_bwd/dgrad2");
    LUFFY_CHECK(gemm_rows(L->dtype, EPI_STORE, scratch_dpre, w1, nullptr, d_recv, nullptr, off, G, rows, d, f, 0, stream,
                          rdp, sgp), "ffn_bwd/dgrad1");
    LUFFY_CHECK(gemm_wgrad(L->dtype, d_out, saved_act, dw2, nullptr, d, off, G, d, f, d, f, rows, stream), "ffn_bwd/wgrad2");
    LUFFY_CHECK(gemm_wgrad(L->dtype, scratch_dpre, recv, dw1, nullptr, f, off, G, f, d, f, d, rows, stream), "ffn_bwd/wgrad1");
  } else {
    LUFFY_CHECK(gemm_rows(L->dtype, EPI_DSWIGLU, d_out, w2, nullptr, scratch_dpre, const_cast<void*>(saved_pre), off, G,
                          rows, f, d, 0, stream), "ffn_bwd/dgrad2");
    LUFFY_CHECK(gemm_rows(L->dtype, EPI_STORE, scratch_dpre, w1, w3, d_recv, nullptr, off, G, rows, d, 2 * f, 0, stream,
                          rdp, sgp), "ffn_bwd/dgrad1");
    LUFFY_CHECK(gemm_wgrad(L->dtype, d_out, saved_act, dw2, nullptr, d, off, G, d, f, d, f, rows, stream), "ffn_bwd/wgrad2");
    LUFFY_CHECK(gemm_wgrad(L->dtype, scratch_dpre, recv, dw1, dw3, f, off, G, 2 * f, d, 2 * f, d, rows, stream), "ffn_bwd/wgrad1");
  }
  return LUFFY_OK;
}

static luffy_status dispatch_bwd_impl(luffy_layer* L, const void* d_recv, const void* dy_res, bool residual, void* dx,
                                      void* stream, const char* name) {
  LUFFY_NEED(L);
  LUFFY_HEALTHY(L, name);
  LUFFY_NEED(dx);
  LUFFY_ALIGNED(dx);
  LUFFY_STAGE(L, 6, name);
  const void* dsend = d_recv;
  if (L->P == 1) {
    LUFFY_NEED(d_recv);
  } else {
    if (d_recv) return fail(LUFFY_E_INVALID, std::string(name) + ": with world > 1 pass d_recv = NULL");
    LUFFY_CHECK(launch_xwait(L, XP_DBWD, stream), name);
    dsend = L->x_dsend;
  }
  if (residual) {
    if (L->P > 1 && L->mig) {  // the hosts returned every token's dY to its home (luffy_uncondense_bwd)
      if (dy_res) return fail(LUFFY_E_INVALID, std::string(name) + ": with sequence migration pass dy = NULL");
      dy_res = L->x_dy_in;
    } else {
      LUFFY_NEED(dy_res);
      LUFFY_ALIGNED(dy_res);
    }
  }
  LUFFY_CHECK(launch_unpack_bwd(L, dsend, residual ? dy_res : nullptr, dx, stream), name);
  return LUFFY_OK;
}

luffy_status luffy_dispatch_bwd(luffy_layer* L, const void* d_recv, void* dx, void* stream) {
  return dispatch_bwd_impl(L, d_recv, nullptr, false, dx, stream, "luffy_dispatch_bwd");
}

luffy_status luffy_dispatch_bwd_residual(luffy_layer* L, const void* d_recv, const void* dy, void* dx, void* stream) {
  return dispatch_bwd_impl(L, d_recv, dy, true, dx, stream, "luffy_dispatch_bwd_residual");
}

luffy_status luffy_route_bwd(luffy_layer* L, const void* x, const float* w_gate, const float* d_topk_w, void* dx,
                             float* dw_gate, void* stream) {
  LUFFY_NEED(L);
  LUFFY_HEALTHY(L, "luffy_route_bwd");
  LUFFY_NEED(x);
  LUFFY_NEED(w_gate);
  LUFFY_NEED(d_topk_w);
  LUFFY_NEED(dx);
  LUFFY_NEED(dw_gate);
  LUFFY_STAGE(L, 6, "luffy_route_bwd");
  LUFFY_CHECK(launch_route_bwd(L, x, w_gate, d_topk_w, dx, dw_gate, stream), "luffy_route_bwd");
  return LUFFY_OK;
}

// ------------------------------------------------------------------------------- sequence migration

luffy_status luffy_sequence_rows(luffy_layer* L, const int32_t* seq_len, int32_t num_seqs,
                                 const int32_t* num_seqs_all, int64_t* rows_at_all, void* stream) {
  LUFFY_NEED(L);
  LUFFY_HEALTHY(L, "luffy_sequence_rows");
  LUFFY_NEED(seq_len);
  LUFFY_NEED(rows_at_all);
  LUFFY_STAGE(L, 2, "luffy_sequence_rows");
  if (L->stage >= 3) return fail(LUFFY_E_STATE, "luffy_sequence_rows: must precede luffy_dispatch");
  if (L->P == 1) return fail(LUFFY_E_STATE, "luffy_sequence_rows: sequence migration needs world > 1");
  LUFFY_OPEN(L, "luffy_sequence_rows");
  if (num_seqs < 1 || num_seqs > L->Smax) return fail(LUFFY_E_INVALID, "luffy_sequence_rows: 1 <= num_seqs <= max_seqs");
  std::vector<int32_t> start(num_seqs + 1, 0);
  for (int s = 0; s < num_seqs; ++s) {
    if (seq_len[s] < 1) return fail(LUFFY_E_INVALID, "luffy_sequence_rows: sequence lengths must be >= 1");
    start[s + 1] = start[s] + seq_len[s];
  }
  if (start[num_seqs] != L->T) return fail(LUFFY_E_INVALID, "luffy_sequence_rows: lengths must sum to T");
  for (int q = 0; q < L->P; ++q) {
    const int32_t c = num_seqs_all ? num_seqs_all[q] : num_seqs;
    if (c < 1 || c > L->Smax) return fail(LUFFY_E_INVALID, "luffy_sequence_rows: 1 <= num_seqs_all[q] <= max_seqs");
    L->Sq[q] = c;
  }
  if (L->Sq[L->rank] != num_seqs) return fail(LUFFY_E_INVALID, "luffy_sequence_rows: num_seqs_all[rank] != num_seqs");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  LUFFY_CHECK(cudaMemcpyAsync(L->seq_start, start.data(), sizeof(int32_t) * (num_seqs + 1), cudaMemcpyHostToDevice, st),
              "seq_start");
  L->S = num_seqs;
  LUFFY_CHECK(launch_seq_rows(L, stream), "luffy_sequence_rows");
  std::vector<int32_t> all((size_t)L->P * L->Smax * L->P);
  LUFFY_CHECK(cudaMemcpyAsync(all.data(), L->x_mig_inbox, sizeof(int32_t) * all.size(), cudaMemcpyDeviceToHost, st),
              "rows_at D2H");
  LUFFY_CHECK(cudaStreamSynchronize(st), "rows_at sync");
  size_t row = 0;
  for (int q = 0; q < L->P; ++q)
    for (int s = 0; s < L->Sq[q]; ++s, ++row)
      for (int j = 0; j < L->P; ++j) rows_at_all[row * L->P + j] = all[((size_t)q * L->Smax + s) * L->P + j];
  return LUFFY_OK;
}

luffy_status luffy_set_migration(luffy_layer* L, const int32_t* seq_len_all, const int32_t* seq_dest, int64_t* out_rows,
                                 void* stream) {
  LUFFY_NEED(L);
  LUFFY_HEALTHY(L, "luffy_set_migration");
  LUFFY_NEED(seq_len_all);
  LUFFY_NEED(seq_dest);
  if (L->S < 1) return fail(LUFFY_E_STATE, "luffy_set_migration: call luffy_sequence_rows first (this step)");
  if (L->stage >= 3) return fail(LUFFY_E_STATE, "luffy_set_migration: must precede luffy_dispatch");
  const int P = L->P, S = L->S;
  int total = 0;
  for (int q = 0; q < P; ++q) total += L->Sq[q];
  for (int i = 0; i < total; ++i)
    if (seq_dest[i] < 0 || seq_dest[i] >= P) return fail(LUFFY_E_INVALID, "luffy_set_migration: seq_dest out of range");
  // output rows of each destination: sequences in (home rank, sequence) order
  std::vector<int64_t> fill(P, 0);
  std::vector<int32_t> out_start(S), dest(S);
  int i = 0;
  for (int q = 0; q < P; ++q)
    for (int s = 0; s < L->Sq[q]; ++s, ++i) {
      const int g = seq_dest[i];
      if (q == L->rank) {
        out_start[s] = (int32_t)fill[g];
        dest[s] = g;
      }
      fill[g] += seq_len_all[i];
    }
  if (fill[L->rank] > (int64_t)P * L->Tmax) return fail(LUFFY_E_CAPACITY, "luffy_set_migration: output capacity");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // the per-sequence tables go through the layer's pinned staging buffer (no stream synchronisation): the
  // previous call's copy must have left it first
  if (!L->mig_stage_h) {
    LUFFY_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&L->mig_stage_h), sizeof(int32_t) * 2 * L->Smax, cudaHostAllocDefault),
                "migration staging");
    cudaEvent_t ev;
    LUFFY_CHECK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "migration staging event");
    L->mig_stage_ev = ev;
  } else {
    LUFFY_CHECK(cudaEventSynchronize(static_cast<cudaEvent_t>(L->mig_stage_ev)), "migration staging");
  }
  std::memcpy(L->mig_stage_h, dest.data(), sizeof(int32_t) * S);
  std::memcpy(L->mig_stage_h + L->Smax, out_start.data(), sizeof(int32_t) * S);
  LUFFY_CHECK(cudaMemcpyAsync(L->seq_dest_l, L->mig_stage_h, sizeof(int32_t) * S, cudaMemcpyHostToDevice, st), "seq_dest");
  LUFFY_CHECK(cudaMemcpyAsync(L->out_start, L->mig_stage_h + L->Smax, sizeof(int32_t) * S, cudaMemcpyHostToDevice, st),
              "out_start");
  LUFFY_CHECK(cudaEventRecord(static_cast<cudaEvent_t>(L->mig_stage_ev), st), "migration staging event");
  LUFFY_CHECK(launch_set_migration(L, stream), "luffy_set_migration");
  L->n_out = fill[L->rank];
  L->mig = true;
  if (out_rows) *out_rows = L->n_out;
  return LUFFY_OK;
}

luffy_status luffy_migration_out_tokens(const luffy_layer* L, int32_t* home_rank, int32_t* home_token) {
  LUFFY_NEED(L);
  if (!L->mig) return fail(LUFFY_E_STATE, "luffy_migration_out_tokens: no migration this step");
  if (L->stage < 5) return fail(LUFFY_E_STATE, "luffy_migration_out_tokens: after luffy_combine");
  std::vector<int32_t> m((size_t)L->n_out * (2 + L->k));
  if (!m.empty())
    LUFFY_CHECK(cudaMemcpy(m.data(), L->x_meta, sizeof(int32_t) * m.size(), cudaMemcpyDeviceToHost), "meta D2H");
  for (int64_t i = 0; i < L->n_out; ++i) {
    if (home_rank) home_rank[i] = m[i * (2 + L->k)];
    if (home_token) home_token[i] = m[i * (2 + L->k) + 1];
  }
  return LUFFY_OK;
}

luffy_status luffy_layer_set_history(luffy_layer* L, const luffy_layer* prev, float S1, float S2) {
  LUFFY_NEED(L);
  if (!L->fast_measure) return fail(LUFFY_E_STATE, "luffy_layer_set_history: the layer was created without fast_measure");
  if (!(S2 >= 0.f && S2 < S1 && S1 <= 1.f)) return fail(LUFFY_E_INVALID, "luffy_layer_set_history: need 0 <= S2 < S1 <= 1");
  if (prev == L) return fail(LUFFY_E_INVALID, "luffy_layer_set_history: prev must be another layer");
  if (prev && !prev->fast_measure) return fail(LUFFY_E_INVALID, "luffy_layer_set_history: prev was created without fast_measure");
  if (prev && prev->ctx->device != L->ctx->device) return fail(LUFFY_E_INVALID, "luffy_layer_set_history: prev is on another device");
  L->hist_prev = prev;
  L->hist_S1 = S1;
  L->hist_S2 = S2;
  return LUFFY_OK;
}

luffy_status luffy_debug_gram_dump(luffy_layer* L, float* dst, size_t capacity_floats) {
  LUFFY_NEED(L);
  if (dst && reinterpret_cast<uintptr_t>(dst) % 16) return fail(LUFFY_E_INVALID, "luffy_debug_gram_dump: dst must be 16-byte aligned");
  L->dbg_gram = dst;
  L->dbg_gram_cap = dst ? capacity_floats : 0;
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
    case LUFFY_DBG_HONE: src = L->hone; n = L->hist_valid ? sizeof(uint32_t) * adjE : 0; break;
    case LUFFY_DBG_HZERO: src = L->hzero; n = L->hist_valid ? sizeof(uint32_t) * adjE : 0; break;
    case LUFFY_DBG_DEC1: src = L->dec1; n = (L->hist_valid && L->hist_prev) ? sizeof(uint32_t) * adjE : 0; break;
    case LUFFY_DBG_DEC0: src = L->dec0; n = (L->hist_valid && L->hist_prev) ? sizeof(uint32_t) * adjE : 0; break;
    case LUFFY_DBG_TSKIP: {
      int64_t nt = 0;
      std::vector<int32_t> go(L->E + 1);
      LUFFY_CHECK(cudaMemcpy(go.data(), L->goff, sizeof(int32_t) * (L->E + 1), cudaMemcpyDeviceToHost), "debug");
      for (int e = 0; e < L->E; ++e) {
        const int64_t pb = ((go[e + 1] - go[e]) / 128 + 1) / 2;
        nt += pb * (pb + 1) / 2;
      }
      src = L->tskip;
      n = (L->hist_valid && L->hist_prev) ? nt : 0;
      break;
    }
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
