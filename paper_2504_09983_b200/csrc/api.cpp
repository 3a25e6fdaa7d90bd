// C-ABI runtime: shard store layout, context, schedule binding, and the
// gather / release / reduce-scatter+Adam / offload entry points of dc.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "dc_internal.h"

namespace dc {
static thread_local std::string g_err;
static thread_local int64_t g_launches = 0;
void set_global_error(const std::string& s) { g_err = s; }
void count_launch() { ++g_launches; }
int64_t launch_count() { return g_launches; }
void reset_launch_count() { g_launches = 0; }

static int64_t align256(int64_t b) { return (b + 255) / 256 * 256; }
static int64_t shard_len(int64_t numel, int world) { return (numel + 8LL * world - 1) / (8LL * world) * 8; }

static dc_status make_layout(int world, int n, const int64_t* numel, const int32_t* layer_of, int max_ops,
                             Layout* L, std::string* err) {
  if (world < 1 || world > MAXW) { *err = "world must be in [1, 8]"; return DC_EINVAL; }
  if (n < 1 || !numel || !layer_of) { *err = "empty parameter table"; return DC_EINVAL; }
  L->S.resize(n); L->store_off.resize(n); L->goff.resize(n);
  int64_t off = 0;
  int prev_layer = -1;
  std::map<int, int64_t> slot_bytes;
  for (int i = 0; i < n; ++i) {
    if (numel[i] <= 0) { *err = "numel must be > 0"; return DC_EINVAL; }
    if (layer_of[i] < prev_layer || layer_of[i] < 0) { *err = "layer_of must be non-decreasing"; return DC_EINVAL; }
    if (layer_of[i] != prev_layer) {
      if (layer_of[i] != (int)L->layer_first.size()) { *err = "layers must be numbered 0..L-1"; return DC_EINVAL; }
      L->layer_first.push_back(i);
      L->layer_count.push_back(0);
      prev_layer = layer_of[i];
    }
    L->layer_count.back()++;
    L->S[i] = shard_len(numel[i], world);
    L->store_off[i] = off;
    off += L->S[i];
    L->goff[i] = slot_bytes[layer_of[i]];
    slot_bytes[layer_of[i]] += align256(L->S[i] * world * 2);
  }
  L->shard_elems = off;
  L->n_layers = (int)L->layer_first.size();
  for (auto& kv : slot_bytes) L->grad_slot_bytes = std::max(L->grad_slot_bytes, kv.second);
  const int64_t ops = std::max(max_ops, 1);
  L->f_ready = 0;
  L->f_done = L->f_ready + ops * world;
  L->f_chunk = L->f_done + ops;
  L->f_gready = L->f_chunk + (int64_t)n * world * AG_CHUNKS;
  L->f_gcons = L->f_gready + 2 * world;
  L->f_rsdone = L->f_gcons + 2 * world;
  L->f_scal = L->f_rsdone + 1;
  L->f_dep = L->f_scal + 2;
  L->f_bar = L->f_dep + 1;
  L->flag_words = L->f_bar + 2 * world;
  return DC_OK;
}

}  // namespace dc

using namespace dc;

struct FragInfo {
  int layer, state;
  int64_t off, elems, host_off;
  cudaEvent_t d2h, h2d;
  float* slot = nullptr;      // host-resident mode: device ring slot of an offloaded fragment
};

struct dc_ctx {
  int rank = 0, world = 1, device = 0;
  uint32_t flags = 0;
  int n_params = 0;
  std::vector<int64_t> numel;
  std::vector<int32_t> layer_of;
  Layout L;
  void* shard = nullptr;
  float *master = nullptr, *m = nullptr, *v = nullptr;
  float* grad_acc = nullptr;            // fp32 accumulated grad shard (micro_steps > 1)
  int micro_steps = 1;
  std::vector<uint64_t> grad_peers, flag_peers, arena_peers;
  uint64_t grad_bytes = 0, flag_bytes = 0, arena_bytes = 0;
  void* host_pinned = nullptr;
  uint64_t host_pinned_bytes = 0;
  double lr = 1e-3, beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
  uint64_t seed = 0;
  uint64_t timeout_ns = 20ull * 1000 * 1000 * 1000;
  int max_ops = 0;
  // schedule
  const dc_schedule* sched = nullptr;
  std::map<int, int> op_index;          // schedule op id -> index (ag / rel)
  std::vector<int64_t> cur_off;         // param -> arena byte offset of its live buffer (-1)
  std::vector<int> initial_ready;       // gathers whose ready is posted at step start
  std::map<int, int> ag_ctas;           // gather id -> CTAs per launch
  std::map<int, int> ag_launches;
  uint32_t epoch = 0;                   // caller's step number (monotone)
  uint32_t fepoch = 0;                  // flag epoch: steps since the last bind
  int slot_use[2] = {0, 0};
  std::vector<int> layer_use;
  uint32_t rs_done_total = 0;
  int rs_ctas = 0, rs_threads = 256, rs_ctas_default = 296;
  int rs_bulk = 0;                      // 1: bulk-copy pipelined rs_adam (UPDATE / FINAL), one CTA per SM
  int num_sms = 148;
  // error record (ERR_RECORD_WORDS words): host-mapped pinned, written by the
  // device on a flag-wait timeout: code, claimed, target, observed, address
  uint32_t* err_host = nullptr;
  uint32_t* err_dev = nullptr;
  std::vector<FragInfo> frags;
  // host-resident optimizer states (reading D28)
  bool states_bound = true;             // false from dc_init(DC_DEFER_STATES) until the bind
  bool host_states = false;
  std::vector<float*> lay_m, lay_v;     // per layer: m / v base for rs_adam (ring slot) or null
  cudaEvent_t gt_start = nullptr, gt_end = nullptr;   // one-shot gather timing (profiling)
  int ag_ce = 0;                        // 1: gathers as copy-engine peer copies (no SM time)
  int ag_bulk = 0;                      // 1: the push's data path on the bulk-copy (TMA) engine
  int ag_skip_waits = 0;                // profiling only: push without the ready / done flag waits
  // NVLS: multicast addresses of the arena / grad slots / flag
  // table (dc_bind_multicast; 0 = none) and option "nvls" (bit 0 gathers,
  // bit 1 reduce-scatter)
  uint64_t arena_mc = 0, grad_mc = 0, flags_mc = 0;
  int nvls = 0;
  // fused all-gather -> GEMM (option "fused_ag"): gathers push
  // in chunks and post per-chunk values; the executor's GEMMs wait per tile.
  // ag_inst[gid][j] = 1-based instance of member j's gather among that param's
  // gathers in the schedule; the value posted at flag epoch e is
  // (e - 1) * ag_ninst + instance (monotone over steps and within a step)
  int fused_ag = 0;
  std::map<int, std::vector<uint32_t>> ag_inst;
  uint32_t ag_ninst = 1;
  uint32_t ag_delay_us = 0;             // testing: each push starts this long after its ready wait
  // testing (SURVEY §5 race detection): random delays in [0, jitter_us) before
  // every push, every release's ready posts and every reduce-scatter, from a
  // counter-based hash of (seed, rank, op, epoch) — reorders the ranks
  uint32_t jitter_us = 0, jitter_seed = 0;
  uint32_t jitter(int op) const {
    if (!jitter_us) return 0;
    uint64_t z = ((uint64_t)jitter_seed << 40) ^ ((uint64_t)rank << 32) ^ ((uint64_t)(uint32_t)op << 12) ^ fepoch;
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return (uint32_t)((z ^ (z >> 31)) % jitter_us);
  }
  // push CTAs per gather: 64 x 256 threads x 8 x 16 B keeps ~2 MB of stores in
  // flight (NVLink latency x 900 GB/s) and fits beside a GEMM CTA per SM
  int ag_max_ctas = 64;
  // graph mode (N = 1): every step restarts the grad-slot / rs counters and
  // their flags from zero and reads its Adam scalars from device memory, so a
  // captured step replays unchanged (dc_model_graph_capture)
  bool graph_mode = false;
  std::string err;

  uint32_t* flag(int q, int64_t word) const { return reinterpret_cast<uint32_t*>(flag_peers[q]) + word; }
  uint32_t* myflag(int64_t word) const { return flag(rank, word); }
  uint8_t* slot_ptr(int q, int s) const { return reinterpret_cast<uint8_t*>(grad_peers[q]) + (int64_t)s * L.grad_slot_bytes; }
};

static dc_status fail(dc_ctx* c, dc_status s, const std::string& m) {
  if (c) c->err = m;
  set_global_error(m);
  return s;
}

// Which flag a timed-out wait was spinning on, from the address in the
// error record: the table (by peer base address) and the word's role in the
// flag layout (make_layout).
static std::string describe_flag(const dc_ctx* c, uint64_t addr) {
  const Layout& L = c->L;
  for (int q = 0; q < (int)c->flag_peers.size(); ++q) {
    const uint64_t base = c->flag_peers[q];
    if (addr < base || addr >= base + (uint64_t)L.flag_words * 4) continue;
    const int64_t w = (int64_t)(addr - base) / 4;
    char b[160];
    const int W = c->world;
    if (w < L.f_done)
      snprintf(b, sizeof b, "ready[gather %lld][sender %lld]", (long long)(w / W), (long long)(w % W));
    else if (w < L.f_chunk)
      snprintf(b, sizeof b, "done[gather %lld]", (long long)(w - L.f_done));
    else if (w < L.f_gready)
      snprintf(b, sizeof b, "chunk[param %lld][sender %lld][%lld]", (long long)((w - L.f_chunk) / (W * AG_CHUNKS)),
               (long long)((w - L.f_chunk) / AG_CHUNKS % W), (long long)((w - L.f_chunk) % AG_CHUNKS));
    else if (w < L.f_gcons)
      snprintf(b, sizeof b, "grad_ready[slot %lld][sender %lld]", (long long)((w - L.f_gready) / W),
               (long long)((w - L.f_gready) % W));
    else if (w < L.f_rsdone)
      snprintf(b, sizeof b, "consumed[slot %lld][owner %lld]", (long long)((w - L.f_gcons) / W),
               (long long)((w - L.f_gcons) % W));
    else if (w >= L.f_bar)
      snprintf(b, sizeof b, "step_barrier[round %lld][rank %lld]", (long long)((w - L.f_bar) / W),
               (long long)((w - L.f_bar) % W));
    else
      snprintf(b, sizeof b, "word %lld", (long long)w);
    return std::string(b) + " in rank " + std::to_string(q) + "'s flag table";
  }
  char b[48];
  snprintf(b, sizeof b, "address 0x%llx (not a flag table)", (unsigned long long)addr);
  return b;
}

static dc_status check_sticky(dc_ctx* c) {
  volatile uint32_t* e = c->err_host;
  if (e && e[0]) {
    static const char* what[] = {"?", "gather: receivers ready", "gather: stores landed", "reduce-scatter: grads ready",
                                 "flag wait", "graph step barrier", "GEMM: gathered chunk landed"};
    const uint32_t code = e[0];
    const uint32_t k = (code >> 8) < 7 ? (code >> 8) : 0;
    const uint64_t addr = (uint64_t)e[4] | ((uint64_t)e[5] << 32);
    char b[160];
    snprintf(b, sizeof b, "rank %d: device flag wait timed out after %.1f s (code 0x%x, %s) on ", c->rank,
             c->timeout_ns * 1e-9, code, what[k]);
    char v[96];
    snprintf(v, sizeof v, ": observed %u, waiting for >= %u", e[3], e[2]);
    return fail(c, DC_ETIMEOUT, b + describe_flag(c, addr) + v);
  }
  return DC_OK;
}

extern "C" const char* dc_last_error(const dc_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }
extern "C" const char* dc_version(void) { return "dc-b200 0.1 (sm_100a)"; }

extern "C" dc_status dc_layout_query(const dc_layout_args* a, dc_layout* out) {
  if (!a || !out) { set_global_error("dc_layout_query: null argument"); return DC_EINVAL; }
  Layout L;
  std::string err;
  dc_status s = make_layout(a->world, a->n_params, a->numel, a->layer_of, a->max_s0_ops, &L, &err);
  if (s != DC_OK) { set_global_error(err); return s; }
  out->shard_elems = L.shard_elems;
  out->grad_slot_bytes = L.grad_slot_bytes;
  out->flag_bytes = L.flag_words * 4;
  out->n_layers = L.n_layers;
  return DC_OK;
}

extern "C" dc_status dc_init(const dc_init_args* a, dc_ctx** out) {
  if (!a || !out) { set_global_error("dc_init: null argument"); return DC_EINVAL; }
  auto c = std::make_unique<dc_ctx>();
  std::string err;
  dc_status s = make_layout(a->world, a->n_params, a->numel, a->layer_of, a->max_s0_ops, &c->L, &err);
  if (s != DC_OK) return fail(nullptr, s, "dc_init: " + err);
  if (a->rank < 0 || a->rank >= a->world) return fail(nullptr, DC_EINVAL, "dc_init: rank out of range");
  const bool defer = (a->flags & DC_DEFER_STATES) != 0;
  if (!a->shard_param || !a->master || (!defer && (!a->exp_avg || !a->exp_avg_sq)) || !a->grad_peer_ptrs ||
      !a->flag_peer_ptrs)
    return fail(nullptr, DC_EINVAL, "dc_init: null buffer");
  if (a->grad_bytes < (uint64_t)(2 * c->L.grad_slot_bytes)) return fail(nullptr, DC_EOOM, "dc_init: grad buffer < 2 slots");
  if (a->flag_bytes < (uint64_t)(c->L.flag_words * 4)) return fail(nullptr, DC_EOOM, "dc_init: flag table too small");
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (!al16(a->shard_param) || !al16(a->master) || !al16(a->exp_avg) || !al16(a->exp_avg_sq) || !al16(a->grad_acc))
    return fail(nullptr, DC_EINVAL, "dc_init: buffers must be 16-byte aligned");
  if (a->micro_steps < 0 || a->micro_steps > 4096) return fail(nullptr, DC_EINVAL, "dc_init: micro_steps in [0, 4096]");
  if (a->micro_steps > 1 && !a->grad_acc) return fail(nullptr, DC_EINVAL, "dc_init: micro_steps > 1 needs grad_acc");
  c->rank = a->rank; c->world = a->world; c->device = a->device; c->flags = a->flags;
  c->n_params = a->n_params;
  c->numel.assign(a->numel, a->numel + a->n_params);
  c->layer_of.assign(a->layer_of, a->layer_of + a->n_params);
  c->shard = a->shard_param; c->master = a->master; c->m = a->exp_avg; c->v = a->exp_avg_sq;
  c->micro_steps = std::max(1, a->micro_steps);
  c->grad_acc = a->grad_acc;
  c->grad_peers.assign(a->grad_peer_ptrs, a->grad_peer_ptrs + a->world);
  c->flag_peers.assign(a->flag_peer_ptrs, a->flag_peer_ptrs + a->world);
  c->grad_bytes = a->grad_bytes; c->flag_bytes = a->flag_bytes;
  c->host_pinned = a->host_pinned; c->host_pinned_bytes = a->host_pinned_bytes;
  c->lr = a->lr; c->beta1 = a->beta1; c->beta2 = a->beta2; c->eps = a->eps;
  c->seed = a->seed;
  c->max_ops = std::max(a->max_s0_ops, 1);
  if (a->spin_limit) c->timeout_ns = (uint64_t)a->spin_limit * 1000ull * 1000ull;   // spin_limit in ms
  c->cur_off.assign(a->n_params, -1);
  c->layer_use.assign(c->L.n_layers, 0);
  // rs_adam grid.  N = 1: two 256-thread CTAs per SM — a local HBM-bound pass,
  // fastest when it has the SMs to itself (profiles/r01g/rs_coresidency_ab.md).
  // N > 1: one 128-thread CTA per SM (128 x 112 registers fits beside a pair-GEMM
  // CTA), so the NVLink-bound reduce-scatter of layer l+1 runs during layer l's
  // backward GEMMs instead of waiting for their SMs.  DC_RS_CTAS / DC_RS_THREADS override.
  c->rs_ctas = a->world > 1 ? 148 : 296;
  c->rs_threads = a->world > 1 ? 128 : 256;
  c->rs_ctas_default = c->rs_ctas;
  if (const char* e = getenv("DC_RS_CTAS")) c->rs_ctas = std::max(1, atoi(e));
  if (const char* e = getenv("DC_RS_THREADS")) c->rs_threads = atoi(e) == 128 ? 128 : 256;
  DC_CUDA_TRY(cudaSetDevice(a->device), &c->err);
  DC_CUDA_TRY(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, a->device), &c->err);
  // bulk-copy rs_adam at N = 1: 5.75 vs 4.9 TB/s in-step (profiles/r02/rs_bulk/);
  // at N > 1 the LDG kernel's small CTAs co-reside with the backward GEMMs it overlaps
  c->rs_bulk = a->world == 1;
  if (const char* e = getenv("DC_RS_BULK")) c->rs_bulk = atoi(e) != 0;
  if (const char* e = getenv("DC_AG_MAX_CTAS")) c->ag_max_ctas = std::max(1, std::min(1024, atoi(e)));
  DC_CUDA_TRY(preload_glue_kernels(), &c->err);
  DC_CUDA_TRY(preload_comm_kernels(), &c->err);
  DC_CUDA_TRY(preload_nvls_kernels(), &c->err);
  DC_CUDA_TRY(preload_gemm_kernels(), &c->err);
  DC_CUDA_TRY(preload_moe_kernels(), &c->err);
  DC_CUDA_TRY(cudaHostAlloc(&c->err_host, ERR_RECORD_WORDS * 4, cudaHostAllocMapped), &c->err);
  memset(c->err_host, 0, ERR_RECORD_WORDS * 4);
  DC_CUDA_TRY(cudaHostGetDevicePointer(&c->err_dev, c->err_host, 0), &c->err);
  cudaStream_t st = 0;
  c->states_bound = !defer;
  if (!defer) {
    DC_CUDA_TRY(cudaMemsetAsync(c->m, 0, c->L.shard_elems * 4, st), &c->err);
    DC_CUDA_TRY(cudaMemsetAsync(c->v, 0, c->L.shard_elems * 4, st), &c->err);
  }
  DC_CUDA_TRY(cudaMemsetAsync(reinterpret_cast<void*>(c->grad_peers[c->rank]), 0, 2 * c->L.grad_slot_bytes, st), &c->err);
  DC_CUDA_TRY(cudaMemsetAsync(c->myflag(0), 0, c->L.flag_words * 4, st), &c->err);
  if (a->flags & DC_INIT_WEIGHTS) {
    for (int i = 0; i < a->n_params; ++i) {
      const float k = a->init_k ? a->init_k[i] : 0.0f;
      k_init_param(a->seed, i, c->numel[i], c->world, c->rank, c->L.S[i], k, c->master + c->L.store_off[i],
                   reinterpret_cast<uint16_t*>(c->shard) + c->L.store_off[i], st);
    }
  }
  DC_CUDA_TRY(cudaStreamSynchronize(st), &c->err);
  DC_CUDA_TRY(cudaGetLastError(), &c->err);
  *out = c.release();
  return DC_OK;
}

extern "C" dc_status dc_destroy(dc_ctx* c) {
  if (!c) return DC_OK;
  for (auto& f : c->frags) { cudaEventDestroy(f.d2h); cudaEventDestroy(f.h2d); }
  if (c->err_host) cudaFreeHost(c->err_host);
  delete c;
  return DC_OK;
}

extern "C" dc_status dc_poll(dc_ctx* c) {
  if (!c) return fail(nullptr, DC_EINVAL, "dc_poll: null ctx");
  return check_sticky(c);
}

extern "C" dc_status dc_shard_range(const dc_ctx* c, int32_t p, int64_t* off, int64_t* S) {
  if (!c || p < 0 || p >= c->n_params) { set_global_error("dc_shard_range: bad param"); return DC_EINVAL; }
  if (off) *off = c->L.store_off[p];
  if (S) *S = c->L.S[p];
  return DC_OK;
}

extern "C" dc_status dc_grad_offset(const dc_ctx* c, int32_t p, int64_t* b) {
  if (!c || p < 0 || p >= c->n_params) { set_global_error("dc_grad_offset: bad param"); return DC_EINVAL; }
  *b = c->L.goff[p];
  return DC_OK;
}

// ------------------------------------------------------------------ schedule
extern "C" dc_status dc_bind_schedule(dc_ctx* c, const dc_schedule* s, const uint64_t* arena_peer_ptrs,
                                      uint64_t arena_bytes, cudaStream_t st) {
  if (!c || !s) return fail(c, DC_EINVAL, "dc_bind_schedule: null argument");
  const int n = sched_num_ops(s);
  c->op_index.clear();
  c->initial_ready.clear();
  c->ag_ctas.clear();
  c->ag_launches.clear();
  c->ag_inst.clear();
  c->ag_ninst = 1;
  std::vector<uint32_t> inst_cnt(c->n_params, 0);
  for (int i = 0; i < n; ++i) {
    int kind, id, nm, np, nw;
    const int64_t* mem; const int* posts; const int* waits;
    int64_t off, bytes;
    sched_op(s, i, &kind, &id, &mem, &nm, &off, &bytes, &posts, &np, &waits, &nw);
    if (kind == K_AG)
      for (int j = 0; j < nm; ++j)
        if (mem[j] >= 0 && mem[j] < c->n_params) {
          c->ag_inst[id].push_back(++inst_cnt[mem[j]]);
          c->ag_ninst = std::max(c->ag_ninst, inst_cnt[mem[j]]);
        }
    if (kind == K_AG || kind == K_REL) {
      if (id < 0 || id >= c->max_ops) return fail(c, DC_EINVAL, "dc_bind_schedule: op id exceeds max_s0_ops");
      c->op_index[id] = i;
    }
    for (int j = 0; j < nm && (kind == K_AG || kind == K_REL); ++j)
      if (mem[j] < 0 || mem[j] >= c->n_params) return fail(c, DC_EINVAL, "dc_bind_schedule: param out of range");
    if (kind == K_AG) {
      if (c->world > 1 && off + bytes > (int64_t)arena_bytes) return fail(c, DC_EOOM, "dc_bind_schedule: arena too small");
      if (nw == 0) c->initial_ready.push_back(id);
      int64_t shard_bytes = 0;
      for (int j = 0; j < nm; ++j) shard_bytes += c->L.S[mem[j]] * 2;
      int ctas = (int)std::min<int64_t>(c->ag_max_ctas, std::max<int64_t>(1, shard_bytes / (32 * 1024)));
      c->ag_ctas[id] = c->ag_ce ? 1 : ctas;             // done bumps per sender per gather
      c->ag_launches[id] = c->ag_ce ? 1 : (nm + 47) / 48;
    }
  }
  c->sched = s;
  c->arena_peers.assign(arena_peer_ptrs ? arena_peer_ptrs : nullptr, arena_peer_ptrs ? arena_peer_ptrs + c->world : nullptr);
  if (c->world > 1 && (int)c->arena_peers.size() != c->world) return fail(c, DC_EINVAL, "dc_bind_schedule: arena peers");
  c->arena_bytes = arena_bytes;
  c->arena_mc = 0;                      // a new arena: its multicast mapping is bound again
  c->epoch = 0;
  c->fepoch = 0;
  c->slot_use[0] = c->slot_use[1] = 0;
  std::fill(c->layer_use.begin(), c->layer_use.end(), 0);
  c->rs_done_total = 0;
  std::fill(c->cur_off.begin(), c->cur_off.end(), -1);
  DC_CUDA_TRY(cudaMemsetAsync(c->myflag(0), 0, c->L.flag_words * 4, st), &c->err);
  DC_CUDA_TRY(cudaStreamSynchronize(st), &c->err);
  return DC_OK;
}

static PeerFlags peers_at(const dc_ctx* c, int64_t word) {
  PeerFlags f{};
  f.n = c->world;
  for (int q = 0; q < c->world; ++q) f.p[q] = c->flag(q, word);
  return f;
}

extern "C" dc_status dc_step_begin(dc_ctx* c, int32_t epoch, cudaStream_t st) {
  if (!c || !c->sched) return fail(c, DC_ESTATE, "dc_step_begin: no schedule bound");
  if (dc_status e = check_sticky(c)) return e;
  if ((uint32_t)epoch <= c->epoch) return fail(c, DC_EINVAL, "dc_step_begin: epochs must increase");
  c->epoch = (uint32_t)epoch;
  ++c->fepoch;
  if (c->graph_mode) {
    // every step restarts its flag protocol from zero, so one captured step is
    // valid for all (the previous step's streams joined `st`).  N > 1: a
    // two-round barrier on a device step counter brackets the reset — round A:
    // every rank finished the previous step (no post of it still in flight);
    // round B: every rank zeroed its table (no post of this step lands early)
    uint32_t* dep = c->myflag(c->L.f_dep);
    if (c->world > 1) {
      k_inc_dev(dep, st);
      k_post_dev(peers_at(c, c->L.f_bar + c->rank), dep, st);
      k_wait_dev(c->myflag(c->L.f_bar), c->world, dep, c->timeout_ns, c->err_dev, st);
    }
    c->fepoch = 1;
    c->slot_use[0] = c->slot_use[1] = 0;
    std::fill(c->layer_use.begin(), c->layer_use.end(), 0);
    c->rs_done_total = 0;
    DC_CUDA_TRY(cudaMemsetAsync(c->myflag(0), 0, c->L.f_scal * 4, st), &c->err);
    if (c->world > 1) {
      k_post_dev(peers_at(c, c->L.f_bar + c->world + c->rank), dep, st);
      k_wait_dev(c->myflag(c->L.f_bar + c->world), c->world, dep, c->timeout_ns, c->err_dev, st);
    }
  }
  if (c->world == 1) return DC_OK;
  // ready flags for gathers without an in-step predecessor release (D26):
  // ready[g][me] in every rank's table
  for (int g : c->initial_ready) {
    k_post_flags(peers_at(c, c->L.f_ready + (int64_t)g * c->world + c->rank), c->fepoch, st);
  }
  if (cudaGetLastError() != cudaSuccess) return fail(c, DC_ECUDA, "dc_step_begin: launch failed");
  return DC_OK;
}

extern "C" dc_status dc_gather(dc_ctx* c, int32_t gid, cudaStream_t st, cudaEvent_t done_evt) {
  if (!c || !c->sched) return fail(c, DC_ESTATE, "dc_gather: no schedule bound");
  if (dc_status e = check_sticky(c)) return e;
  auto it = c->op_index.find(gid);
  if (it == c->op_index.end()) return fail(c, DC_EINVAL, "dc_gather: unknown gather id");
  int kind, id, nm, np, nw;
  const int64_t* mem; const int* posts; const int* waits;
  int64_t off, bytes;
  sched_op(c->sched, it->second, &kind, &id, &mem, &nm, &off, &bytes, &posts, &np, &waits, &nw);
  if (kind != K_AG) return fail(c, DC_EINVAL, "dc_gather: op is not a gather");
  if (c->world == 1) {
    for (int j = 0; j < nm; ++j) c->cur_off[mem[j]] = -2;   // alias of the shard
  } else {
    if (c->fepoch == 0) return fail(c, DC_ESTATE, "dc_gather: call dc_step_begin first");
    std::vector<AgMember> am;
    int64_t cur = off;
    for (int j = 0; j < nm; ++j) {
      const int p = (int)mem[j];
      AgMember a;
      a.src = reinterpret_cast<const uint16_t*>(c->shard) + c->L.store_off[p];
      a.dst_off_bytes = cur + (int64_t)c->rank * c->L.S[p] * 2;
      a.bytes = c->L.S[p] * 2;
      if (c->fused_ag) {
        a.chunk_word = c->L.f_chunk + ((int64_t)p * c->world + c->rank) * AG_CHUNKS;
        a.chunk_value = (c->fepoch - 1) * c->ag_ninst + c->ag_inst[gid][j];
      }
      am.push_back(a);
      c->cur_off[p] = cur;
      cur += align256(c->numel[p] > 0 ? c->L.S[p] * c->world * 2 : 0);
    }
    const int ctas = c->ag_ctas[gid];
    const uint32_t target = c->fepoch * (uint32_t)(c->world * ctas * c->ag_launches[gid]);
    dc_status s = ((c->nvls & 1) && c->arena_mc && !c->ag_ce)
        ? k_ag_multimem(am, reinterpret_cast<uint8_t*>(c->arena_mc),
                        reinterpret_cast<uint32_t*>(c->flags_mc) + c->L.f_done + gid, ctas,
                        c->myflag(c->L.f_ready + (int64_t)gid * c->world), c->world, c->fepoch,
                        c->myflag(c->L.f_done + gid), target, c->timeout_ns, c->err_dev, st, c->gt_start)
        : c->ag_ce
        ? k_ag_copy(am, c->world, c->arena_peers.data(), c->myflag(c->L.f_ready + (int64_t)gid * c->world), c->fepoch,
                    peers_at(c, c->L.f_done + gid), c->myflag(c->L.f_done + gid), target, c->timeout_ns, c->err_dev,
                    st, c->gt_start)
        : k_ag_push(am, c->world, c->rank, c->arena_peers.data(), c->myflag(c->L.f_ready + (int64_t)gid * c->world),
                    c->fepoch, peers_at(c, c->L.f_done + gid), c->myflag(c->L.f_done + gid), target, ctas,
                    c->timeout_ns, c->err_dev, st, c->gt_start, c->ag_skip_waits != 0,
                    c->ag_delay_us + c->jitter(gid), c->flag_peers.data(), c->ag_bulk != 0);
    if (s != DC_OK) return fail(c, s, "dc_gather: launch failed");
    if (c->gt_end) record_event(c->gt_end, st);
  }
  c->gt_start = c->gt_end = nullptr;
  if (done_evt) DC_CUDA_TRY(cudaEventRecord(done_evt, st), &c->err);
  return DC_OK;
}

extern "C" dc_status dc_gather_timing(dc_ctx* c, cudaEvent_t after_ready, cudaEvent_t after_done) {
  if (!c) return fail(c, DC_EINVAL, "dc_gather_timing: null ctx");
  c->gt_start = after_ready;
  c->gt_end = after_done;
  return DC_OK;
}

extern "C" dc_status dc_set_option(dc_ctx* c, const char* key, int64_t value) {
  if (!c || !key) return fail(c, DC_EINVAL, "dc_set_option: null argument");
  if (!strcmp(key, "graph_mode")) {
    if (c->sched) return fail(c, DC_ESTATE, "dc_set_option: graph_mode must be set before dc_bind_schedule");
    c->graph_mode = value != 0;
    return DC_OK;
  }
  if (!strcmp(key, "ag_skip_waits")) {
    // profiling only (ncu serialises kernels, so a flag wait on another rank's
    // kernel would never return): the push runs without its ready / done
    // waits — the caller guarantees the receivers' buffers are free and reads
    // nothing it gathered this way
    c->ag_skip_waits = value != 0;
    return DC_OK;
  }
  if (!strcmp(key, "rs_bulk")) {   // may change between steps (the launch reads it)
    c->rs_bulk = value != 0;
    return DC_OK;
  }
  if (!strcmp(key, "ag_bulk")) {   // any time (read at each dc_gather)
    c->ag_bulk = value != 0;
    return DC_OK;
  }
  if (!strcmp(key, "fused_ag")) {   // chunked pushes + per-tile GEMM waits (dc_model_step), SURVEY §8 f-4
    if (c->sched) return fail(c, DC_ESTATE, "dc_set_option: fused_ag must be set before dc_bind_schedule");
    c->fused_ag = value != 0;
    return DC_OK;
  }
  if (!strcmp(key, "ag_delay_us")) {   // testing: start every push this long after its ready wait
    if (value < 0 || value > 1000000) return fail(c, DC_EINVAL, "dc_set_option: ag_delay_us in [0, 1e6]");
    c->ag_delay_us = (uint32_t)value;
    return DC_OK;
  }
  if (!strcmp(key, "jitter_us")) {   // testing: random delays (value = max us; the seed is set by "jitter_seed")
    if (value < 0 || value > 1000000) return fail(c, DC_EINVAL, "dc_set_option: jitter_us in [0, 1e6]");
    c->jitter_us = (uint32_t)value;
    return DC_OK;
  }
  if (!strcmp(key, "jitter_seed")) {
    c->jitter_seed = (uint32_t)value;
    return DC_OK;
  }
  if (!strcmp(key, "nvls")) {   // bit 0: multimem gathers, bit 1: multimem.ld_reduce reduce-scatter
    if (value < 0 || value > 3) return fail(c, DC_EINVAL, "dc_set_option: nvls in [0, 3]");
    c->nvls = (int)value;
    return DC_OK;
  }
  if (!strcmp(key, "ag_copy_engine")) {
    if (c->sched) return fail(c, DC_ESTATE, "dc_set_option: ag_copy_engine must be set before dc_bind_schedule");
    c->ag_ce = value != 0;
    return DC_OK;
  }
  return fail(c, DC_EINVAL, std::string("dc_set_option: unknown key ") + key);
}

extern "C" dc_status dc_bind_multicast(dc_ctx* c, uint64_t arena_mc, uint64_t grad_mc, uint64_t flags_mc) {
  if (!c) return fail(c, DC_EINVAL, "dc_bind_multicast: null ctx");
  if (!c->sched) return fail(c, DC_ESTATE, "dc_bind_multicast: bind a schedule (and its arena) first");
  if ((arena_mc || grad_mc || flags_mc) && (c->world < 2 || (c->flags & DC_VIRTUAL_RANKS)))
    return fail(c, DC_EINVAL, "dc_bind_multicast: multicast needs N > 1 ranks on N GPUs (not virtual ranks)");
  if ((arena_mc || grad_mc) && !flags_mc)
    return fail(c, DC_EINVAL, "dc_bind_multicast: the flag table's multicast address is required");
  if ((arena_mc | grad_mc | flags_mc) & 15) return fail(c, DC_EINVAL, "dc_bind_multicast: addresses must be 16 B aligned");
  c->arena_mc = arena_mc;
  c->grad_mc = grad_mc;
  c->flags_mc = flags_mc;
  return DC_OK;
}

extern "C" dc_status dc_tensor_ptr(const dc_ctx* c, int32_t p, void** ptr) {
  if (!c || p < 0 || p >= c->n_params || !ptr) { set_global_error("dc_tensor_ptr: bad param"); return DC_EINVAL; }
  if (c->world == 1) {
    *ptr = reinterpret_cast<uint16_t*>(c->shard) + c->L.store_off[p];
    return DC_OK;
  }
  if (c->cur_off[p] < 0) { set_global_error("dc_tensor_ptr: param is not gathered"); return DC_ESTATE; }
  *ptr = reinterpret_cast<uint8_t*>(c->arena_peers[c->rank]) + c->cur_off[p];
  return DC_OK;
}

extern "C" dc_status dc_release(dc_ctx* c, int32_t rid, cudaStream_t st) {
  if (!c || !c->sched) return fail(c, DC_ESTATE, "dc_release: no schedule bound");
  auto it = c->op_index.find(rid);
  if (it == c->op_index.end()) return fail(c, DC_EINVAL, "dc_release: unknown release id");
  int kind, id, nm, np, nw;
  const int64_t* mem; const int* posts; const int* waits;
  int64_t off, bytes;
  sched_op(c->sched, it->second, &kind, &id, &mem, &nm, &off, &bytes, &posts, &np, &waits, &nw);
  if (kind != K_REL) return fail(c, DC_EINVAL, "dc_release: op is not a release");
  if (c->world > 1 && (c->flags & DC_DEBUG_POISON) && c->cur_off[mem[0]] >= 0)   // stale reads become NaN
    DC_CUDA_TRY(cudaMemsetAsync(reinterpret_cast<uint8_t*>(c->arena_peers[c->rank]) + c->cur_off[mem[0]], 0xFF,
                                c->L.S[mem[0]] * c->world * 2, st), &c->err);
  if (c->world > 1) c->cur_off[mem[0]] = -1;
  if (c->world == 1) return DC_OK;
  k_delay(c->jitter(rid + 0x40000), st);
  for (int j = 0; j < np; ++j)
    k_post_flags(peers_at(c, c->L.f_ready + (int64_t)posts[j] * c->world + c->rank), c->fepoch, st);
  if (cudaGetLastError() != cudaSuccess) return fail(c, DC_ECUDA, "dc_release: launch failed");
  return DC_OK;
}

// ------------------------------------------------------------------ grads
extern "C" dc_status dc_grad_slot(const dc_ctx* c, int32_t layer, void** p) {
  if (!c || layer < 0 || layer >= c->L.n_layers || !p) { set_global_error("dc_grad_slot: bad layer"); return DC_EINVAL; }
  *p = c->slot_ptr(c->rank, layer & 1);
  return DC_OK;
}

extern "C" dc_status dc_grad_slot_acquire(dc_ctx* c, int32_t layer, cudaStream_t st) {
  if (!c || layer < 0 || layer >= c->L.n_layers) return fail(c, DC_EINVAL, "dc_grad_slot_acquire: bad layer");
  if (dc_status e = check_sticky(c)) return e;
  const int s = layer & 1;
  const int u = ++c->slot_use[s];
  c->layer_use[layer] = u;
  if (u > 1)   // every owner consumed the previous use of this slot
    k_wait_flags(c->myflag(c->L.f_gcons + (int64_t)s * c->world), c->world, (uint32_t)(u - 1), c->timeout_ns,
                 c->err_dev, st);
  return DC_OK;
}

extern "C" dc_status dc_grad_slot_publish(dc_ctx* c, int32_t layer, cudaStream_t st) {
  if (!c || layer < 0 || layer >= c->L.n_layers) return fail(c, DC_EINVAL, "dc_grad_slot_publish: bad layer");
  const int s = layer & 1;
  k_post_flags(peers_at(c, c->L.f_gready + (int64_t)s * c->world + c->rank), (uint32_t)c->layer_use[layer], st);
  return DC_OK;
}

namespace dc {
void ctx_adam_scalars(const dc_ctx* c, int step_t, EpiAdam* o) {
  const double bc1 = 1.0 - std::pow(c->beta1, step_t);
  const double bc2 = 1.0 - std::pow(c->beta2, step_t);
  o->w1 = (float)(1.0 - c->beta1);
  o->w2 = (float)(1.0 - c->beta2);
  o->b2 = (float)c->beta2;
  o->neg_s = -(float)(c->lr / bc1);
  o->c = (float)std::sqrt(bc2);
  o->eps = (float)c->eps;
}

bool ctx_fused_ag(const dc_ctx* c) { return c->fused_ag && c->world > 1 && !c->ag_ce && !(c->nvls & 1); }
bool ctx_virtual(const dc_ctx* c) { return (c->flags & DC_VIRTUAL_RANKS) != 0; }
void ctx_wait_err(dc_ctx* c, uint32_t** err, uint64_t* timeout_ns) {
  *err = c->err_dev;
  *timeout_ns = c->timeout_ns;
}
bool ctx_chunk_wait(const dc_ctx* c, int gid, int param, ChunkWait* out) {
  auto it = c->op_index.find(gid);
  auto in = c->ag_inst.find(gid);
  if (it == c->op_index.end() || in == c->ag_inst.end()) return false;
  int kind, id, nm, np, nw;
  const int64_t* mem; const int* posts; const int* waits;
  int64_t off, bytes;
  sched_op(c->sched, it->second, &kind, &id, &mem, &nm, &off, &bytes, &posts, &np, &waits, &nw);
  for (int j = 0; j < nm; ++j)
    if (mem[j] == param) {
      out->flags = c->myflag(c->L.f_chunk + (int64_t)param * c->world * AG_CHUNKS);
      out->S = c->L.S[param];
      out->E = ag_chunk_elems(out->S);
      out->value = (c->fepoch - 1) * c->ag_ninst + in->second[j];
      return true;
    }
  return false;
}

void ctx_param_state(const dc_ctx* c, int p, float** master, float** m, float** v, void** shard) {
  const int64_t o = c->L.store_off[p];
  *master = c->master + o;
  *m = c->m + o;
  *v = c->v + o;
  *shard = reinterpret_cast<uint16_t*>(c->shard) + o;
}

dc_status ctx_side_job(dc_ctx* c, int layer, int step_t, SideJob* o) {
  if (c->world != 1) return fail(c, DC_EINVAL, "side job: N == 1 only");
  if (c->layer_use[layer] == 0) return fail(c, DC_ESTATE, "side job: grad slot of layer never acquired");
  const int first = c->L.layer_first[layer], n = c->L.layer_count[layer];
  if (n > 9) return fail(c, DC_EINVAL, "side job: at most 9 params per layer");
  *o = SideJob{};
  o->nm = n;
  o->cum[0] = 0;
  for (int i = 0; i < n; ++i) {
    o->goff[i] = c->L.goff[first + i];
    o->store_off[i] = c->L.store_off[first + i];
    o->cum[i + 1] = o->cum[i] + c->L.S[first + i] / 8;
  }
  o->slot = c->slot_ptr(c->rank, layer & 1);
  o->master = c->master;
  o->m = c->m;
  o->v = c->v;
  o->shard = reinterpret_cast<__nv_bfloat16*>(c->shard);
  EpiAdam a{};
  ctx_adam_scalars(c, step_t, &a);
  o->w1 = a.w1; o->w2 = a.w2; o->b2 = a.b2; o->neg_s = a.neg_s; o->c = a.c; o->eps = a.eps;
  o->g0 = 0;
  o->g1 = o->cum[n];
  return DC_OK;
}

dc_status ctx_post_consumed(dc_ctx* c, int layer, cudaStream_t st) {
  const int s = layer & 1;
  k_post_flags(peers_at(c, c->L.f_gcons + (int64_t)s * c->world + c->rank), (uint32_t)c->layer_use[layer], st);
  return cudaGetLastError() == cudaSuccess ? DC_OK : fail(c, DC_ECUDA, "post consumed: launch failed");
}

dc_status reduce_scatter_params(dc_ctx* c, int layer, int step_t, int micro, const std::vector<int>& params,
                                cudaStream_t st) {
  if (dc_status e = check_sticky(c)) return e;
  if (micro < 0 || micro >= c->micro_steps) return fail(c, DC_EINVAL, "dc_reduce_scatter_step: micro out of range");
  const int n = c->micro_steps;
  const int mode = n == 1 ? RS_UPDATE : micro == 0 ? RS_FIRST : micro < n - 1 ? RS_ADD : RS_FINAL;
  const int s = layer & 1;
  const int u = c->layer_use[layer];
  if (u == 0) return fail(c, DC_ESTATE, "dc_reduce_scatter_step: grad slot of layer never acquired");
  if (!c->states_bound) return fail(c, DC_ESTATE, "dc_reduce_scatter_step: optimizer states not bound (DC_DEFER_STATES)");
  // host-resident fragments are updated in their ring slot (base shifted so
  // that base + store_off lands at the slot)
  float* mb = (c->host_states && c->lay_m[layer]) ? c->lay_m[layer] : c->m;
  float* vb = (c->host_states && c->lay_v[layer]) ? c->lay_v[layer] : c->v;
  std::vector<RsMember> mem;
  int64_t elems = 0;
  for (int i : params) {
    mem.push_back({c->L.goff[i], c->L.S[i], c->L.store_off[i]});
    elems += c->L.S[i];
  }
  std::vector<uint64_t> slots(c->world);
  for (int q = 0; q < c->world; ++q) slots[q] = reinterpret_cast<uint64_t>(c->slot_ptr(q, s));
  const double bc1 = 1.0 - std::pow(c->beta1, step_t);
  const double bc2 = 1.0 - std::pow(c->beta2, step_t);
  const float sc = (float)(c->lr / bc1);
  const float cc = (float)std::sqrt(bc2);
  const bool bulk = c->rs_bulk && (mode == RS_UPDATE || mode == RS_FINAL);
  int ctas = (int)std::min<int64_t>(c->rs_ctas, std::max<int64_t>(1, elems / 8 / c->rs_threads));
  if (bulk) {   // a fixed number of CTAs per SM (or one per chunk, if fewer)
    int64_t chunks = 0;
    for (int i : params) chunks += (c->L.S[i] + RS_BULK_CHUNK - 1) / RS_BULK_CHUNK;
    ctas = (int)std::min<int64_t>((int64_t)c->num_sms * rs_bulk_ctas_per_sm(), std::max<int64_t>(1, chunks));
  }
  c->rs_done_total += (uint32_t)ctas;
  k_delay(c->jitter(layer + 0x80000), st);
  if ((c->nvls & 2) && c->grad_mc) {      // f-3: the switch sums the slices (not bit-exact, opt-in)
    dc_status r = k_rs_adam_nvls(mem, c->world, c->rank,
                                 reinterpret_cast<const uint8_t*>(c->grad_mc) + (int64_t)s * c->L.grad_slot_bytes,
                                 c->myflag(c->L.f_gready + (int64_t)s * c->world), (uint32_t)u,
                                 peers_at(c, c->L.f_gcons + (int64_t)s * c->world + c->rank), (uint32_t)u,
                                 c->myflag(c->L.f_rsdone), c->rs_done_total, c->master, mb, vb, c->shard, c->grad_acc,
                                 mode, n, sc, cc, c->beta1, c->beta2, c->eps, ctas, c->timeout_ns, c->err_dev, st,
                                 c->graph_mode ? reinterpret_cast<const float*>(c->myflag(c->L.f_scal)) : nullptr);
    return r == DC_OK ? DC_OK : fail(c, r, "dc_reduce_scatter_step: NVLS launch failed");
  }
  dc_status r = k_rs_adam(mem, c->world, c->rank, slots.data(), c->myflag(c->L.f_gready + (int64_t)s * c->world),
                          (uint32_t)u, peers_at(c, c->L.f_gcons + (int64_t)s * c->world + c->rank), (uint32_t)u,
                          c->myflag(c->L.f_rsdone), c->rs_done_total, c->master, mb, vb, c->shard, c->grad_acc,
                          mode, n, sc, cc,
                          c->beta1, c->beta2, c->eps, ctas, c->rs_threads, c->timeout_ns, c->err_dev, st,
                          c->graph_mode ? reinterpret_cast<const float*>(c->myflag(c->L.f_scal)) : nullptr, bulk);
  if (r != DC_OK) return fail(c, r, "dc_reduce_scatter_step: launch failed");
  return DC_OK;
}
}  // namespace dc

extern "C" dc_status dc_reduce_scatter_step(dc_ctx* c, int32_t layer, int32_t step_t, int32_t micro,
                                            cudaStream_t st) {
  if (!c || layer < 0 || layer >= c->L.n_layers) return fail(c, DC_EINVAL, "dc_reduce_scatter_step: bad layer");
  if (step_t < 1) return fail(c, DC_EINVAL, "dc_reduce_scatter_step: step_t is 1-based");
  std::vector<int> params;
  for (int i = c->L.layer_first[layer]; i < c->L.layer_first[layer] + c->L.layer_count[layer]; ++i) params.push_back(i);
  return reduce_scatter_params(c, layer, step_t, micro, params, st);
}

// ------------------------------------------------------------------ offload
extern "C" dc_status dc_offload_fragments(dc_ctx* c, int64_t max_bytes, dc_fragment* out, int32_t* n_inout) {
  if (!c || !n_inout || max_bytes < 32) return fail(c, DC_EINVAL, "dc_offload_fragments: bad argument");
  for (auto& f : c->frags) { cudaEventDestroy(f.d2h); cudaEventDestroy(f.h2d); }
  c->frags.clear();
  const int64_t chunk = max_bytes / 4 / 8 * 8;
  int64_t host_off = 0;
  for (int l = 0; l < c->L.n_layers; ++l) {
    const int first = c->L.layer_first[l];
    const int64_t lo = c->L.store_off[first];
    const int64_t hi = lo + [&] { int64_t e = 0; for (int i = first; i < first + c->L.layer_count[l]; ++i) e += c->L.S[i]; return e; }();
    for (int st = 0; st < 2; ++st)
      for (int64_t o = lo; o < hi; o += chunk) {
        FragInfo f{};
        f.layer = l; f.state = st; f.off = o; f.elems = std::min(chunk, hi - o); f.host_off = host_off;
        host_off += f.elems * 4;
        c->frags.push_back(f);
      }
  }
  const int n = (int)c->frags.size();
  for (auto& f : c->frags) {
    DC_CUDA_TRY(cudaEventCreateWithFlags(&f.d2h, cudaEventDisableTiming), &c->err);
    DC_CUDA_TRY(cudaEventCreateWithFlags(&f.h2d, cudaEventDisableTiming), &c->err);
  }
  if (out) {
    if (*n_inout < n) { *n_inout = n; return fail(c, DC_EOOM, "dc_offload_fragments: output array too small"); }
    for (int i = 0; i < n; ++i) out[i] = {c->frags[i].layer, c->frags[i].state, c->frags[i].off, c->frags[i].elems};
  }
  *n_inout = n;
  return DC_OK;
}

extern "C" dc_status dc_offload(dc_ctx* c, int32_t fi, int32_t op, cudaStream_t st) {
  if (!c || fi < 0 || fi >= (int)c->frags.size()) return fail(c, DC_EINVAL, "dc_offload: bad fragment");
  FragInfo& f = c->frags[fi];
  if ((uint64_t)(f.host_off + f.elems * 4) > c->host_pinned_bytes || !c->host_pinned)
    return fail(c, DC_EOOM, "dc_offload: pinned host buffer too small");
  char* host = reinterpret_cast<char*>(c->host_pinned) + f.host_off;
  if (c->host_states && f.slot) {   // reading D28: the host copy is authoritative
    switch (op) {
      case DC_D2H_START:
      case DC_D2H_SYNC_FREE:
        return DC_OK;                 // already written back after the last update
      case DC_H2D_START:
        DC_CUDA_TRY(cudaMemcpyAsync(f.slot, host, f.elems * 4, cudaMemcpyHostToDevice, st), &c->err);
        DC_CUDA_TRY(cudaEventRecord(f.h2d, st), &c->err);
        return DC_OK;
      case DC_H2D_SYNC:
        DC_CUDA_TRY(cudaStreamWaitEvent(st, f.h2d, 0), &c->err);
        return DC_OK;
      case DC_WRITEBACK:
        DC_CUDA_TRY(cudaMemcpyAsync(host, f.slot, f.elems * 4, cudaMemcpyDeviceToHost, st), &c->err);
        return DC_OK;
      default:
        return fail(c, DC_EINVAL, "dc_offload: bad op");
    }
  }
  if (op == DC_WRITEBACK) return fail(c, DC_ESTATE, "dc_offload: DC_WRITEBACK needs host-resident states");
  if (!c->states_bound) return fail(c, DC_ESTATE, "dc_offload: optimizer states not bound");
  float* dev = (f.state == 0 ? c->m : c->v) + f.off;
  switch (op) {
    case DC_D2H_START:
      DC_CUDA_TRY(cudaMemcpyAsync(host, dev, f.elems * 4, cudaMemcpyDeviceToHost, st), &c->err);
      DC_CUDA_TRY(cudaEventRecord(f.d2h, st), &c->err);
      break;
    case DC_D2H_SYNC_FREE:
      DC_CUDA_TRY(cudaStreamWaitEvent(st, f.d2h, 0), &c->err);
      // debug: the device slice is "freed" — poison it (all-ones = NaN) so a
      // missing or misordered reload corrupts the update instead of passing
      if (c->flags & DC_DEBUG_POISON)
        DC_CUDA_TRY(cudaMemsetAsync(dev, 0xFF, f.elems * 4, st), &c->err);
      break;
    case DC_H2D_START:
      DC_CUDA_TRY(cudaMemcpyAsync(dev, host, f.elems * 4, cudaMemcpyHostToDevice, st), &c->err);
      DC_CUDA_TRY(cudaEventRecord(f.h2d, st), &c->err);
      break;
    case DC_H2D_SYNC:
      DC_CUDA_TRY(cudaStreamWaitEvent(st, f.h2d, 0), &c->err);
      break;
    default:
      return fail(c, DC_EINVAL, "dc_offload: bad op");
  }
  return DC_OK;
}

// internal accessors for model.cu
namespace dc {
int ctx_num_frags(const dc_ctx* c) { return (int)c->frags.size(); }
bool ctx_graph_mode(const dc_ctx* c) { return c->graph_mode; }
dc_status ctx_set_step_scalars(dc_ctx* c, int step_t, cudaStream_t st) {
  // the same host arithmetic as reduce_scatter_params (reading D18)
  const double bc1 = 1.0 - std::pow(c->beta1, step_t);
  const double bc2 = 1.0 - std::pow(c->beta2, step_t);
  k_set_scalars(reinterpret_cast<float*>(c->myflag(c->L.f_scal)), (float)(c->lr / bc1), (float)std::sqrt(bc2), st);
  return cudaGetLastError() == cudaSuccess ? DC_OK : fail(c, DC_ECUDA, "set step scalars: launch failed");
}
void ctx_set_gather_timing(dc_ctx* c, cudaEvent_t start, cudaEvent_t end) { c->gt_start = start; c->gt_end = end; }
void ctx_frag(const dc_ctx* c, int i, int* layer, int* state, int64_t* off, int64_t* elems) {
  const FragInfo& f = c->frags[i];
  *layer = f.layer; *state = f.state; *off = f.off; *elems = f.elems;
}
uint64_t ctx_frag_host_end(const dc_ctx* c, int i) { return (uint64_t)(c->frags[i].host_off + c->frags[i].elems * 4); }
dc_status ctx_bind_host_states(dc_ctx* c, float* m_dev, int64_t m_first, float* v_dev, int64_t v_first,
                               const std::vector<float*>& frag_slot, void* host_pinned, uint64_t host_bytes) {
  if (frag_slot.size() != c->frags.size()) return fail(c, DC_EINVAL, "host states: fragment table changed");
  if (host_pinned) {
    c->host_pinned = host_pinned;
    c->host_pinned_bytes = host_bytes;
  }
  if (!c->host_pinned) return fail(c, DC_EINVAL, "host states: no pinned host buffer (dc_init_args.host_pinned)");
  const int64_t E = c->L.shard_elems;
  // base pointers: element i of m lives at m_dev[i - m_first] (never read below m_first)
  c->m = reinterpret_cast<float*>(reinterpret_cast<uintptr_t>(m_dev) - (uintptr_t)(m_first * 4));
  c->v = reinterpret_cast<float*>(reinterpret_cast<uintptr_t>(v_dev) - (uintptr_t)(v_first * 4));
  c->lay_m.assign(c->L.n_layers, nullptr);
  c->lay_v.assign(c->L.n_layers, nullptr);
  c->host_states = false;
  for (size_t i = 0; i < c->frags.size(); ++i) {
    FragInfo& f = c->frags[i];
    f.slot = frag_slot[i];
    if (!f.slot) continue;
    c->host_states = true;
    float* base = reinterpret_cast<float*>(reinterpret_cast<uintptr_t>(f.slot) - (uintptr_t)(f.off * 4));
    (f.state == 0 ? c->lay_m : c->lay_v)[f.layer] = base;
    if ((uint64_t)(f.host_off + f.elems * 4) > c->host_pinned_bytes)
      return fail(c, DC_EOOM, "host states: pinned host buffer too small");
    memset(reinterpret_cast<char*>(c->host_pinned) + f.host_off, 0, f.elems * 4);   // states start at zero
  }
  if (m_first < E) DC_CUDA_TRY(cudaMemset(m_dev, 0, (E - m_first) * 4), &c->err);
  if (v_first < E) DC_CUDA_TRY(cudaMemset(v_dev, 0, (E - v_first) * 4), &c->err);
  DC_CUDA_TRY(cudaDeviceSynchronize(), &c->err);
  c->states_bound = true;
  return DC_OK;
}
const Layout& ctx_layout(const dc_ctx* c) { return c->L; }
int ctx_world(const dc_ctx* c) { return c->world; }
int ctx_rank(const dc_ctx* c) { return c->rank; }
const dc_schedule* ctx_sched(const dc_ctx* c) { return c->sched; }
int64_t ctx_numel(const dc_ctx* c, int p) { return c->numel[p]; }
int ctx_micro_steps(const dc_ctx* c) { return c->micro_steps; }
uint32_t ctx_flags(const dc_ctx* c) { return c->flags; }
void ctx_set_rs_ctas(dc_ctx* c, int ctas) {
  c->rs_ctas = ctas > 0 ? ctas : c->rs_ctas_default;
  if (const char* e = getenv("DC_RS_CTAS")) c->rs_ctas = std::max(1, atoi(e));
}
}  // namespace dc
