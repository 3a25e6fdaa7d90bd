// The synthetic Llama-shaped layer stack and the native step executor.
//
// The executor walks the bound schedule (S_0 or the planned S) and issues, per
// op: gathers on the AG stream (ordered after the compute-stream position of
// the op — reading D23), releases and layer compute on the compute stream,
// reduce-scatter + Adam on the RS stream, offload copies on the copy stream.
// With profiling on it records per-op CUDA-event durations and the analytic
// resident-memory profile P_mem(o) for dc_plan.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "dc_internal.h"

using namespace dc;

namespace {

enum OpCode {
  F_ATTN_NORM, F_QKV, F_ATTN_MIX, F_O, F_MLP_NORM, F_GATE_UP, F_ACT, F_DOWN, F_LOSS,
  B_DOWN, B_ACT, B_GATE_UP, B_MLP_NORM, B_O, B_ATTN_MIX, B_QKV, B_ATTN_NORM, RS_OP,
  // Mixtral-shaped MoE MLP (per-expert ops carry the expert index)
  F_ROUTER, F_MOE_GATHER, F_EXP_GU, F_EXP_ACT, F_EXP_DOWN, F_MOE_COMBINE,
  B_MOE_COMBINE, B_EXP_DOWN, B_EXP_ACT, B_EXP_GU, B_ROUTER
};
const char* op_name(int c) {
  static const char* n[] = {"attn_norm", "qkv", "attn_mix", "o_proj", "mlp_norm", "gate_up", "act", "down", "loss",
                            "down_bwd", "act_bwd", "gate_up_bwd", "mlp_norm_bwd", "o_bwd", "attn_mix_bwd",
                            "qkv_bwd", "attn_norm_bwd", "rs",
                            "router", "moe_gather", "exp_gu", "exp_act", "exp_down", "moe_combine",
                            "moe_combine_bwd", "exp_down_bwd", "exp_act_bwd", "exp_gu_bwd", "router_bwd"};
  return n[c];
}
// param slots inside a layer (llama order of synth/models.py)
enum { P_G1, P_Q, P_K, P_V, P_O, P_G2, P_GATE, P_UP, P_DOWN, P_N };
// MoE layer (synth/models.py moe_names): attention slots, router, then
// per expert e: w1 (gate) 7 + 3e, w3 (up) 8 + 3e, w2 (down) 9 + 3e
enum { P_ROUTER = 6, P_EXP0 = 7 };
inline int p_w1(int e) { return P_EXP0 + 3 * e; }
inline int p_w3(int e) { return P_EXP0 + 3 * e + 1; }
inline int p_w2(int e) { return P_EXP0 + 3 * e + 2; }

struct S0 {
  int kind;       // K_COMPUTE / K_AG / K_REL / K_RS
  int code;       // OpCode for compute-like ops
  bool fwd;
  int micro, layer;
  std::vector<int> params;
  bool re = false;  // forward op re-run in the backward (activation checkpointing)
  int e = -1;       // expert of a per-expert MoE op
};

// ops whose every param is read only as a GEMM B operand (their gathers may be
// consumed chunk by chunk: fused all-gather -> GEMM); norm gains and the router
// are read by other kernels and always wait for the whole gather
static bool gemm_b_op(int code) {
  switch (code) {
    case F_QKV: case B_QKV: case F_O: case B_O: case F_GATE_UP: case B_GATE_UP: case F_DOWN: case B_DOWN:
    case F_EXP_GU: case B_EXP_GU: case F_EXP_DOWN: case B_EXP_DOWN:
      return true;
    default:
      return false;
  }
}

std::string op_label(const S0& o) {
  std::string s = (o.re ? "re_" : "") + std::string(op_name(o.code));
  if (o.e >= 0) s += "_" + std::to_string(o.e);
  return s;
}

// MoE: gu / act / X / O hold all experts' rows, expert-major ([E][R][.])
struct LayerAct { int64_t h1, rstd1, qkv, a, x2, h2, rstd2, gu, act, y, g01, X, O; };

}  // namespace

struct dc_model {
  dc_ctx* ctx = nullptr;
  dc_model_dims d{};
  int qd = 0, kvd = 0, qkvd = 0, grp = 0;
  std::vector<S0> s0;
  std::vector<LayerAct> la;
  int64_t ws_dA = 0, ws_dB = 0, ws_dact = 0, ws_dgu = 0, ws_dh = 0, ws_dx2 = 0, ws_dqkv = 0, ws_dgp = 0,
          ws_lossp = 0, ws_loss = 0;
  int64_t ws_dO = 0, ws_dX = 0, ws_dl0 = 0, ws_rgp = 0;   // MoE backward
  int64_t ws_sk = 0;                                     // stream-K workspace of the compute-stream GEMMs
  int E = 0, R = 0;                                      // experts, rows per expert (2T/E)
  uint64_t act_bytes = 0, layer_act_bytes = 0, ws_bytes = 0;
  uint8_t* act = nullptr;
  const void* x = nullptr;
  const void* target = nullptr;
  std::vector<cudaEvent_t> ev_pos, ev_done, ev_t0, ev_t1;
  cudaEvent_t ev_join[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  std::vector<int64_t> dur_us;       // per S_0 op
  std::vector<int64_t> p_mem;        // per S_0 op
  int32_t epoch = 0;
  int64_t launches = 0;
  int cur_d = 0;                     // which of dA/dB holds dL/d(layer output)
  bool profile_pending = false;      // per-op events recorded, not yet read
  bool fused_adam = false;           // N = 1: Adam in the dW GEMM epilogues (option)
  bool fused_active = false;         // ... and the bound schedule has no offload
  bool side_adam = false;            // N = 1: RS + Adam as GEMM side jobs (option)
  bool side_active = false;
  int pending_layer = -1;            // layer whose RS + Adam rides on the current GEMMs
  SideJob pending{};
  int64_t pending_assigned = 0;      // groups handed out so far
  __int128 pending_mnk = 0;          // sum of M*N*K of the hosting GEMMs so far
  int64_t bwd_mnk = 0;               // sum of M*N*K of one layer's backward GEMMs
  int step_t = 0;
  int n_micro = 1;                   // gradient-accumulation micro-steps (ctx)
  int stream_k = 1;                  // stream-K GEMM tails (off when ranks share a GPU)
  int rs_overlap = 1;                // RS + Adam on its own stream
  int comm_sms = 0;                  // > 0: SM partition (GEMMs | comm + Adam), green contexts
  SmPartition part{};
  int gemm_sms = 0;                  // SMs the layer GEMMs may use (0 = all)
  // fused all-gather -> GEMM (ctx option fused_ag): the current
  // op's B operands whose gathers the GEMM waits for per chunk (instead of the
  // compute stream waiting for the whole gather)
  std::vector<std::pair<const void*, ChunkWait>> cw;
  bool fused_ag = false;
  // backward: the dW GEMMs of an op run on a second stream beside its dX GEMM,
  // so their tiles fill the dX GEMM's last partial wave (option dw_concurrent)
  int dw_conc = 1;
  // CUDA graph of one step (graph mode, N = 1): captured by
  // dc_model_graph_capture, replayed by dc_model_graph_launch
  bool capturing = false;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  cudaStream_t cs2 = nullptr;
  bool cs2_own = true;                // false: the caller's (option "dw_stream")
  cudaEvent_t ev_fork = nullptr, ev_joinw = nullptr;
  int fuse_act = 0;                  // bit 0: SiLU*up in the gate|up GEMM epilogue; bit 1: its backward
                                     // in the down dX epilogue.  Bit-identical; measured no faster in
                                     // the power-capped N = 1 step (profiles/r01g/fuse_act_ab.md): off
  // host-resident optimizer states (reading D28): fragments written back after RS(layer)
  bool host_states = false;
  // the paper's comparison point for adaptive offload: every
  // optimizer-state fragment host-resident, reloaded synchronously right before
  // its layer's update (the compute stream waits too), whatever the plan says
  int offload_all_sync = 0;
  std::vector<std::vector<int>> wb_frags;   // per layer
  // write-backs (D2H) run on their own stream so they overlap the reloads
  // (H2D, copy stream): PCIe is full duplex.  wb_ev[f] = f's last write-back;
  // a reload waits for every write-back of its ring slot (and of itself)
  cudaStream_t wb_stream = nullptr;
  bool wb_own = true;                 // false: the caller's (option "wb_stream")
  std::vector<cudaEvent_t> wb_ev;
  std::vector<int> frag_slot;
  std::string err;

  int pid(int layer, int slot) const { return ctx_layout(ctx).layer_first[layer] + slot; }
  void* W(int layer, int slot) const {
    void* p = nullptr;
    dc_tensor_ptr(ctx, pid(layer, slot), &p);
    return p;
  }
  uint8_t* A(int64_t off) const { return act + off; }
};

static dc_status mfail(dc_model* m, dc_status s, const std::string& e) {
  if (m) m->err = e;
  set_global_error(e);
  return s;
}

static void build_s0(dc_model* m) {
  const int L = m->d.layers;
  std::vector<S0> comp;
  using CE = std::pair<int, int>;   // (code, expert)
  std::vector<CE> fwd_codes, bwd_codes, re_codes;
  for (int c : {F_ATTN_NORM, F_QKV, F_ATTN_MIX, F_O, F_MLP_NORM}) fwd_codes.push_back({c, -1});
  if (m->E == 0) {
    for (int c : {F_GATE_UP, F_ACT, F_DOWN}) fwd_codes.push_back({c, -1});
    for (int c : {B_DOWN, B_ACT, B_GATE_UP}) bwd_codes.push_back({c, -1});
  } else {   // synth/models.py moe_compute_ops
    fwd_codes.push_back({F_ROUTER, -1});
    fwd_codes.push_back({F_MOE_GATHER, -1});
    for (int e = 0; e < m->E; ++e)
      for (int c : {F_EXP_GU, F_EXP_ACT, F_EXP_DOWN}) fwd_codes.push_back({c, e});
    fwd_codes.push_back({F_MOE_COMBINE, -1});
    bwd_codes.push_back({B_MOE_COMBINE, -1});
    for (int e = 0; e < m->E; ++e)
      for (int c : {B_EXP_DOWN, B_EXP_ACT, B_EXP_GU}) bwd_codes.push_back({c, e});
    bwd_codes.push_back({B_ROUTER, -1});
  }
  for (int c : {B_MLP_NORM, B_O, B_ATTN_MIX, B_QKV, B_ATTN_NORM}) bwd_codes.push_back({c, -1});
  // layer checkpointing: the forward ops the layer's gradients need
  // (all but the op that forms the layer output from the saved pieces)
  for (const CE& ce : fwd_codes)
    if (ce.first != F_DOWN && ce.first != F_MOE_COMBINE) re_codes.push_back(ce);
  auto params_of = [&](int code, int e, int l) -> std::vector<int> {
    switch (code) {
      case F_ATTN_NORM: case B_ATTN_NORM: return {m->pid(l, P_G1)};
      case F_QKV: case B_QKV: return {m->pid(l, P_Q), m->pid(l, P_K), m->pid(l, P_V)};
      case F_O: case B_O: return {m->pid(l, P_O)};
      case F_MLP_NORM: case B_MLP_NORM: return {m->pid(l, P_G2)};
      case F_GATE_UP: case B_GATE_UP: return {m->pid(l, P_GATE), m->pid(l, P_UP)};
      case F_DOWN: case B_DOWN: return {m->pid(l, P_DOWN)};
      case F_ROUTER: case B_ROUTER: return {m->pid(l, P_ROUTER)};
      case F_EXP_GU: case B_EXP_GU: return {m->pid(l, p_w1(e)), m->pid(l, p_w3(e))};
      case F_EXP_DOWN: case B_EXP_DOWN: return {m->pid(l, p_w2(e))};
      default: return {};
    }
  };
  auto op = [&](const CE& ce, bool fwd, int mu, int l, bool re) {
    S0 o{K_COMPUTE, ce.first, fwd, mu, l, params_of(ce.first, ce.second, l)};
    o.re = re;
    o.e = ce.second;
    return o;
  };
  // n micro-steps; every micro-step reduce-scatters its gradients
  // into the partitioned accumulator, the last one also updates
  for (int mu = 0; mu < m->n_micro; ++mu) {
    for (int l = 0; l < L; ++l)
      for (const CE& c : fwd_codes) comp.push_back(op(c, true, mu, l, false));
    comp.push_back({K_COMPUTE, F_LOSS, true, mu, L - 1, {}});
    for (int l = L - 1; l >= 0; --l) {
      if (m->d.checkpoint)
        for (const CE& c : re_codes) comp.push_back(op(c, false, mu, l, true));
      for (const CE& c : bwd_codes) comp.push_back(op(c, false, mu, l, false));
      comp.push_back({K_RS, RS_OP, false, mu, l, {}});
    }
  }
  // S_0: gather before first use, release after last use, per region
  m->s0.clear();
  size_t i = 0;
  while (i < comp.size()) {
    size_t j = i;
    while (j < comp.size() && comp[j].fwd == comp[i].fwd && comp[j].micro == comp[i].micro) ++j;
    std::map<int, size_t> first, last;
    for (size_t k = i; k < j; ++k)
      for (int p : comp[k].params) {
        if (!first.count(p)) first[p] = k;
        last[p] = k;
      }
    for (size_t k = i; k < j; ++k) {
      for (auto& kv : first)
        if (kv.second == k) m->s0.push_back({K_AG, -1, comp[k].fwd, comp[k].micro, comp[k].layer, {kv.first}});
      m->s0.push_back(comp[k]);
      for (auto& kv : last)
        if (kv.second == k) m->s0.push_back({K_REL, -1, comp[k].fwd, comp[k].micro, comp[k].layer, {kv.first}});
    }
    i = j;
  }
}

extern "C" dc_status dc_model_create(dc_ctx* ctx, const dc_model_dims* d, dc_model** out) {
  if (!ctx || !d || !out) return mfail(nullptr, DC_EINVAL, "dc_model_create: null argument");
  auto m = std::make_unique<dc_model>();
  m->ctx = ctx;
  m->d = *d;
  m->n_micro = ctx_micro_steps(ctx);
  // virtual ranks run their persistent GEMMs concurrently on one GPU: a
  // stream-K tail could then wait on a pair that cannot become resident
  m->stream_k = !((ctx_flags(ctx) & DC_VIRTUAL_RANKS) && ctx_world(ctx) > 1);
  // RS + Adam beside the backward GEMMs at N > 1, where the reduce-scatter is
  // NVLink-bound and must hide behind compute.  At N = 1 it is a local
  // HBM-bound pass that only trades SMs and clock with the power-capped GEMMs:
  // in compute-stream order the step is as fast (graph replay: 185.8-186.2 vs
  // 185.5-186.5 ms, profiles/r01g/rs_order_ab.md) and no GEMM waits for SMs
  // held by an rs_adam, so stream order is the N = 1 default
  m->rs_overlap = ctx_world(ctx) > 1 ? 1 : 0;
  const Layout& L = ctx_layout(ctx);
  if (d->layers != L.n_layers) return mfail(nullptr, DC_EINVAL, "dc_model_create: layer count mismatch");
  if (d->n_heads % d->n_kv) return mfail(nullptr, DC_EINVAL, "dc_model_create: n_heads % n_kv != 0");
  m->qd = d->n_heads * d->head_dim;
  m->kvd = d->n_kv * d->head_dim;
  m->qkvd = m->qd + 2 * m->kvd;
  m->grp = d->n_heads / d->n_kv;
  if (d->hidden % 256 || d->ffn % 256 || m->qd % 256 || m->kvd % 256 || d->hidden > 8192 || d->tokens % 8)
    return mfail(nullptr, DC_EINVAL, "dc_model_create: hidden/ffn/q/kv dims must be multiples of 256, hidden <= 8192");
  const int64_t h = d->hidden, f = d->ffn;
  // the elementwise glue kernels index [tokens][width] activations with 32-bit math
  if ((int64_t)d->tokens * std::max<int64_t>({2 * f, (int64_t)m->qkvd, h}) >= (1LL << 32))
    return mfail(nullptr, DC_EINVAL, "dc_model_create: tokens x widest activation must stay below 2^32 elements");
  m->E = d->n_experts;
  if (m->E != 0 && (m->E < 2 || m->E > 8 || d->tokens % (4 * m->E)))
    return mfail(nullptr, DC_EINVAL, "dc_model_create: n_experts is 0 or 2..8, tokens % (4 n_experts) == 0");
  m->R = m->E ? 2 * d->tokens / m->E : 0;
  std::vector<int64_t> want = {h, m->qd * h, m->kvd * h, m->kvd * h, h * m->qd, h};
  if (m->E == 0) {
    for (int64_t n : {f * h, f * h, h * f}) want.push_back(n);
  } else {
    want.push_back(m->E * h);
    for (int e = 0; e < m->E; ++e)
      for (int64_t n : {f * h, f * h, h * f}) want.push_back(n);
  }
  for (int l = 0; l < d->layers; ++l) {
    if (L.layer_count[l] != (int)want.size())
      return mfail(nullptr, DC_EINVAL, "dc_model_create: params per layer: 9 (Llama) or 7 + 3E (MoE) expected");
    for (int s = 0; s < (int)want.size(); ++s)
      if (ctx_numel(ctx, L.layer_first[l] + s) != want[s])
        return mfail(nullptr, DC_EINVAL, "dc_model_create: param shape mismatch");
  }
  // activation layout (256-byte aligned pieces)
  const int64_t T = d->tokens;
  uint64_t off = 0;
  auto take = [&](int64_t bytes) { int64_t o = (int64_t)off; off += (bytes + 255) / 256 * 256; return o; };
  m->la.resize(d->layers);
  if (d->checkpoint != 0 && d->checkpoint != 1) return mfail(nullptr, DC_EINVAL, "dc_model_create: checkpoint is 0 or 1");
  for (int l = 0; l < d->layers; ++l) {
    LayerAct& a = m->la[l];
    if (l > 0 && d->checkpoint) {          // one shared set of layer activations,
      a = m->la[0];                        // each layer keeps only its output y
      a.y = take(T * h * 2);
      continue;
    }
    a.h1 = take(T * h * 2); a.rstd1 = take(T * 4); a.qkv = take(T * m->qkvd * 2); a.a = take(T * m->qd * 2);
    a.x2 = take(T * h * 2); a.h2 = take(T * h * 2); a.rstd2 = take(T * 4);
    const int64_t rows = m->E ? 2 * T : T;          // top-2: every token in two experts
    if (m->E) { a.g01 = take(T * 2 * 4); a.X = take(rows * h * 2); }
    a.gu = take(rows * 2 * f * 2);
    a.act = take(rows * f * 2);
    if (m->E) a.O = take(rows * h * 2);
    a.y = take(T * h * 2);
    if (l == 0) m->layer_act_bytes = off;
  }
  const uint64_t ws0 = off;
  m->ws_dA = take(T * h * 2); m->ws_dB = take(T * h * 2); m->ws_dact = take(T * f * 2);
  m->ws_dgu = take(T * 2 * f * 2); m->ws_dh = take(T * h * 2); m->ws_dx2 = take(T * h * 2);
  m->ws_dqkv = take(T * m->qkvd * 2); m->ws_dgp = take(rmsnorm_bwd_ws_floats((int)T, (int)h) * 4);   // dg partials (+ row dots)
  m->ws_lossp = take(1024 * 4); m->ws_loss = take(4 * (int64_t)m->n_micro);
  m->ws_sk = take((int64_t)gemm_workspace_bytes());
  if (m->E) {
    m->ws_dO = take(2 * T * h * 2); m->ws_dX = take(2 * T * h * 2); m->ws_dl0 = take(T * 4);
    m->ws_rgp = take((int64_t)moe_router_dw_blocks((int)T) * m->E * h * 4);
  }
  m->ws_bytes = off - ws0;
  m->act_bytes = off;
  build_s0(m.get());
  // opt-in (dc_model_set_option): bit-identical, but the epilogue becomes
  // HBM-bound and slows the dW GEMMs more than it saves (profiles/r01)
  m->fused_adam = false;
  // opt-in: bit-identical and relieves the SM contention, but the 1 kW power
  // cap lowers the clock by as much as the overlap gains (profiles/r01)
  m->side_adam = false;
  if (const char* e = getenv("DC_FUSE_ACT")) m->fuse_act = atoi(e) & 3;   // A/B knob
  {
    const int64_t T_ = d->tokens, H_ = d->hidden, F_ = d->ffn, qd_ = m->qd, kvd_ = m->kvd, qkvd_ = m->qkvd;
    m->bwd_mnk = T_ * F_ * H_ + H_ * F_ * T_ +                       // down_bwd: dX, dW
                 T_ * H_ * 2 * F_ + 2 * (F_ * H_ * T_) +            // gate_up_bwd: dX, dWg, dWu
                 T_ * qd_ * H_ + H_ * qd_ * T_ +                    // o_bwd: dX, dW
                 T_ * H_ * qkvd_ + qd_ * H_ * T_ + 2 * (kvd_ * H_ * T_);   // qkv_bwd: dX, dWq/k/v
  }
  const size_t n = m->s0.size();
  m->dur_us.assign(n, 0);
  m->p_mem.assign(n, 0);
  m->ev_pos.resize(n); m->ev_done.resize(n); m->ev_t0.resize(n); m->ev_t1.resize(n);
  for (size_t i = 0; i < n; ++i) {
    if (cudaEventCreateWithFlags(&m->ev_pos[i], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&m->ev_done[i], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreate(&m->ev_t0[i]) != cudaSuccess || cudaEventCreate(&m->ev_t1[i]) != cudaSuccess)
      return mfail(nullptr, DC_ECUDA, "dc_model_create: event creation failed");
  }
  for (auto& e : m->ev_join) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  if (cudaStreamCreateWithFlags(&m->cs2, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&m->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&m->ev_joinw, cudaEventDisableTiming) != cudaSuccess)
    return mfail(nullptr, DC_ECUDA, "dc_model_create: stream creation failed");
  if (const char* e = getenv("DC_DW_CONCURRENT")) m->dw_conc = atoi(e) != 0;   // A/B knob
  *out = m.release();
  return DC_OK;
}

extern "C" dc_status dc_model_destroy(dc_model* m) {
  if (!m) return DC_OK;
  for (size_t i = 0; i < m->ev_pos.size(); ++i) {
    cudaEventDestroy(m->ev_pos[i]); cudaEventDestroy(m->ev_done[i]);
    cudaEventDestroy(m->ev_t0[i]); cudaEventDestroy(m->ev_t1[i]);
  }
  for (auto& e : m->ev_join) if (e) cudaEventDestroy(e);
  for (auto& e : m->wb_ev) cudaEventDestroy(e);
  if (m->wb_stream && m->wb_own) cudaStreamDestroy(m->wb_stream);
  if (m->graph_exec) cudaGraphExecDestroy(m->graph_exec);
  if (m->graph) cudaGraphDestroy(m->graph);
  if (m->cs2 && m->cs2_own) cudaStreamDestroy(m->cs2);
  if (m->ev_fork) cudaEventDestroy(m->ev_fork);
  if (m->ev_joinw) cudaEventDestroy(m->ev_joinw);
  sm_partition_destroy(&m->part);
  delete m;
  return DC_OK;
}

extern "C" dc_status dc_model_act_bytes(const dc_model* m, uint64_t* b) {
  if (!m || !b) return mfail(nullptr, DC_EINVAL, "dc_model_act_bytes: null argument");
  *b = m->act_bytes;
  return DC_OK;
}

extern "C" dc_status dc_model_bind(dc_model* m, void* buf, uint64_t bytes, const void* x, const void* target) {
  if (!m || !buf || !x || !target) return mfail(m, DC_EINVAL, "dc_model_bind: null argument");
  if (bytes < m->act_bytes) return mfail(m, DC_EOOM, "dc_model_bind: activation buffer too small");
  if ((reinterpret_cast<uintptr_t>(buf) & 255) || (reinterpret_cast<uintptr_t>(x) & 15) ||
      (reinterpret_cast<uintptr_t>(target) & 15))
    return mfail(m, DC_EINVAL, "dc_model_bind: buffer alignment");
  m->act = reinterpret_cast<uint8_t*>(buf);
  m->x = x;
  m->target = target;
  // the stream-K workspace starts zero-filled (dc_gemm_args.workspace)
  if (cudaMemset(m->A(m->ws_sk), 0, gemm_workspace_bytes()) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess)
    return mfail(m, DC_ECUDA, "dc_model_bind: workspace clear failed");
  gemm_sk_reset(m->A(m->ws_sk), 0);
  return DC_OK;
}

// ------------------------------------------------------------------ layer ops
struct Glu { int mode; void* aux; int64_t ld_aux, off; };   // dc_gemm_args.epilogue 2 / 3

static dc_status gemm(dc_model* m, int M, int N, int K, const void* A, int64_t lda, int a_mn,
                      std::initializer_list<const void*> Bs, std::initializer_list<int64_t> ldbs,
                      std::initializer_list<int> ends, int b_mn, int split_k, void* C, int64_t ldc,
                      const void* R, int64_t ldr, cudaStream_t st, const EpiAdam* adam = nullptr,
                      const Glu* glu = nullptr) {
  // a backward GEMM carries its share of the pending layer's RS + Adam (not a
  // GLU-epilogue GEMM: its share moves to the next one)
  SideJob sj{};
  const SideJob* side = nullptr;
  if (m->pending_layer >= 0 && glu) {
    m->pending_mnk += (__int128)M * N * K;
  } else if (m->pending_layer >= 0) {
    m->pending_mnk += (__int128)M * N * K;
    const int64_t G = m->pending.g1;
    int64_t target = (int64_t)((__int128)G * m->pending_mnk / m->bwd_mnk);
    if (target > G) target = G;
    if (target > m->pending_assigned) {
      sj = m->pending;
      sj.g0 = m->pending_assigned;
      sj.g1 = target;
      m->pending_assigned = target;
      side = &sj;
    }
  }
  dc_gemm_args g{};
  g.M = M; g.N = N; g.K = K; g.A = A; g.lda = lda; g.a_mn_major = a_mn;
  int i = 0;
  for (const void* b : Bs) g.B[i++] = b;
  g.n_bseg = i;
  i = 0;
  for (int64_t l : ldbs) g.ldb[i++] = l;
  i = 0;
  for (int e : ends) g.bseg_end[i++] = e;
  g.b_mn_major = b_mn; g.b_split_k = split_k;
  for (int s = 0; s < g.n_bseg; ++s)
    for (const auto& w : m->cw)
      if (w.first == g.B[s]) {
        g.chunk_flags[s] = w.second.flags;
        g.chunk_S[s] = w.second.S;
        g.chunk_E[s] = w.second.E;
        g.chunk_numel[s] = w.second.S * ctx_world(m->ctx);
        g.chunk_value[s] = w.second.value;
      }
  if (!m->cw.empty()) ctx_wait_err(m->ctx, &g.chunk_err, &g.chunk_timeout_ns);
  g.C = C; g.ldc = ldc; g.R = R; g.ldr = ldr;
  // a stream-K pair spins on another pair's partial: never two such kernels at
  // once, so the GEMMs beside the dX GEMM (second stream) are data-parallel only
  g.stream_k = (st == m->cs2 || (m->fused_ag && ctx_virtual(m->ctx))) ? 0 : m->stream_k;
  g.workspace = g.stream_k ? m->A(m->ws_sk) : nullptr;
  g.workspace_bytes = g.stream_k ? gemm_workspace_bytes() : 0;
  g.num_sms = m->gemm_sms;
  if (glu) {
    g.epilogue = glu->mode;
    g.aux = glu->aux;
    g.ld_aux = glu->ld_aux;
    g.glu_off = glu->off;
  }
  std::string err;
  dc_status s = launch_gemm(&g, st, &err, adam, side);
  if (s != DC_OK) return mfail(m, s, err);
  return DC_OK;
}

// RMSNorm backward: dx = dres + rstd (dh g - n mean(dh g n)), dg = sum_rows dh n
// (one pass with register-resident rows, or two passes for other H; then the
// dg column sum of the partial rows)
static dc_status rmsnorm_bwd(dc_model* m, const void* dh, const void* x, const void* g, const float* rstd,
                             const void* dres, void* dx, void* dg, cudaStream_t st) {
  const int T = m->d.tokens, H = m->d.hidden;
  const int nblk = k_rmsnorm_bwd(dh, x, g, rstd, dres, dx, (float*)m->A(m->ws_dgp), T, H, st);
  k_colsum_to_bf16((float*)m->A(m->ws_dgp), nblk, H, dg, st);
  return DC_OK;
}

// micro-batch mu of the bound [n][T][H] inputs
static const void* micro_in(const dc_model* m, const void* base, int mu) {
  return reinterpret_cast<const uint8_t*>(base) + (int64_t)mu * m->d.tokens * m->d.hidden * 2;
}
static const void* layer_in(const dc_model* m, int l, int mu) {
  return l == 0 ? micro_in(m, m->x, mu) : m->A(m->la[l - 1].y);
}

static dc_status run_op(dc_model* m, const S0& o, cudaStream_t st) {
  const int T = m->d.tokens, H = m->d.hidden, F = m->d.ffn, qd = m->qd, kvd = m->kvd, qkvd = m->qkvd;
  const int l = o.layer;
  LayerAct& a = m->la[l];
  uint8_t* dcur = m->A(m->cur_d ? m->ws_dB : m->ws_dA);
  uint8_t* dnext = m->A(m->cur_d ? m->ws_dA : m->ws_dB);
  void* gslot = nullptr;
  if (!o.fwd && o.code != RS_OP) dc_grad_slot(m->ctx, l, &gslot);
  auto G = [&](int slot) {
    int64_t b = 0;
    dc_grad_offset(m->ctx, m->pid(l, slot), &b);
    return reinterpret_cast<uint8_t*>(gslot) + b;
  };
  // fused reduce-scatter + Adam in the dW epilogue (N = 1): the update of the
  // param's shard replaces the grad-slot write
  EpiAdam epi{};
  auto ADAM = [&](int slot) -> const EpiAdam* {
    if (!m->fused_active) return nullptr;
    ctx_adam_scalars(m->ctx, m->step_t, &epi);
    ctx_param_state(m->ctx, m->pid(l, slot), &epi.master, &epi.m, &epi.v, &epi.shard);
    return &epi;
  };
  dc_status s = DC_OK;
  // dW GEMMs on the second stream (forked before the dX GEMM, joined at the end
  // of the op; both only read the op's inputs and write disjoint outputs)
  cudaStream_t sw = st;
  auto fork = [&]() {
    if (!m->dw_conc || m->comm_sms > 0 || (m->fused_ag && ctx_virtual(m->ctx))) return;
    cudaEventRecord(m->ev_fork, st);
    cudaStreamWaitEvent(m->cs2, m->ev_fork, 0);
    sw = m->cs2;
  };
  switch (o.code) {
    case F_ATTN_NORM:
      k_rmsnorm_fwd(layer_in(m, l, o.micro), m->W(l, P_G1), m->A(a.h1), (float*)m->A(a.rstd1), T, H, st);
      break;
    case F_QKV:
      s = gemm(m, T, qkvd, H, m->A(a.h1), H, 0, {m->W(l, P_Q), m->W(l, P_K), m->W(l, P_V)}, {H, H, H},
               {qd / 256, (qd + kvd) / 256, qkvd / 256}, 0, 0, m->A(a.qkv), qkvd, nullptr, 0, st);
      break;
    case F_ATTN_MIX:
      k_attn_mix_fwd(m->A(a.qkv), m->A(a.a), T, qd, kvd, m->d.head_dim, m->grp, st);
      break;
    case F_O:
      s = gemm(m, T, H, qd, m->A(a.a), qd, 0, {m->W(l, P_O)}, {qd}, {H / 256}, 0, 0, m->A(a.x2), H,
               layer_in(m, l, o.micro), H, st);
      break;
    case F_MLP_NORM:
      k_rmsnorm_fwd(m->A(a.x2), m->W(l, P_G2), m->A(a.h2), (float*)m->A(a.rstd2), T, H, st);
      break;
    case F_GATE_UP:
      if (m->fuse_act & 1) {   // gu and act = SiLU(gate) * up from one GEMM (epilogue 2)
        const Glu glu{2, m->A(a.act), F, F};
        s = gemm(m, T, F, H, m->A(a.h2), H, 0, {m->W(l, P_GATE), m->W(l, P_UP)}, {H, H}, {0, 0}, 0, 0,
                 m->A(a.gu), 2 * F, nullptr, 0, st, nullptr, &glu);
      } else {
        s = gemm(m, T, 2 * F, H, m->A(a.h2), H, 0, {m->W(l, P_GATE), m->W(l, P_UP)}, {H, H},
                 {F / 256, 2 * F / 256}, 0, 0, m->A(a.gu), 2 * F, nullptr, 0, st);
      }
      break;
    case F_ACT:
      if (!(m->fuse_act & 1)) k_act_fwd(m->A(a.gu), m->A(a.act), T, F, st);
      break;
    case F_DOWN:
      s = gemm(m, T, H, F, m->A(a.act), F, 0, {m->W(l, P_DOWN)}, {F}, {H / 256}, 0, 0, m->A(a.y), H,
               m->A(a.x2), H, st);
      break;
    case F_LOSS:
      m->cur_d = 0;
      k_loss(m->A(a.y), micro_in(m, m->target, o.micro), m->A(m->ws_dA), (float*)m->A(m->ws_lossp),
             (float*)m->A(m->ws_loss) + o.micro,
             (int64_t)T * H, st);
      break;
    case B_DOWN:
      // (the executor has enqueued dc_grad_slot_acquire for this layer)
      // dact = dy Wd  (A K-major [T,H]; B = Wd [H rows = K][F] MN-major); fused:
      // the epilogue turns dact into d(gate | up) with gu (epilogue 3)
      fork();
      if (m->fuse_act & 2) {
        const Glu glu{3, m->A(a.gu), 2 * F, F};
        s = gemm(m, T, F, H, dcur, H, 0, {m->W(l, P_DOWN)}, {F}, {F / 256}, 1, 0, m->A(m->ws_dgu), 2 * F, nullptr, 0,
                 st, nullptr, &glu);
      } else {
        s = gemm(m, T, F, H, dcur, H, 0, {m->W(l, P_DOWN)}, {F}, {F / 256}, 1, 0, m->A(m->ws_dact), F, nullptr, 0, st);
      }
      if (s == DC_OK)  // dWd = dy^T act : A = dy stored [T][H] (MN-major), B = act [T][F] (MN-major)
        s = gemm(m, H, F, T, dcur, H, 1, {m->A(a.act)}, {F}, {F / 256}, 1, 0, G(P_DOWN), F, nullptr, 0, sw, ADAM(P_DOWN));
      break;
    case B_ACT:
      if (!(m->fuse_act & 2)) k_act_bwd(m->A(m->ws_dact), m->A(a.gu), m->A(m->ws_dgu), T, F, st);
      break;
    case B_GATE_UP:
      // dh2 = dgate Wg + dup Wu : A = dgu [T, 2F] K-major, B split along K
      fork();
      s = gemm(m, T, H, 2 * F, m->A(m->ws_dgu), 2 * F, 0, {m->W(l, P_GATE), m->W(l, P_UP)}, {H, H},
               {F / 64, 2 * F / 64}, 1, 1, m->A(m->ws_dh), H, nullptr, 0, st);
      if (s == DC_OK)
        s = gemm(m, F, H, T, m->A(m->ws_dgu), 2 * F, 1, {m->A(a.h2)}, {H}, {H / 256}, 1, 0, G(P_GATE), H, nullptr, 0, sw, ADAM(P_GATE));
      if (s == DC_OK)
        s = gemm(m, F, H, T, m->A(m->ws_dgu) + (int64_t)F * 2, 2 * F, 1, {m->A(a.h2)}, {H}, {H / 256}, 1, 0, G(P_UP),
                 H, nullptr, 0, sw, ADAM(P_UP));
      break;
    case B_MLP_NORM:
      s = rmsnorm_bwd(m, m->A(m->ws_dh), m->A(a.x2), m->W(l, P_G2), (float*)m->A(a.rstd2), dcur, m->A(m->ws_dx2),
                      G(P_G2), st);
      break;
    case B_O:
      // da -> dqkv[:, :qd] ; dWo = dx2^T a
      fork();
      s = gemm(m, T, qd, H, m->A(m->ws_dx2), H, 0, {m->W(l, P_O)}, {qd}, {qd / 256}, 1, 0, m->A(m->ws_dqkv), qkvd,
               nullptr, 0, st);
      if (s == DC_OK)
        s = gemm(m, H, qd, T, m->A(m->ws_dx2), H, 1, {m->A(a.a)}, {qd}, {qd / 256}, 1, 0, G(P_O), qd, nullptr, 0, sw, ADAM(P_O));
      break;
    case B_ATTN_MIX:
      k_attn_mix_bwd(m->A(m->ws_dqkv), m->A(a.qkv), T, qd, kvd, m->d.head_dim, m->grp, st);
      break;
    case B_QKV:
      fork();
      s = gemm(m, T, H, qkvd, m->A(m->ws_dqkv), qkvd, 0, {m->W(l, P_Q), m->W(l, P_K), m->W(l, P_V)}, {H, H, H},
               {qd / 64, (qd + kvd) / 64, qkvd / 64}, 1, 1, m->A(m->ws_dh), H, nullptr, 0, st);
      if (s == DC_OK)
        s = gemm(m, qd, H, T, m->A(m->ws_dqkv), qkvd, 1, {m->A(a.h1)}, {H}, {H / 256}, 1, 0, G(P_Q), H, nullptr, 0, sw, ADAM(P_Q));
      if (s == DC_OK)
        s = gemm(m, kvd, H, T, m->A(m->ws_dqkv) + (int64_t)qd * 2, qkvd, 1, {m->A(a.h1)}, {H}, {H / 256}, 1, 0, G(P_K),
                 H, nullptr, 0, sw, ADAM(P_K));
      if (s == DC_OK)
        s = gemm(m, kvd, H, T, m->A(m->ws_dqkv) + (int64_t)(qd + kvd) * 2, qkvd, 1, {m->A(a.h1)}, {H}, {H / 256}, 1,
                 0, G(P_V), H, nullptr, 0, sw, ADAM(P_V));
      break;
    case B_ATTN_NORM: {
      s = rmsnorm_bwd(m, m->A(m->ws_dh), layer_in(m, l, o.micro), m->W(l, P_G1), (float*)m->A(a.rstd1),
                      m->A(m->ws_dx2), dnext, G(P_G1), st);
      if (s != DC_OK) return mfail(m, s, "rmsnorm backward launch failed");
      if ((s = dc_grad_slot_publish(m->ctx, l, st)) != DC_OK) return s;
      if (m->pending_layer >= 0) {     // the hosted RS + Adam is complete (stream order)
        if (m->pending_assigned != m->pending.g1) return mfail(m, DC_ESTATE, "side job not fully assigned");
        if ((s = ctx_post_consumed(m->ctx, m->pending_layer, st)) != DC_OK) return s;
        m->pending_layer = -1;
      }
      m->cur_d ^= 1;
      break;
    }
    // ---- Mixtral-shaped MoE MLP; expert e's R rows
    // sit at row e R of X / gu / act / O and of the dO / dX workspaces
    case F_ROUTER:
      k_moe_router_fwd(m->A(a.h2), m->W(l, P_ROUTER), (float*)m->A(a.g01), T, H, m->E, st);
      break;
    case F_MOE_GATHER:
      k_moe_gather(m->A(a.h2), m->A(a.X), T, H, m->E, st);
      break;
    case F_EXP_GU: {
      const int e = o.e, R = m->R;
      if (m->fuse_act & 1) {
        const Glu glu{2, m->A(a.act) + (int64_t)e * R * F * 2, F, F};
        s = gemm(m, R, F, H, m->A(a.X) + (int64_t)e * R * H * 2, H, 0, {m->W(l, p_w1(e)), m->W(l, p_w3(e))},
                 {H, H}, {0, 0}, 0, 0, m->A(a.gu) + (int64_t)e * R * 2 * F * 2, 2 * F, nullptr, 0, st, nullptr, &glu);
      } else {
        s = gemm(m, R, 2 * F, H, m->A(a.X) + (int64_t)e * R * H * 2, H, 0, {m->W(l, p_w1(e)), m->W(l, p_w3(e))},
                 {H, H}, {F / 256, 2 * F / 256}, 0, 0, m->A(a.gu) + (int64_t)e * R * 2 * F * 2, 2 * F, nullptr, 0, st);
      }
      break;
    }
    case F_EXP_ACT:
      if (!(m->fuse_act & 1))
        k_act_fwd(m->A(a.gu) + (int64_t)o.e * m->R * 2 * F * 2, m->A(a.act) + (int64_t)o.e * m->R * F * 2, m->R, F,
                  st);
      break;
    case F_EXP_DOWN: {
      const int e = o.e, R = m->R;
      s = gemm(m, R, H, F, m->A(a.act) + (int64_t)e * R * F * 2, F, 0, {m->W(l, p_w2(e))}, {F}, {H / 256}, 0, 0,
               m->A(a.O) + (int64_t)e * R * H * 2, H, nullptr, 0, st);
      break;
    }
    case F_MOE_COMBINE:
      k_moe_combine(m->A(a.x2), m->A(a.O), (const float*)m->A(a.g01), m->A(a.y), T, H, m->E, st);
      break;
    case B_MOE_COMBINE:
      // (the executor has enqueued dc_grad_slot_acquire for this layer)
      k_moe_combine_bwd(dcur, m->A(a.O), (const float*)m->A(a.g01), m->A(m->ws_dO), (float*)m->A(m->ws_dl0), T, H,
                        m->E, st);
      break;
    case B_EXP_DOWN: {
      const int e = o.e, R = m->R;
      uint8_t* dOe = m->A(m->ws_dO) + (int64_t)e * R * H * 2;
      // dact_e = dO_e W2_e (fused: -> d(gate | up)_e with gu_e) ; dW2_e = dO_e^T act_e
      fork();
      if (m->fuse_act & 2) {
        const Glu glu{3, m->A(a.gu) + (int64_t)e * R * 2 * F * 2, 2 * F, F};
        s = gemm(m, R, F, H, dOe, H, 0, {m->W(l, p_w2(e))}, {F}, {F / 256}, 1, 0, m->A(m->ws_dgu), 2 * F, nullptr, 0,
                 st, nullptr, &glu);
      } else {
        s = gemm(m, R, F, H, dOe, H, 0, {m->W(l, p_w2(e))}, {F}, {F / 256}, 1, 0, m->A(m->ws_dact), F, nullptr, 0, st);
      }
      if (s == DC_OK)
        s = gemm(m, H, F, R, dOe, H, 1, {m->A(a.act) + (int64_t)e * R * F * 2}, {F}, {F / 256}, 1, 0, G(p_w2(e)), F,
                 nullptr, 0, sw);
      break;
    }
    case B_EXP_ACT:
      if (!(m->fuse_act & 2))
        k_act_bwd(m->A(m->ws_dact), m->A(a.gu) + (int64_t)o.e * m->R * 2 * F * 2, m->A(m->ws_dgu), m->R, F, st);
      break;
    case B_EXP_GU: {
      const int e = o.e, R = m->R;
      const uint8_t* Xe = m->A(a.X) + (int64_t)e * R * H * 2;
      // dX_e = d(gate|up)_e [W1_e; W3_e] (B split along K) ; dW1_e, dW3_e = d(gate), d(up)^T X_e
      fork();
      s = gemm(m, R, H, 2 * F, m->A(m->ws_dgu), 2 * F, 0, {m->W(l, p_w1(e)), m->W(l, p_w3(e))}, {H, H},
               {F / 64, 2 * F / 64}, 1, 1, m->A(m->ws_dX) + (int64_t)e * R * H * 2, H, nullptr, 0, st);
      if (s == DC_OK)
        s = gemm(m, F, H, R, m->A(m->ws_dgu), 2 * F, 1, {Xe}, {H}, {H / 256}, 1, 0, G(p_w1(e)), H, nullptr, 0, sw);
      if (s == DC_OK)
        s = gemm(m, F, H, R, m->A(m->ws_dgu) + (int64_t)F * 2, 2 * F, 1, {Xe}, {H}, {H / 256}, 1, 0, G(p_w3(e)), H,
                 nullptr, 0, sw);
      break;
    }
    case B_ROUTER:
      // dh2 = dX_e0 + dX_e1 + dlogits Wr ; dWr = dlogits^T h2 (block partials, fixed-order column sum)
      k_moe_router_bwd(m->A(m->ws_dX), (const float*)m->A(m->ws_dl0), m->W(l, P_ROUTER), m->A(a.h2), m->A(m->ws_dh),
                       (float*)m->A(m->ws_rgp), T, H, m->E, st);
      k_colsum_to_bf16((float*)m->A(m->ws_rgp), moe_router_dw_blocks(T), m->E * H, G(P_ROUTER), st);
      break;
    default:
      return mfail(m, DC_EINVAL, "run_op: bad op");
  }
  if (sw != st) {                    // join the dW stream (the op ends when both do)
    cudaEventRecord(m->ev_joinw, sw);
    cudaStreamWaitEvent(st, m->ev_joinw, 0);
  }
  if (s != DC_OK) return s;
  if (cudaGetLastError() != cudaSuccess) return mfail(m, DC_ECUDA, std::string("layer op launch failed: ") + op_name(o.code));
  return DC_OK;
}

// resident-memory profile P_mem(o): static state (bf16 shard, fp32
// master, grad slots, workspace, inputs; NOT Adam m/v — reading D14) + live
// gathered buffers under S_0 + saved activations of layers between their
// forward op and the end of their backward.
static void compute_pmem(dc_model* m) {
  const Layout& L = ctx_layout(m->ctx);
  const int N = ctx_world(m->ctx);
  const int64_t T = m->d.tokens, h = m->d.hidden;
  int64_t stat = L.shard_elems * 6 + 2 * L.grad_slot_bytes + (int64_t)m->ws_bytes + 2 * m->n_micro * T * h * 2 +
                 (m->n_micro > 1 ? L.shard_elems * 4 : 0);   // fp32 grad accumulator
  int64_t live_ag = 0, act = 0;
  const int64_t f = m->d.ffn, R = m->R;
  // bytes of saved activation a forward op produces
  auto piece = [&](int code) -> int64_t {
    switch (code) {
      case F_ATTN_NORM: return T * h * 2 + T * 4;
      case F_QKV: return T * m->qkvd * 2;
      case F_ATTN_MIX: return T * m->qd * 2;
      case F_O: return T * h * 2;
      case F_MLP_NORM: return T * h * 2 + T * 4;
      case F_GATE_UP: return T * 2 * f * 2;
      case F_ACT: return T * f * 2;
      case F_DOWN: return T * h * 2;
      case F_ROUTER: return T * 2 * 4;
      case F_MOE_GATHER: return 2 * T * h * 2;
      case F_EXP_GU: return R * 2 * f * 2;
      case F_EXP_ACT: return R * f * 2;
      case F_EXP_DOWN: return R * h * 2;
      case F_MOE_COMBINE: return T * h * 2;
      default: return 0;
    }
  };
  const int out_code = m->E ? F_MOE_COMBINE : F_DOWN;   // forms the layer output y
  int64_t layer_total = 0;
  for (const S0& o : m->s0)
    if (o.kind == K_COMPUTE && o.fwd && o.layer == 0 && o.micro == 0) layer_total += piece(o.code);
  // checkpointing: one shared layer activation set (static) + each layer's y
  if (m->d.checkpoint) stat += (int64_t)m->layer_act_bytes - T * h * 2;
  for (size_t i = 0; i < m->s0.size(); ++i) {
    const S0& o = m->s0[i];
    m->p_mem[i] = stat + live_ag + act;
    if (o.kind == K_AG) live_ag += L.S[o.params[0]] * N * 2;
    else if (o.kind == K_REL) live_ag -= L.S[o.params[0]] * N * 2;
    else if (o.kind == K_COMPUTE && m->d.checkpoint) {
      if (o.fwd && o.code == out_code) act += piece(out_code);
      else if (!o.fwd && o.code == B_ATTN_NORM) act -= piece(out_code);
    } else if (o.kind == K_COMPUTE) {
      if (o.fwd) act += piece(o.code);
      else if (o.code == B_ATTN_NORM) act -= layer_total;
    }
  }
}

// Read the per-op CUDA-event durations of the last profiled step (µs).
static dc_status collect_profile(dc_model* m) {
  const bool timed_ag = ctx_world(m->ctx) > 1;
  std::vector<char> gathered(m->s0.size(), 0);   // gathers issued by the bound schedule
  if (timed_ag) {
    const dc_schedule* sc = ctx_sched(m->ctx);
    for (int i = 0, n = sc ? sched_num_ops(sc) : 0; i < n; ++i) {
      int kind, id, nm, np, nw;
      const int64_t* mem; const int* posts; const int* waits;
      int64_t off, bytes;
      sched_op(sc, i, &kind, &id, &mem, &nm, &off, &bytes, &posts, &np, &waits, &nw);
      if (kind == K_AG && id >= 0 && id < (int)gathered.size()) gathered[id] = 1;
    }
  }
  for (size_t i = 0; i < m->s0.size(); ++i) {
    if (m->s0[i].kind == K_AG) {     // N > 1: the gather's transfer time (0 if unsharded / fused away)
      m->dur_us[i] = 0;
      if (!gathered[i]) continue;
      if (cudaEventSynchronize(m->ev_t1[i]) != cudaSuccess) return mfail(m, DC_ECUDA, "profile: event sync failed");
      float ms = 0.0f;
      if (cudaEventElapsedTime(&ms, m->ev_t0[i], m->ev_t1[i]) == cudaSuccess)
        m->dur_us[i] = std::max<int64_t>(1, (int64_t)std::llround(ms * 1000.0));
      continue;
    }
    if (m->s0[i].kind != K_COMPUTE && m->s0[i].kind != K_RS) continue;
    if (cudaEventSynchronize(m->ev_t1[i]) != cudaSuccess) return mfail(m, DC_ECUDA, "profile: event sync failed");
    float ms = 0.0f;
    if (cudaEventElapsedTime(&ms, m->ev_t0[i], m->ev_t1[i]) == cudaSuccess)
      m->dur_us[i] = std::max<int64_t>(1, (int64_t)std::llround(ms * 1000.0));
  }
  m->profile_pending = false;
  return DC_OK;
}

extern "C" dc_status dc_model_profile_json(const dc_model* mc, char* buf, size_t* len) {
  dc_model* m = const_cast<dc_model*>(mc);
  if (!m || !len) return mfail(nullptr, DC_EINVAL, "dc_model_profile_json: null argument");
  if (m->profile_pending) {
    dc_status s = collect_profile(m);
    if (s != DC_OK) return s;
  }
  compute_pmem(m);
  const Layout& L = ctx_layout(m->ctx);
  const int N = ctx_world(m->ctx);
  std::string s = "{\"ops\":[";
  for (size_t i = 0; i < m->s0.size(); ++i) {
    const S0& o = m->s0[i];
    if (i) s += ',';
    const char* kind = o.kind == K_AG ? "ag" : o.kind == K_REL ? "rel" : o.kind == K_RS ? "rs" : "compute";
    s += "{\"dur_us\":" + std::to_string(m->dur_us[i]) + ",\"id\":" + std::to_string(i) + ",\"kind\":\"" + kind +
         "\",\"layer\":" + std::to_string(o.layer) + ",\"micro\":" + std::to_string(o.micro) + ",\"name\":\"" +
         (o.kind == K_AG ? "ag" : o.kind == K_REL ? "rel" : op_label(o)) +
         "\",\"p_mem\":" +
         std::to_string(m->p_mem[i]) + ",\"params\":[";
    for (size_t j = 0; j < o.params.size(); ++j) s += (j ? "," : "") + std::to_string(o.params[j]);
    s += "],\"phase\":\"" + std::string(o.fwd ? "fwd" : "bwd") + "\",\"transient\":0}";
  }
  s += "],\"params\":[";
  for (int p = 0; p < (int)L.S.size(); ++p) {
    if (p) s += ',';
    int layer = 0;
    for (int l = 0; l < L.n_layers; ++l)
      if (p >= L.layer_first[l]) layer = l;
    s += "{\"bytes\":" + std::to_string(L.S[p] * N * 2) + ",\"id\":" + std::to_string(p) + ",\"layer\":" +
         std::to_string(layer) + "}";
  }
  s += "]}";
  const size_t cap = *len;
  *len = s.size();
  if (!buf) return DC_OK;
  if (cap < s.size() + 1) return mfail(m, DC_EOOM, "dc_model_profile_json: buffer too small");
  memcpy(buf, s.c_str(), s.size() + 1);
  return DC_OK;
}

// per-op timing event: inside a graph capture an external event-record node,
// so every replay records it (the timed replays keep their per-op breakdown)
static void prof_rec(dc_model* m, cudaEvent_t ev, cudaStream_t st) {
  if (m->capturing) cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal);
  else cudaEventRecord(ev, st);
}

extern "C" dc_status dc_model_step(dc_model* m, int32_t step_t, int32_t profile, cudaStream_t ucs, cudaStream_t ags,
                                   cudaStream_t rss, cudaStream_t cps) {
  if (!m || !m->act) return mfail(m, DC_ESTATE, "dc_model_step: model not bound");
  const dc_schedule* sc = ctx_sched(m->ctx);
  if (!sc) return mfail(m, DC_ESTATE, "dc_model_step: no schedule bound");
  const int64_t l0 = launch_count();
  const int N = ctx_world(m->ctx);
  if (step_t < 1) return mfail(m, DC_EINVAL, "dc_model_step: step_t is 1-based");
  m->step_t = step_t;
  // the caller's compute stream orders the step; with an SM partition the work
  // runs on the partition's streams (GEMM side / communication + Adam side)
  cudaStream_t cs = ucs;
  if (m->comm_sms > 0) {
    if (!m->part.ctx_gemm) {
      int dev = 0;
      cudaGetDevice(&dev);
      std::string err;
      dc_status ps = sm_partition_create(dev, m->comm_sms, &m->part, &err);
      if (ps != DC_OK) return mfail(m, ps, "dc_model_step: " + err);
    }
    cs = m->part.compute;
    rss = m->part.rs;
    ags = m->part.ag;
    m->gemm_sms = m->part.gemm_sms;
    ctx_set_rs_ctas(m->ctx, 2 * m->part.comm_sms);
  } else {
    m->gemm_sms = 0;
    ctx_set_rs_ctas(m->ctx, 0);
  }
  m->fused_ag = N > 1 && ctx_fused_ag(m->ctx);
  if (m->fused_ag && ctx_virtual(m->ctx)) {
    // virtual ranks share one GPU: a GEMM waiting for another rank's chunks
    // must not keep that rank's GEMMs off the SMs, so every rank's persistent
    // GEMM gets 1/N of the SMs (all N resident at once) and no second GEMM
    // stream; one process per GPU needs none of this
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    m->gemm_sms = std::max(2, sms / N / 2 * 2);
  }
  if (!m->rs_overlap) rss = cs;
  // an offloaded fragment is reloaded before its layer's RS op (reading D17),
  // i.e. after the dW GEMMs: the fused update needs every state resident
  // (both also assume one micro-step: the update consumes the slot directly)
  m->fused_active = m->fused_adam && m->n_micro == 1;
  m->side_active = m->side_adam && !m->fused_adam && m->n_micro == 1;
  m->pending_layer = -1;
  for (int i = 0, n = sched_num_ops(sc); i < n && (m->fused_active || m->side_active); ++i) {
    int kind, id, nm, np, nw;
    const int64_t* mem; const int* posts; const int* waits;
    int64_t off, bytes;
    sched_op(sc, i, &kind, &id, &mem, &nm, &off, &bytes, &posts, &np, &waits, &nw);
    if (kind >= K_OFF) m->fused_active = m->side_active = false;
  }
  if (m->offload_all_sync) {
    m->fused_active = m->side_active = false;
  }
  dc_status s = dc_step_begin(m->ctx, ++m->epoch, ucs);
  if (s != DC_OK) return mfail(m, s, dc_last_error(m->ctx));
  // graph mode: the stream-K flags restart from zero with the step too
  if (ctx_graph_mode(m->ctx)) gemm_sk_reset(m->A(m->ws_sk), ucs);
  // graph mode: this step's Adam scalars go to device memory (a captured step
  // leaves this to dc_model_graph_launch, which writes them before each replay)
  if (ctx_graph_mode(m->ctx) && !m->capturing && (s = ctx_set_step_scalars(m->ctx, step_t, ucs)) != DC_OK)
    return mfail(m, s, dc_last_error(m->ctx));
  // streams must not run ahead of the previous step's tail on the compute stream
  cudaEventRecord(m->ev_join[0], ucs);
  if (cs != ucs) cudaStreamWaitEvent(cs, m->ev_join[0], 0);
  cudaStreamWaitEvent(ags, m->ev_join[0], 0);
  cudaStreamWaitEvent(rss, m->ev_join[0], 0);
  cudaStreamWaitEvent(cps, m->ev_join[0], 0);
  if (m->host_states) cudaStreamWaitEvent(m->wb_stream, m->ev_join[0], 0);
  std::vector<cudaEvent_t> gather_ev(ctx_layout(m->ctx).S.size(), nullptr);
  std::vector<int> gather_id(ctx_layout(m->ctx).S.size(), -1);
  const int nops = sched_num_ops(sc);
  for (int i = 0; i < nops; ++i) {
    int kind, id, nm, np, nw;
    const int64_t* mem; const int* posts; const int* waits;
    int64_t off, bytes;
    sched_op(sc, i, &kind, &id, &mem, &nm, &off, &bytes, &posts, &np, &waits, &nw);
    switch (kind) {
      case K_AG:
        if (N > 1) {
          cudaEventRecord(m->ev_pos[id], cs);
          cudaStreamWaitEvent(ags, m->ev_pos[id], 0);
          if (profile) ctx_set_gather_timing(m->ctx, m->ev_t0[id], m->ev_t1[id]);   // transfer time
          else if (m->fused_ag) ctx_set_gather_timing(m->ctx, m->ev_t0[id], nullptr);
          // (fused: ev_t0[id] = every receiver ready, the push is next on the AG stream)
          s = dc_gather(m->ctx, id, ags, m->ev_done[id]);
          for (int j = 0; j < nm; ++j) {
            gather_ev[mem[j]] = m->ev_done[id];
            gather_id[mem[j]] = id;
          }
        } else {
          s = dc_gather(m->ctx, id, ags, nullptr);
        }
        break;
      case K_REL:
        s = dc_release(m->ctx, id, cs);
        break;
      case K_COMPUTE: {
        const S0& o = m->s0[id];
        m->cw.clear();
        if (N > 1)
          for (int p : o.params) {
            if (!gather_ev[p]) continue;
            ChunkWait w;
            if (m->fused_ag && gemm_b_op(o.code) && ctx_chunk_wait(m->ctx, gather_id[p], p, &w)) {
              void* full = nullptr;           // the op's GEMMs wait per chunk of this B operand
              dc_tensor_ptr(m->ctx, p, &full);
              m->cw.push_back({full, w});
              // ... but start only once the push is the next kernel on the AG stream: the
              // persistent GEMM then never holds the SMs ahead of the push it waits for
              cudaStreamWaitEvent(cs, m->ev_t0[gather_id[p]], 0);
            } else {
              cudaStreamWaitEvent(cs, gather_ev[p], 0);
            }
          }
        if (o.code == B_DOWN || o.code == B_MOE_COMBINE) {   // first non-recompute backward op of the layer
          s = dc_grad_slot_acquire(m->ctx, o.layer, cs);
          if (s != DC_OK) return mfail(m, s, dc_last_error(m->ctx));
        }
        if (profile) prof_rec(m, m->ev_t0[id], cs);
        s = run_op(m, o, cs);
        m->cw.clear();
        if (profile) prof_rec(m, m->ev_t1[id], cs);
        break;
      }
      case K_RS: {
        const S0& o = m->s0[id];
        cudaEventRecord(m->ev_pos[id], cs);
        cudaStreamWaitEvent(rss, m->ev_pos[id], 0);
        if (m->host_states && m->offload_all_sync) {
          // baseline: reload this layer's fragments now and block on them
          cudaStreamWaitEvent(cps, m->ev_pos[id], 0);
          for (int f : m->wb_frags[o.layer]) {
            for (size_t g = 0; g < m->frag_slot.size(); ++g)
              if (m->frag_slot[g] == m->frag_slot[f]) cudaStreamWaitEvent(cps, m->wb_ev[g], 0);
            if ((s = dc_offload(m->ctx, f, DC_H2D_START, cps)) != DC_OK) break;
            if ((s = dc_offload(m->ctx, f, DC_H2D_SYNC, rss)) != DC_OK) break;
            if ((s = dc_offload(m->ctx, f, DC_H2D_SYNC, cs)) != DC_OK) break;
          }
          if (s != DC_OK) break;
        }
        if (profile) prof_rec(m, m->ev_t0[id], rss);
        if (m->fused_active)   // the weights were updated in their dW epilogues; the norm gains remain
          s = reduce_scatter_params(m->ctx, o.layer, step_t, o.micro, {m->pid(o.layer, P_G1), m->pid(o.layer, P_G2)},
                                    rss);
        else if (m->side_active && o.layer > 0) {   // rides on layer l-1's backward GEMMs
          s = ctx_side_job(m->ctx, o.layer, step_t, &m->pending);
          m->pending_layer = o.layer;
          m->pending_assigned = 0;
          m->pending_mnk = 0;
        } else
          s = dc_reduce_scatter_step(m->ctx, o.layer, step_t, o.micro, rss);
        if (profile) prof_rec(m, m->ev_t1[id], rss);
        if (s == DC_OK && m->host_states && !m->wb_frags[o.layer].empty()) {
          // reading D28: the updated host-resident fragments go straight back
          cudaEventRecord(m->ev_done[id], rss);
          cudaStreamWaitEvent(m->wb_stream, m->ev_done[id], 0);
          for (int f : m->wb_frags[o.layer]) {
            if ((s = dc_offload(m->ctx, f, DC_WRITEBACK, m->wb_stream)) != DC_OK) break;
            cudaEventRecord(m->wb_ev[f], m->wb_stream);
          }
        }
        break;
      }
      case K_OFF:
        s = dc_offload(m->ctx, (int)mem[0], DC_D2H_START, cps);
        break;
      case K_OFFSYNC:
        s = dc_offload(m->ctx, (int)mem[0], DC_D2H_SYNC_FREE, cs);
        break;
      case K_RELOAD:
        cudaEventRecord(m->ev_join[1], cs);
        cudaStreamWaitEvent(cps, m->ev_join[1], 0);
        if (m->host_states && mem[0] < (int64_t)m->frag_slot.size() && m->frag_slot[mem[0]] >= 0)
          for (size_t g = 0; g < m->frag_slot.size(); ++g)      // the slot's earlier occupants are written back
            if (m->frag_slot[g] == m->frag_slot[mem[0]]) cudaStreamWaitEvent(cps, m->wb_ev[g], 0);
        s = dc_offload(m->ctx, (int)mem[0], DC_H2D_START, cps);
        break;
      case K_RELOADSYNC:
        s = dc_offload(m->ctx, (int)mem[0], DC_H2D_SYNC, rss);
        break;
      default:
        return mfail(m, DC_EINVAL, "dc_model_step: bad schedule op");
    }
    if (s != DC_OK) return mfail(m, s, std::string("dc_model_step: ") + dc_last_error(m->ctx) + " / " + m->err);
  }
  // join every stream into the caller's compute stream (step end)
  cudaEventRecord(m->ev_join[1], ags);
  cudaEventRecord(m->ev_join[2], rss);
  cudaEventRecord(m->ev_join[3], cps);
  cudaStreamWaitEvent(ucs, m->ev_join[1], 0);
  cudaStreamWaitEvent(ucs, m->ev_join[2], 0);
  cudaStreamWaitEvent(ucs, m->ev_join[3], 0);
  // host-resident states (D28): the write-backs of the last updated fragments
  // are NOT joined here — they overlap the next step's forward (the next
  // reload of a fragment, and of its ring slot, waits for them: wb_ev);
  // dc_model_join_states orders a stream after them
  if (cs != ucs) {
    cudaEventRecord(m->ev_join[4], cs);
    cudaStreamWaitEvent(ucs, m->ev_join[4], 0);
  }
  if (cudaGetLastError() != cudaSuccess) return mfail(m, DC_ECUDA, "dc_model_step: CUDA error");
  m->launches = launch_count() - l0;
  if (profile) {
    m->profile_pending = true;
    if (profile == 1) return collect_profile(m);   // 2: events only, read later
  }
  return DC_OK;
}

extern "C" dc_status dc_model_join_states(dc_model* m, cudaStream_t stream) {
  if (!m) return mfail(nullptr, DC_EINVAL, "dc_model_join_states: null model");
  if (!m->host_states || !m->wb_stream) return DC_OK;
  if (cudaEventRecord(m->ev_join[3], m->wb_stream) != cudaSuccess ||
      cudaStreamWaitEvent(stream, m->ev_join[3], 0) != cudaSuccess)
    return mfail(m, DC_ECUDA, "dc_model_join_states: event failed");
  return DC_OK;
}

extern "C" dc_status dc_model_loss_ptr(const dc_model* m, float** loss) {
  if (!m || !loss || !m->act) return mfail(nullptr, DC_EINVAL, "dc_model_loss_ptr: not bound");
  *loss = (float*)m->A(m->ws_loss);
  return DC_OK;
}

extern "C" dc_status dc_model_act_ptr(const dc_model* m, int32_t layer, int32_t which, void** p) {
  if (!m || !p || !m->act || layer < 0 || layer >= m->d.layers) return mfail(nullptr, DC_EINVAL, "dc_model_act_ptr: bad args");
  const LayerAct& a = m->la[layer];
  const int64_t offs[] = {a.h1, a.qkv, a.a, a.x2, a.h2, a.gu, a.act, a.y, m->ws_dA, m->ws_dB, a.g01, a.X, a.O};
  const int nw = m->E ? 13 : 10;
  if (which < 0 || which >= nw) return mfail(nullptr, DC_EINVAL, "dc_model_act_ptr: which in [0, 10) (MoE: [0, 13))");
  *p = m->A(offs[which]);
  return DC_OK;
}

extern "C" dc_status dc_model_set_option(dc_model* m, const char* key, int64_t value) {
  if (!m || !key) return mfail(nullptr, DC_EINVAL, "dc_model_set_option: null argument");
  if (!strcmp(key, "dw_stream") || !strcmp(key, "wb_stream")) {
    // caller-supplied (not owned) stream for the concurrent dW GEMMs / the
    // host-state write-backs instead of one the library creates: several
    // virtual ranks in one process then draw every stream from one pool whose
    // streams sit on distinct hardware queues, so no rank's spin-wait can
    // block a peer's dW GEMM or copy (profiles/r02/stalls/)
    if (!value) return mfail(m, DC_EINVAL, "dw_stream / wb_stream: null stream");
    if (m->graph_exec) return mfail(m, DC_ESTATE, "dw_stream / wb_stream: set before graph capture");
    cudaStream_t sv = reinterpret_cast<cudaStream_t>(static_cast<intptr_t>(value));
    cudaStream_t& slot = key[0] == 'd' ? m->cs2 : m->wb_stream;
    bool& own = key[0] == 'd' ? m->cs2_own : m->wb_own;
    if (slot && own) {
      cudaStreamSynchronize(slot);
      cudaStreamDestroy(slot);
    }
    slot = sv;
    own = false;
    return DC_OK;
  }
  if (!strcmp(key, "side_adam")) {
    if (value && ctx_world(m->ctx) != 1) return mfail(m, DC_EINVAL, "side_adam needs N == 1");
    if (value && m->E) return mfail(m, DC_EINVAL, "side_adam: Llama-shaped layers only");
    m->side_adam = value != 0;
    return DC_OK;
  }
  if (!strcmp(key, "comm_sms")) {
    if (value < 0 || value > 64) return mfail(m, DC_EINVAL, "comm_sms in [0, 64]");
    if (value && (ctx_flags(m->ctx) & DC_VIRTUAL_RANKS) && ctx_world(m->ctx) > 1)
      return mfail(m, DC_EINVAL, "comm_sms needs one rank per GPU");
    if (m->part.ctx_gemm && value != m->comm_sms) sm_partition_destroy(&m->part);
    m->comm_sms = (int)value;
    return DC_OK;
  }
  if (!strcmp(key, "dw_concurrent")) {
    m->dw_conc = value != 0;
    return DC_OK;
  }
  if (!strcmp(key, "offload_all_sync")) {
    if (m->host_states) return mfail(m, DC_ESTATE, "offload_all_sync must be set before dc_model_bind_host_states");
    m->offload_all_sync = value != 0;
    return DC_OK;
  }
  if (!strcmp(key, "fuse_act")) {
    if (value < 0 || value > 3) return mfail(m, DC_EINVAL, "fuse_act in [0, 3] (bit 0 forward, bit 1 backward)");
    m->fuse_act = (int)value;
    return DC_OK;
  }
  if (!strcmp(key, "rs_overlap")) {
    m->rs_overlap = value != 0;
    return DC_OK;
  }
  if (!strcmp(key, "stream_k")) {
    if (value && (ctx_flags(m->ctx) & DC_VIRTUAL_RANKS) && ctx_world(m->ctx) > 1)
      return mfail(m, DC_EINVAL, "stream_k needs one rank per GPU");
    m->stream_k = value != 0;
    return DC_OK;
  }
  if (!strcmp(key, "fused_adam")) {
    if (value && ctx_world(m->ctx) != 1) return mfail(m, DC_EINVAL, "fused_adam needs N == 1");
    if (value && m->E) return mfail(m, DC_EINVAL, "fused_adam: Llama-shaped layers only");
    m->fused_adam = value != 0;
    return DC_OK;
  }
  return mfail(m, DC_EINVAL, std::string("dc_model_set_option: unknown key ") + key);
}

// ------------------------------------------------------------------ host-resident states (D28)
namespace {
struct HostPlan {
  std::vector<int> slot_of;      // per fragment: ring slot, -1 = resident on the device
  int n_slots = 0;
  int64_t slot_elems = 0, m_first = 0, v_first = 0;
};
}  // namespace

static dc_status host_plan(dc_model* m, HostPlan* hp, int avail_slots = 0) {
  const dc_schedule* sc = ctx_sched(m->ctx);
  if (!sc) return mfail(m, DC_ESTATE, "host states: no schedule bound");
  if (m->n_micro != 1) return mfail(m, DC_ESTATE, "host states: gradient accumulation (micro_steps > 1) unsupported");
  const Layout& L = ctx_layout(m->ctx);
  const int nf = ctx_num_frags(m->ctx);
  hp->slot_of.assign(nf, -1);
  std::vector<char> off(nf, 0);
  const int nops = sched_num_ops(sc);
  for (int i = 0; i < nops; ++i) {
    int kind, id, nm, np, nw;
    const int64_t* mem; const int* posts; const int* waits;
    int64_t ao, bytes;
    sched_op(sc, i, &kind, &id, &mem, &nm, &ao, &bytes, &posts, &np, &waits, &nw);
    if (kind == K_OFF) {
      if (mem[0] < 0 || mem[0] >= nf) return mfail(m, DC_EINVAL, "host states: plan fragment id out of range");
      off[mem[0]] = 1;
    }
  }
  if (m->offload_all_sync) {
    if (nf == 0) return mfail(m, DC_EINVAL, "offload_all_sync: call dc_offload_fragments first");
    std::fill(off.begin(), off.end(), (char)1);
  }
  // whole (layer, state) fragments forming a prefix per state
  auto lay_lo = [&](int l) { return L.store_off[L.layer_first[l]]; };
  auto lay_n = [&](int l) {
    int64_t e = 0;
    for (int p = L.layer_first[l]; p < L.layer_first[l] + L.layer_count[l]; ++p) e += L.S[p];
    return e;
  };
  std::vector<int> n_off(2, 0);
  std::vector<std::vector<char>> lay_off(2, std::vector<char>(L.n_layers, 0));
  for (int f = 0; f < nf; ++f) {
    if (!off[f]) continue;
    int layer, state;
    int64_t o, elems;
    ctx_frag(m->ctx, f, &layer, &state, &o, &elems);
    if (o != lay_lo(layer) || elems != lay_n(layer))
      return mfail(m, DC_EINVAL, "host states: offloaded fragments must be whole (layer, state) slices "
                                 "(dc_offload_fragments with max bytes >= a layer's state)");
    lay_off[state][layer] = 1;
    hp->slot_elems = std::max(hp->slot_elems, (elems + 63) / 64 * 64);
  }
  for (int st = 0; st < 2; ++st) {
    int a = 0;
    while (a < L.n_layers && lay_off[st][a]) ++a;
    for (int l = a; l < L.n_layers; ++l)
      if (lay_off[st][l]) return mfail(m, DC_EINVAL, "host states: offloaded layers must be a prefix per state");
    n_off[st] = a;
  }
  hp->m_first = n_off[0] < L.n_layers ? lay_lo(n_off[0]) : L.shard_elems;
  hp->v_first = n_off[1] < L.n_layers ? lay_lo(n_off[1]) : L.shard_elems;
  // ring slots in schedule order: a reload takes a free slot, the write-back
  // after its layer's RS returns it.  Minimal pool: the lowest free slot.
  // With more slots than the minimum: the least recently freed one, so a
  // reload does not wait for the write-back just issued (PCIe full duplex)
  auto assign = [&](int n_fifo) -> dc_status {
    std::vector<char> busy;
    std::vector<int> fifo;
    for (int q = 0; q < n_fifo; ++q) fifo.push_back(q);
    hp->slot_of.assign(nf, -1);
    for (int i = 0; i < nops; ++i) {
      int kind, id, nm, np, nw;
      const int64_t* mem; const int* posts; const int* waits;
      int64_t ao, bytes;
      sched_op(sc, i, &kind, &id, &mem, &nm, &ao, &bytes, &posts, &np, &waits, &nw);
      // offload_all_sync: a layer's fragments are reloaded at its RS op
      std::vector<int> take;
      if (kind == K_RELOAD && off[mem[0]] && !m->offload_all_sync) take.push_back((int)mem[0]);
      if (kind == K_RS && m->offload_all_sync) {
        const int layer = m->s0[id].layer;
        for (int f = 0; f < nf; ++f) {
          int fl, fs;
          int64_t o, e;
          ctx_frag(m->ctx, f, &fl, &fs, &o, &e);
          if (fl == layer) take.push_back(f);
        }
      }
      for (int f : take) {
        int sl = 0;
        if (n_fifo) {
          if (fifo.empty()) return mfail(m, DC_EOOM, "host states: pool slots exhausted");
          sl = fifo.front();
          fifo.erase(fifo.begin());
        } else {
          while (sl < (int)busy.size() && busy[sl]) ++sl;
          if (sl == (int)busy.size()) busy.push_back(0);
          busy[sl] = 1;
        }
        hp->slot_of[f] = sl;
      }
      if (kind == K_RS) {
        const int layer = m->s0[id].layer;
        for (int f = 0; f < nf; ++f) {
          int fl, fs;
          int64_t o, e;
          ctx_frag(m->ctx, f, &fl, &fs, &o, &e);
          if (off[f] && fl == layer) {
            if (hp->slot_of[f] < 0) return mfail(m, DC_EINVAL, "host states: fragment updated before its reload");
            if (n_fifo) fifo.push_back(hp->slot_of[f]);
            else busy[hp->slot_of[f]] = 0;
          }
        }
      }
    }
    for (int f = 0; f < nf; ++f)
      if (off[f] && hp->slot_of[f] < 0) return mfail(m, DC_EINVAL, "host states: offloaded fragment never reloaded");
    hp->n_slots = n_fifo ? n_fifo : (int)busy.size();
    return DC_OK;
  };
  dc_status s = assign(0);
  if (s == DC_OK && avail_slots > hp->n_slots) s = assign(avail_slots);
  return s;
}

extern "C" dc_status dc_model_host_states_query(dc_model* m, int64_t* m_first, int64_t* v_first, uint64_t* pool_bytes,
                                                uint64_t* host_bytes) {
  if (!m || !m_first || !v_first || !pool_bytes || !host_bytes)
    return mfail(nullptr, DC_EINVAL, "dc_model_host_states_query: null");
  HostPlan hp;
  dc_status s = host_plan(m, &hp);
  if (s != DC_OK) return s;
  *host_bytes = 0;
  for (int f = 0; f < (int)hp.slot_of.size(); ++f)
    if (hp.slot_of[f] >= 0) *host_bytes = std::max<uint64_t>(*host_bytes, ctx_frag_host_end(m->ctx, f));
  *m_first = hp.m_first;
  *v_first = hp.v_first;
  *pool_bytes = (uint64_t)hp.n_slots * hp.slot_elems * 4;
  return DC_OK;
}

extern "C" dc_status dc_model_bind_host_states(dc_model* m, float* m_dev, float* v_dev, void* pool, uint64_t pool_bytes,
                                               void* host_pinned, uint64_t host_bytes) {
  if (!m) return mfail(nullptr, DC_EINVAL, "dc_model_bind_host_states: null model");
  HostPlan hp;
  dc_status s = host_plan(m, &hp);
  if (s != DC_OK) return s;
  const Layout& L = ctx_layout(m->ctx);
  uint64_t need = (uint64_t)hp.n_slots * hp.slot_elems * 4;
  if (need && pool_bytes / (hp.slot_elems * 4) > (uint64_t)hp.n_slots) {   // extra slots given: use them
    s = host_plan(m, &hp, (int)std::min<uint64_t>(pool_bytes / (hp.slot_elems * 4), 1 << 20));
    if (s != DC_OK) return s;
    need = (uint64_t)hp.n_slots * hp.slot_elems * 4;
  }
  if (pool_bytes < need || (need && !pool)) return mfail(m, DC_EOOM, "dc_model_bind_host_states: pool too small");
  if ((hp.m_first < L.shard_elems && !m_dev) || (hp.v_first < L.shard_elems && !v_dev))
    return mfail(m, DC_EINVAL, "dc_model_bind_host_states: null state array");
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (!al16(m_dev) || !al16(v_dev) || !al16(pool)) return mfail(m, DC_EINVAL, "dc_model_bind_host_states: alignment");
  const int nf = ctx_num_frags(m->ctx);
  std::vector<float*> slot(nf, nullptr);
  m->wb_frags.assign(L.n_layers, {});
  if (!m->wb_stream && cudaStreamCreateWithFlags(&m->wb_stream, cudaStreamNonBlocking) != cudaSuccess)
    return mfail(m, DC_ECUDA, "dc_model_bind_host_states: stream creation failed");
  for (auto& e : m->wb_ev) cudaEventDestroy(e);
  m->wb_ev.assign(nf, nullptr);
  for (auto& e : m->wb_ev)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
      return mfail(m, DC_ECUDA, "dc_model_bind_host_states: event creation failed");
  m->frag_slot = hp.slot_of;
  for (int f = 0; f < nf; ++f) {
    if (hp.slot_of[f] < 0) continue;
    slot[f] = reinterpret_cast<float*>(pool) + (int64_t)hp.slot_of[f] * hp.slot_elems;
    int layer, state;
    int64_t o, e;
    ctx_frag(m->ctx, f, &layer, &state, &o, &e);
    m->wb_frags[layer].push_back(f);
  }
  s = ctx_bind_host_states(m->ctx, m_dev, hp.m_first, v_dev, hp.v_first, slot, host_pinned, host_bytes);
  if (s != DC_OK) return mfail(m, s, dc_last_error(m->ctx));
  m->host_states = need > 0;
  return DC_OK;
}

// ------------------------------------------------------------------ CUDA graph of a step (N = 1)
extern "C" dc_status dc_model_graph_capture(dc_model* m, int32_t step_t, cudaStream_t ucs, cudaStream_t ags,
                                            cudaStream_t rss, cudaStream_t cps) {
  if (!m || !m->act) return mfail(m, DC_ESTATE, "dc_model_graph_capture: model not bound");
  if (!ctx_graph_mode(m->ctx)) return mfail(m, DC_ESTATE, "dc_model_graph_capture: set dc_set_option(graph_mode) first");
  const dc_schedule* sc = ctx_sched(m->ctx);
  if (!sc) return mfail(m, DC_ESTATE, "dc_model_graph_capture: no schedule bound");
  for (int i = 0, n = sched_num_ops(sc); i < n; ++i) {
    int kind, id, nm, np, nw;
    const int64_t* mem; const int* posts; const int* waits;
    int64_t off, bytes;
    sched_op(sc, i, &kind, &id, &mem, &nm, &off, &bytes, &posts, &np, &waits, &nw);
    if (kind >= K_OFF) return mfail(m, DC_EINVAL, "dc_model_graph_capture: offload schedules are not captured");
  }
  if (m->host_states || m->side_adam || m->fused_adam || m->comm_sms > 0)
    return mfail(m, DC_EINVAL, "dc_model_graph_capture: host states / side / fused Adam / SM partition unsupported");
  // at N = 1 no node may wait on another branch of the graph (branches can
  // share a hardware queue): the reduce-scatter runs in compute-stream order
  if (ctx_world(m->ctx) == 1 && m->rs_overlap)
    return mfail(m, DC_EINVAL, "dc_model_graph_capture: set rs_overlap 0 at N = 1");
  if (m->graph_exec) { cudaGraphExecDestroy(m->graph_exec); m->graph_exec = nullptr; }
  if (m->graph) { cudaGraphDestroy(m->graph); m->graph = nullptr; }
  if (cudaStreamBeginCapture(ucs, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
    return mfail(m, DC_ECUDA, "dc_model_graph_capture: begin capture failed");
  m->capturing = true;
  dc_status s = dc_model_step(m, step_t, 2, ucs, ags, rss, cps);   // with per-op event nodes
  m->capturing = false;
  cudaGraph_t g = nullptr;
  const cudaError_t e = cudaStreamEndCapture(ucs, &g);
  if (s != DC_OK) { if (g) cudaGraphDestroy(g); return s; }
  if (e != cudaSuccess || !g) return mfail(m, DC_ECUDA, std::string("dc_model_graph_capture: ") + cudaGetErrorString(e));
  if (cudaGraphInstantiate(&m->graph_exec, g, 0) != cudaSuccess) {
    cudaGraphDestroy(g);
    return mfail(m, DC_ECUDA, "dc_model_graph_capture: instantiate failed");
  }
  m->graph = g;
  return DC_OK;
}

extern "C" dc_status dc_model_graph_launch(dc_model* m, int32_t step_t, cudaStream_t ucs) {
  if (!m || !m->graph_exec) return mfail(m, DC_ESTATE, "dc_model_graph_launch: no captured graph");
  if (step_t < 1) return mfail(m, DC_EINVAL, "dc_model_graph_launch: step_t is 1-based");
  dc_status s = dc_poll(m->ctx);
  if (s != DC_OK) return mfail(m, s, dc_last_error(m->ctx));
  if ((s = ctx_set_step_scalars(m->ctx, step_t, ucs)) != DC_OK) return mfail(m, s, dc_last_error(m->ctx));
  if (cudaGraphLaunch(m->graph_exec, ucs) != cudaSuccess) return mfail(m, DC_ECUDA, "dc_model_graph_launch: launch failed");
  m->profile_pending = true;          // the replay re-recorded the per-op events
  return DC_OK;
}

extern "C" dc_status dc_model_launch_count(const dc_model* m, int64_t* n) {
  if (!m || !n) return mfail(nullptr, DC_EINVAL, "dc_model_launch_count: null");
  *n = m->launches;
  return DC_OK;
}
