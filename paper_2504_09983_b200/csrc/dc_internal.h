// Internal declarations shared by the library's translation units.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/dc.h"

namespace dc {

void set_global_error(const std::string& s);
void count_launch();                 // increments the launch counter (per thread)
int64_t launch_count();
void reset_launch_count();

// Host-mapped error record of a context, written by a timed-out device flag
// wait (comm.cu spin_ge): [0] code (0 = no error; bits 8.. the waiting site,
// low bits the flag index), [1] claimed, [2] target, [3] last observed value,
// [4..5] flag address (lo, hi).
constexpr int ERR_RECORD_WORDS = 8;

#define DC_CUDA_TRY(expr, ctxerr)                                                   \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess) {                                                        \
      *(ctxerr) = std::string(#expr ": ") + cudaGetErrorString(_e);                 \
      return DC_ECUDA;                                                              \
    }                                                                               \
  } while (0)

struct Layout {
  std::vector<int64_t> S, store_off, goff;
  std::vector<int> layer_first, layer_count;
  int64_t shard_elems = 0, grad_slot_bytes = 0, flag_words = 0;
  int n_layers = 0;
  // flag table (uint32 words)
  int64_t f_ready = 0, f_done = 0, f_gready = 0, f_gcons = 0, f_rsdone = 0;
  int64_t f_chunk = 0;  // fused AG -> GEMM: [param][sender][AG_CHUNKS] chunk-landed values
  int64_t f_scal = 0;   // 2 words: this step's Adam scalars (s, c) as fp32 (graph mode)
  int64_t f_dep = 0;    // graph mode: device step counter (local, monotone)
  int64_t f_bar = 0;    // graph mode: 2 x world barrier words (rounds A, B; one per source rank)
};

struct dc_ctx_fwd;
const Layout& ctx_layout(const dc_ctx* c);
int ctx_world(const dc_ctx* c);
int ctx_rank(const dc_ctx* c);
const dc_schedule* ctx_sched(const dc_ctx* c);
int64_t ctx_numel(const dc_ctx* c, int p);
int ctx_micro_steps(const dc_ctx* c);
void ctx_set_rs_ctas(dc_ctx* c, int ctas);   // 0 = default (2 per SM of the device)

// spatial SM partition (green contexts, sm_partition.cpp)
struct SmPartition {
  int gemm_sms = 0, comm_sms = 0;
  cudaStream_t compute = nullptr, rs = nullptr, ag = nullptr;
  void* ctx_gemm = nullptr;
  void* ctx_comm = nullptr;
};
dc_status sm_partition_create(int device, int comm_sms, SmPartition* out, std::string* err);
void sm_partition_destroy(SmPartition* p);
uint32_t ctx_flags(const dc_ctx* c);
int sched_num_ops(const dc_schedule* s);
void sched_op(const dc_schedule* s, int i, int* kind, int* id, const int64_t** members, int* nmem,
              int64_t* arena_off, int64_t* bytes, const int** posts, int* nposts, const int** waits, int* nwaits);
enum { K_COMPUTE, K_AG, K_REL, K_RS, K_OFF, K_OFFSYNC, K_RELOAD, K_RELOADSYNC };

// Fused reduce-scatter + Adam epilogue (N = 1): the GEMM's C[row, col] is the
// gradient of element row * N + col of one parameter.
struct EpiAdam {
  float* master;
  float* m;
  float* v;
  void* shard;
  float w1, w2, b2, neg_s, c, eps;
};
// GEMM side job: groups [g0, g1) of 8 elements over a layer's params
// (concatenated in order; member i spans groups [cum[i], cum[i+1]))
struct SideJob {
  int nm;
  int64_t cum[10];
  int64_t goff[9];          // byte offset of member i's grads in `slot`
  int64_t store_off[9];     // member i's offset in the shard store
  const uint8_t* slot;
  float* master;
  float* m;
  float* v;
  __nv_bfloat16* shard;
  float w1, w2, b2, neg_s, c, eps;
  int64_t g0, g1;
};
dc_status launch_gemm(const dc_gemm_args* g, cudaStream_t stream, std::string* err,
                      const EpiAdam* adam = nullptr, const SideJob* side = nullptr);
// the reduce-scatter + Adam of `layer` as a side job template (N = 1 only);
// and the consumed-flag post that normally ends rs_adam
dc_status ctx_side_job(dc_ctx* c, int layer, int step_t, SideJob* out);
dc_status ctx_post_consumed(dc_ctx* c, int layer, cudaStream_t st);
// Adam scalars of step t from the ctx hyper-parameters (reading D18)
void ctx_adam_scalars(const dc_ctx* c, int step_t, EpiAdam* out);
// shard-store pointers of a param (fp32 master/m/v, bf16 shard) on this rank
void ctx_param_state(const dc_ctx* c, int param, float** master, float** m, float** v, void** shard);
// offload fragments (dc_offload_fragments) and the host-resident state bind
// (reading D28): frag_slot[i] = device ring slot of offloaded fragment i, or null
int ctx_num_frags(const dc_ctx* c);
void ctx_frag(const dc_ctx* c, int i, int* layer, int* state, int64_t* off, int64_t* elems);
dc_status ctx_bind_host_states(dc_ctx* c, float* m_dev, int64_t m_first, float* v_dev, int64_t v_first,
                               const std::vector<float*>& frag_slot, void* host_pinned, uint64_t host_bytes);
uint64_t ctx_frag_host_end(const dc_ctx* c, int i);   // pinned host byte offset after fragment i
// one-shot timing of the next dc_gather (profiling): `start` is recorded once
// every receiver is ready (after the ready-flag wait), `end` once every
// sender's stores have landed here (after the done-counter wait)
void ctx_set_gather_timing(dc_ctx* c, cudaEvent_t start, cudaEvent_t end);
// graph mode (N = 1): per-step counter reset and the step's Adam scalars
bool ctx_graph_mode(const dc_ctx* c);
dc_status ctx_set_step_scalars(dc_ctx* c, int step_t, cudaStream_t st);
// dc_reduce_scatter_step restricted to a subset of the layer's params
dc_status reduce_scatter_params(dc_ctx* c, int layer, int step_t, int micro, const std::vector<int>& params,
                                cudaStream_t st);

// ------------------------------------------------------------------ kernels
// glue.cu
void k_init_param(uint64_t seed, int32_t tensor_id, int64_t numel, int32_t world, int32_t rank,
                  int64_t S, float k, float* master, void* shard, cudaStream_t st);
void k_rmsnorm_fwd(const void* x, const void* g, void* h, float* rstd, int T, int H, cudaStream_t st);
// dg_partial: rmsnorm_bwd_ws_floats(T, H) floats of scratch; returns the number of
// H-float partial rows written at its start (input of k_colsum_to_bf16)
int k_rmsnorm_bwd(const void* dh, const void* x, const void* g, const float* rstd, const void* dres,
                  void* dx, float* dg_partial, int T, int H, cudaStream_t st);
int rmsnorm_bwd_blocks(int T);
int64_t rmsnorm_bwd_ws_floats(int T, int H);
void k_colsum_to_bf16(const float* partial, int nblk, int H, void* out, cudaStream_t st);
void k_attn_mix_fwd(const void* qkv, void* a, int T, int qd, int kvd, int hd, int grp, cudaStream_t st);
void k_attn_mix_bwd(void* dqkv, const void* qkv, int T, int qd, int kvd, int hd, int grp, cudaStream_t st);
void k_act_fwd(const void* gu, void* act, int T, int F, cudaStream_t st);
void k_act_bwd(const void* dact, const void* gu, void* dgu, int T, int F, cudaStream_t st);
void k_loss(const void* y, const void* t, void* dy, float* partial, float* loss, int64_t n, cudaStream_t st);
void k_zero(void* p, int64_t bytes, cudaStream_t st);
// moe.cu: Mixtral-shaped MoE MLP glue (fixed balanced top-2 routing)
void k_moe_router_fwd(const void* h2, const void* wr, float* g01, int T, int H, int E, cudaStream_t st);
void k_moe_gather(const void* h2, void* X, int T, int H, int E, cudaStream_t st);
void k_moe_combine(const void* x2, const void* O, const float* g01, void* y, int T, int H, int E, cudaStream_t st);
void k_moe_combine_bwd(const void* dy, const void* O, const float* g01, void* dO, float* dl0, int T, int H, int E,
                       cudaStream_t st);
void k_moe_router_bwd(const void* dX, const float* dl0, const void* wr, const void* h2, void* dh2, float* part,
                      int T, int H, int E, cudaStream_t st);
int moe_router_dw_blocks(int T);
cudaError_t preload_moe_kernels();
// force-load every kernel of the library (lazy module loading at first launch
// can block behind another rank's spinning flag wait on the same GPU)
cudaError_t preload_glue_kernels();
cudaError_t preload_comm_kernels();
cudaError_t preload_gemm_kernels();

// comm.cu
constexpr int MAXW = 8;                       // max ranks on one NVSwitch box
// fused all-gather -> GEMM: a sender's shard of a param is
// pushed in at most AG_CHUNKS chunks of >= AG_CHUNK_MIN elements (multiples of
// 8); after a chunk's stores land on every receiver the sender writes the
// gather's value into chunk[param][sender][j] of every receiver's flag table.
constexpr int AG_CHUNKS = 64;
constexpr int64_t AG_CHUNK_MIN = 4096;
inline int64_t ag_chunk_elems(int64_t S) {
  int64_t e = (S + AG_CHUNKS - 1) / AG_CHUNKS;
  e = (e + 7) / 8 * 8;
  return e < AG_CHUNK_MIN ? AG_CHUNK_MIN : e;
}
// the consumer side: wait until every chunk overlapping flat elements
// [e0, e1) of a gathered tensor carries `value` (GemmParams / dc_gemm_args)
struct ChunkWait {
  const uint32_t* flags = nullptr;   // &chunk[param][0][0] in this rank's table
  int64_t S = 0, E = 0;              // shard elements, chunk elements
  uint32_t value = 0;
};
bool ctx_fused_ag(const dc_ctx* c);      // option fused_ag at N > 1 (SM push gathers)
bool ctx_virtual(const dc_ctx* c);
void ctx_wait_err(dc_ctx* c, uint32_t** err, uint64_t* timeout_ns);
// the chunk wait of member `param` of gather `gid` issued in the current step
bool ctx_chunk_wait(const dc_ctx* c, int gid, int param, ChunkWait* out);
struct PeerFlags { uint32_t* p[MAXW]; int n; };
struct AgMember {
  const void* src; int64_t dst_off_bytes; int64_t bytes;
  int64_t chunk_word = -1;   // fused AG -> GEMM: word of chunk[param][rank][0] in every table (-1: off)
  uint32_t chunk_value = 0;
};
struct RsMember {
  int64_t goff_bytes;      // member's padded full tensor inside the grad slot
  int64_t S;               // shard elements
  int64_t store_off;       // member's shard offset in the per-rank store
};
dc_status k_ag_push(const std::vector<AgMember>& mem, int world, int rank, const uint64_t* arena_peers,
                    const uint32_t* ready_local, uint32_t epoch, PeerFlags done_peers,
                    const uint32_t* done_local, uint32_t done_target, int ctas, uint64_t timeout_ns,
                    uint32_t* err_flag, cudaStream_t st, cudaEvent_t ev_after_ready = nullptr,
                    bool skip_waits = false, uint32_t delay_us = 0, const uint64_t* flag_peers = nullptr,
                    bool bulk = false);
dc_status k_rs_adam(const std::vector<RsMember>& mem, int world, int rank, const uint64_t* slot_peers,
                    const uint32_t* ready_local, uint32_t ready_target, PeerFlags consumed_peers,
                    uint32_t consumed_value, uint32_t* done_ctr, uint32_t done_target, float* master,
                    float* m, float* v, void* shard, float* acc, int mode, int micro_steps, float s, float c,
                    double beta1, double beta2, double eps, int ctas, int threads, uint64_t timeout_ns,
                    uint32_t* err_flag, cudaStream_t st, const float* dev_scalars = nullptr, bool bulk = false);
constexpr int RS_BULK_CHUNK = 2048;   // elements per chunk of the bulk-copy rs_adam (comm.cu RSB_CH)
int rs_bulk_ctas_per_sm();             // its resident CTAs per SM (grid = SMs x this)
// graph mode: write (s, c) of a step into the flag-table words the rs_adam
// launches read, and reset a stream's stream-K flags / epochs
void k_set_scalars(float* dst, float s, float c, cudaStream_t st);
// device-epoch barrier pieces (graph mode at N > 1): ++*dep; peers' word = *dep;
// wait until every word of mine >= *dep
void k_inc_dev(uint32_t* dep, cudaStream_t st);
void k_post_dev(PeerFlags dst, const uint32_t* dep, cudaStream_t st);
void k_wait_dev(const uint32_t* flags, int n, const uint32_t* dep, uint64_t timeout_ns, uint32_t* err_flag,
                cudaStream_t st);
// event record that survives CUDA-graph capture (an external record node)
void record_event(cudaEvent_t ev, cudaStream_t st);
void gemm_sk_reset(void* workspace, cudaStream_t st);   // graph mode: flags cleared, epoch 0
uint64_t gemm_workspace_bytes();
// reduce-scatter modes (gradient accumulation)
enum { RS_UPDATE = 0, RS_FIRST = 1, RS_ADD = 2, RS_FINAL = 3 };
dc_status k_ag_copy(const std::vector<AgMember>& mem, int world, const uint64_t* arena_peers,
                    const uint32_t* ready_local, uint32_t epoch, PeerFlags done_peers, const uint32_t* done_local,
                    uint32_t done_target, uint64_t timeout_ns, uint32_t* err_flag, cudaStream_t st,
                    cudaEvent_t ev_after_ready);
void k_post_flags(PeerFlags dst, uint32_t value, cudaStream_t st);
void k_delay(uint32_t us, cudaStream_t st);   // one-thread spin on globaltimer (testing)
// nvls.cu: multicast all-gather (one multimem.st per 16 B,
// the switch replicates) and multimem.ld_reduce reduce-scatter + Adam
dc_status k_ag_multimem(const std::vector<AgMember>& mem, uint8_t* arena_mc, uint32_t* done_mc, int ctas,
                        const uint32_t* ready_local, int world, uint32_t epoch, const uint32_t* done_local,
                        uint32_t done_target, uint64_t timeout_ns, uint32_t* err_flag, cudaStream_t st,
                        cudaEvent_t ev_after_ready);
dc_status k_rs_adam_nvls(const std::vector<RsMember>& mem, int world, int rank, const uint8_t* slot_mc,
                         const uint32_t* ready_local, uint32_t ready_target, PeerFlags consumed_peers,
                         uint32_t consumed_value, uint32_t* done_ctr, uint32_t done_target, float* master, float* m,
                         float* v, void* shard, float* acc, int mode, int micro_steps, float s, float c, double beta1,
                         double beta2, double eps, int ctas, uint64_t timeout_ns, uint32_t* err_flag, cudaStream_t st,
                         const float* dev_scalars);
cudaError_t preload_nvls_kernels();
void k_wait_flags(const uint32_t* flags, int n, uint32_t target, uint64_t timeout_ns,
                  uint32_t* err_flag, cudaStream_t st);

}  // namespace dc
