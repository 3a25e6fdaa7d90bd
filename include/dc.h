/*
 * dc.h — C ABI of the B200-native sharded-parameter hot path of DeepCompile
 * (Tanaka et al., arxiv 2504.09983).  Citations: P:n = line n of PAPER.md.
 *
 * The life cycle of a sharded parameter (§4.1): all-gather the shards
 * into an unsharded buffer before a layer's forward and backward (dc_gather),
 * release the buffer after its last use (dc_release), reduce-scatter the
 * gradient fused with the 1/N scale and a partitioned Adam update of the local
 * shard (dc_reduce_scatter_step, P:127/P:440/P:504), under the profile-guided
 * schedule of §4.2-§4.4 (dc_plan) with optimizer-state offload (dc_offload,
 * P:370-408).
 *
 * Conventions (every function):
 *  - returns dc_status; no C++ exception crosses the ABI;
 *  - on error, dc_last_error(ctx) (or dc_last_error(NULL) for ctx-less calls)
 *    returns a message owned by the library, valid until the next call on the
 *    same thread;
 *  - the CALLER owns all device and pinned-host memory (torch allocates it);
 *    the library keeps non-owning pointers until dc_destroy and never
 *    cudaMalloc's.  The library owns dc_ctx, dc_schedule, dc_model and strings;
 *  - enqueue calls are asynchronous on the given stream(s); a CUDA launch error
 *    returns DC_ECUDA immediately; a device-side flag-wait timeout sets a sticky
 *    error that the next call on the ctx returns (DC_ETIMEOUT);
 *  - a ctx is single-threaded (one per rank / virtual rank).
 */
#ifndef DC_H
#define DC_H

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DC_OK = 0,
  DC_EINVAL = 1,       /* bad argument / layout                              */
  DC_EOOM = 2,         /* a caller-provided buffer is too small              */
  DC_EINFEASIBLE = 3,  /* memory limit cannot be met (SPEC Infeasible*)      */
  DC_ECUDA = 4,        /* CUDA runtime / launch error                         */
  DC_ESTATE = 5,       /* call out of order (e.g. step before a schedule)     */
  DC_EPROFILE = 6,     /* profile is not an S_0 schedule (ProfileMismatch)    */
  DC_ETIMEOUT = 7      /* a device-side flag wait exceeded its bound          */
} dc_status;

enum { DC_BF16 = 0, DC_FP32 = 1 };
enum { DC_INIT_WEIGHTS = 1u, DC_VIRTUAL_RANKS = 2u, DC_DEBUG_POISON = 4u,
       DC_DEFER_STATES = 8u   /* exp_avg/exp_avg_sq may be NULL: bound later (dc_model_bind_host_states) */ };
enum { DC_PASS_SHARD = 1u, DC_PASS_PREFETCH = 2u, DC_PASS_UNSHARD = 4u, DC_PASS_OFFLOAD = 8u,
       DC_PASS_HOST_STATES = 16u  /* with OFFLOAD: reload rule for host-resident fragments (reading D28) */ };
enum { DC_D2H_START = 0, DC_D2H_SYNC_FREE = 1, DC_H2D_START = 2, DC_H2D_SYNC = 3,
       DC_WRITEBACK = 4       /* host-resident states: D2H of the updated fragment */ };

typedef struct dc_ctx dc_ctx;
typedef struct dc_schedule dc_schedule;
typedef struct dc_model dc_model;

const char* dc_last_error(const dc_ctx* ctx);
const char* dc_version(void);

/* ------------------------------------------------------------------------
 * Shard layout ("each parameter tensor is evenly partitioned").
 * S_i = ceil(numel_i / (8 N)) * 8 elements; rank r owns elements
 * [r S_i, (r+1) S_i) of the zero-padded flat tensor.  The per-rank shard store
 * concatenates the S_i in param order (offsets are multiples of 8 elements =
 * 16 B for bf16).  The grad slot of a layer holds each of its params as N*S_i
 * bf16 elements (padded full tensor) in param order, 256-byte aligned.
 * ------------------------------------------------------------------------ */
typedef struct {
  int32_t world;                 /* N >= 1                                     */
  int32_t n_params;
  const int64_t* numel;          /* [n_params] in S_0 first-use order          */
  const int32_t* layer_of;       /* [n_params] non-decreasing                  */
  int32_t max_s0_ops;            /* upper bound on S_0 op ids (flag table)     */
} dc_layout_args;

typedef struct {
  int64_t shard_elems;           /* sum S_i: length of every per-rank store    */
  int64_t grad_slot_bytes;       /* max over layers of the layer's grad slot   */
  int64_t flag_bytes;            /* uint32 flag table per rank                 */
  int32_t n_layers;
} dc_layout;

/* Pure host function: sizes the caller must allocate before dc_init. */
dc_status dc_layout_query(const dc_layout_args* a, dc_layout* out);

/* ------------------------------------------------------------------------
 * Context.  Pointers are device pointers unless noted; "peer" tables hold the
 * same buffer as mapped on every rank (torch symmetric memory buffer_ptrs at
 * N>1; in DC_VIRTUAL_RANKS mode, the N virtual ranks' buffers on one GPU).
 * ------------------------------------------------------------------------ */
typedef struct {
  int32_t rank, world, device;
  int32_t n_params;
  const int64_t* numel;          /* host [n_params]                            */
  const int32_t* layer_of;       /* host [n_params]                            */
  const float* init_k;           /* host [n_params] generator scale; 0 -> 1.0  */
  int32_t max_s0_ops;
  void* shard_param;             /* bf16 [shard_elems], caller-owned           */
  float* master;                 /* fp32 [shard_elems]                         */
  float* exp_avg;                /* fp32 [shard_elems]  (Adam m)               */
  float* exp_avg_sq;             /* fp32 [shard_elems]  (Adam v)               */
  const uint64_t* grad_peer_ptrs;  /* host [world]: 2 grad slots per rank,    */
  uint64_t grad_bytes;             /*   each dc_layout.grad_slot_bytes        */
  const uint64_t* flag_peer_ptrs;  /* host [world]: uint32 flag tables        */
  uint64_t flag_bytes;
  void* host_pinned;             /* pinned host memory for offload (may be 0) */
  uint64_t host_pinned_bytes;
  double lr, beta1, beta2, eps;  /* Adam; weight decay 0; host scalars  */
  uint64_t seed;                 /* generator seed (synth/gen.py recipe)       */
  uint32_t flags;                /* DC_INIT_WEIGHTS | DC_VIRTUAL_RANKS | ...   */
  uint32_t spin_limit;           /* flag-wait bound in ms, 0 = 20000           */
  int32_t micro_steps;           /* n gradient-accumulation micro-steps per    */
                                 /*   optimizer step; 0 -> 1          */
  float* grad_acc;               /* fp32 [shard_elems], caller-owned; required */
                                 /*   when micro_steps > 1, else may be NULL   */
} dc_init_args;

/* Validates, computes the layout, zeroes m/v (not with DC_DEFER_STATES: then
 * exp_avg / exp_avg_sq may be NULL until dc_model_bind_host_states, and a
 * reduce-scatter before that is DC_ESTATE) and (with DC_INIT_WEIGHTS) fills
 * master = value(seed, param, idx) and shard = RNE_bf16(master) with the
 * counter-based generator on the device (synchronous). */
dc_status dc_init(const dc_init_args* a, dc_ctx** out);
dc_status dc_destroy(dc_ctx* ctx);
/* Non-blocking check of the sticky device error word (DC_ETIMEOUT if any flag
 * wait of this ctx timed out since dc_init); DC_OK otherwise. */
dc_status dc_poll(dc_ctx* ctx);

/* Offset (elements) of param's shard in the store, and S_i. */
dc_status dc_shard_range(const dc_ctx* ctx, int32_t param, int64_t* offset, int64_t* shard_elems);
/* Byte offset of param inside its layer's grad slot (padded, N*S_i bf16). */
dc_status dc_grad_offset(const dc_ctx* ctx, int32_t param, int64_t* byte_offset);

/* ------------------------------------------------------------------------
 * Planner.  Host-only, deterministic, exact integer arithmetic;
 * no CUDA calls.  profile_json: the S_0 schedule with per-op p_mem (bytes
 * resident before the op, excluding Adam m and v), transient, dur_us, plus
 * params {id, bytes}, frags {id, layer, bytes} and the T_c table (schema:
 * DESIGN.md §11).  mem_budget = M.  Output: dc_schedule (immutable).
 * Errors: DC_EPROFILE (not an S_0 / malformed), DC_EINFEASIBLE.
 * ------------------------------------------------------------------------ */
typedef struct {
  uint64_t M_prefetch;             /* default 2 GiB                    */
  uint32_t alpha_num, alpha_den;   /* default 3/2                      */
  uint32_t passes;                 /* DC_PASS_* bitmask; order fixed P->S->O   */
  uint32_t strict;                 /* reading D4                               */
} dc_plan_opts;

dc_status dc_plan(const char* profile_json, uint64_t mem_budget, const dc_plan_opts* opts,
                  dc_schedule** out);
/* Canonical JSON (keys sorted, no whitespace, integers only).  *len in/out:
 * buffer size in, bytes needed (without NUL) out; DC_EOOM if too small. */
dc_status dc_schedule_json(const dc_schedule* s, char* buf, size_t* len);
uint64_t dc_schedule_capacity(const dc_schedule* s);
void dc_schedule_free(dc_schedule* s);

/* Bind a schedule and the gather arena (peer table of a symmetric buffer of
 * >= dc_schedule_capacity bytes).  Zeroes this rank's flag table: every rank
 * must call it between the same two barriers.  Resets the epoch to 0. */
dc_status dc_bind_schedule(dc_ctx* ctx, const dc_schedule* s, const uint64_t* arena_peer_ptrs,
                           uint64_t arena_bytes, cudaStream_t stream);

/* Begin step `epoch` (1-based, monotone): posts the ready flags of gathers
 * whose arena interval has no earlier release in the step (reading D26). */
dc_status dc_step_begin(dc_ctx* ctx, int32_t epoch, cudaStream_t compute_stream);

/* ------------------------------------------------------------------------
 * Gather / release.  gather_id = the schedule op id of an "ag"
 * op (S_0 id of its first member).  ag_stream must already be ordered after
 * the compute-stream position of the op (issue semantics, reading D23).
 * Kernel ag_push: waits for the ready flag of every receiving rank, stores this
 * rank's shard of every member into every rank's arena at
 * arena_off(member) + rank * S_i * 2 bytes with 16-byte stores, fences, bumps
 * every receiver's done counter, then waits for its own N * CTAs arrivals.
 * At N = 1 the gathered tensor aliases the shard (no copy, no kernel).
 * done_evt (may be NULL) is recorded on ag_stream after the kernel.
 * ------------------------------------------------------------------------ */
dc_status dc_gather(dc_ctx* ctx, int32_t gather_id, cudaStream_t ag_stream, cudaEvent_t done_evt);
/* Profiling: the NEXT dc_gather (N > 1) records after_ready on ag_stream once
 * every receiver's ready flag was seen and after_done once every sender's
 * stores landed here (either may be NULL) — the transfer time T_c of P:305
 * without the wait for the receivers.  One-shot. */
dc_status dc_gather_timing(dc_ctx* ctx, cudaEvent_t after_ready, cudaEvent_t after_done);
/* Context options.  "graph_mode" (default 0; before dc_bind_schedule, else
 * DC_ESTATE): see dc_model_graph_capture.  "ag_copy_engine" (default 0): 1 issues every gather's
 * stores as cudaMemcpyAsync peer copies (copy engines; no SM time beside the
 * GEMMs) under the same ready / done flag protocol; bit-identical
 * gathered buffers.  Set before dc_bind_schedule (DC_ESTATE after).
 * "rs_bulk" (default 1 at N = 1, 0 at N > 1; any time): the reduce-scatter +
 * Adam of dc_reduce_scatter_step (update / final micro-step) runs as the
 * bulk-copy pipelined kernel (two CTAs of 544 threads and ~110 KB of shared
 * memory per SM) instead of the register-streaming one; bit-identical.
 * "ag_skip_waits" (profiling only, default 0): dc_gather launches the push
 * without its ready / done flag waits (for ncu, which serialises kernels);
 * the gathered buffer is then NOT guaranteed complete.
 * "nvls" (default 0, any time; SURVEY §8 f-3, P:438 collectives): bit 0 —
 * gathers store each shard vector ONCE with multimem.st to the arena's
 * multicast address (the NVSwitch replicates it into every rank's arena;
 * bit-identical buffers, same ready / done protocol, done bumped on every rank
 * by one multimem.red); bit 1 — the reduce-scatter reads slice r of every
 * rank's grads with one multimem.ld_reduce (fp32 accumulation in the switch,
 * bf16 result; NOT bit-exact with the ascending-rank fp32 sum) before 1/N and
 * Adam.  Each bit takes effect only while dc_bind_multicast holds the
 * corresponding multicast address; otherwise the unicast kernels run.
 * "fused_ag" (default 0; before dc_bind_schedule, else DC_ESTATE; SURVEY §8
 * f-4): N > 1 gathers by the SM push are stored chunk by chunk (<= 64
 * chunks of >= 4096 elements per shard) and, once a chunk's stores landed on
 * every receiver, the sender writes the gather's value into that chunk's word
 * of every receiver's flag table; dc_model_step's GEMMs that read a gathered
 * weight as their B operand then wait per tile for just the chunks they load
 * (dc_gemm_args.chunk_*) instead of the compute stream waiting for the whole
 * gather.  Bit-identical results.  With virtual ranks every rank's GEMMs get
 * 1/N of the SMs (co-residency on one GPU).
 * "ag_bulk" (default 0, any time): the SM push moves its data with the bulk-
 * copy (TMA) engine — one thread per CTA streams 8 KB pieces of the shard into
 * a 4-stage shared-memory ring (cp.async.bulk + mbarrier) and issues one bulk
 * store per receiver; same done protocol, bit-identical buffers (ignored for
 * fused_ag's chunked pushes).
 * "ag_delay_us" (testing, default 0): every push starts this long after its
 * ready wait (consumers then run ahead of the data).
 * "jitter_us" / "jitter_seed" (testing, default 0): random delays in
 * [0, jitter_us) before every push, every release's ready posts and every
 * reduce-scatter (a counter-based hash of seed, rank, op and step), so ranks
 * interleave differently at every op (race detection). */
dc_status dc_set_option(dc_ctx* ctx, const char* key, int64_t value);
/* Multicast (NVLS) addresses of this rank's symmetric buffers, as mapped by
 * the caller (torch symmetric memory's multicast_ptr): the gather arena bound
 * by the last dc_bind_schedule, the grad slots and the flag table of dc_init
 * (byte addresses of their first byte, 16 B aligned; 0 = not available).
 * dc_bind_schedule forgets arena_mc (a new arena), so call this after every
 * bind.  DC_ESTATE before the first dc_bind_schedule; DC_EINVAL for non-zero
 * addresses with N = 1 or virtual ranks, or arena / grad addresses without
 * the flag table's. */
dc_status dc_bind_multicast(dc_ctx* ctx, uint64_t arena_mc, uint64_t grad_mc, uint64_t flags_mc);
/* Unsharded tensor of param (row-major, numel elements; padding follows):
 * valid between its gather's completion and its release.  At N = 1 the
 * shard itself.  DC_ESTATE if the param is not gathered. */
dc_status dc_tensor_ptr(const dc_ctx* ctx, int32_t param, void** full_ptr);
/* Release op `release_id` (schedule op id): posts the ready flags listed in
 * its posts_ready_for to every peer, on compute_stream.  */
dc_status dc_release(dc_ctx* ctx, int32_t release_id, cudaStream_t compute_stream);

/* ------------------------------------------------------------------------
 * Gradient slot and reduce-scatter + Adam.
 * dc_grad_slot: where the dW GEMMs of `layer` write bf16 full grads; before the
 * first write of a backward the caller enqueues dc_grad_slot_acquire on the
 * compute stream (waits until every owner consumed the slot's previous use);
 * after the last write dc_grad_slot_publish (posts grad-ready to every owner).
 * dc_reduce_scatter_step, kernel rs_adam: for every param of `layer`, owner
 * r computes rs = (((+0 + g_0) + g_1) + ... + g_{N-1}) over fp32(bf16) slice r
 * of every rank's grad slot (peer loads); then, by micro-step `micro` in
 * [0, n) of the n = micro_steps of dc_init (gradient accumulation, P:362,
 * ZeRO-3 semantics P:478 — the accumulated gradient stays partitioned):
 *   n = 1:          g = rs * fp32(1/N), Adam
 *   micro = 0:      acc = rs                      (grad_acc shard, fp32)
 *   0 < micro < n-1: acc = acc + rs
 *   micro = n-1:    g = (acc + rs) * fp32(1/(N n)), Adam
 * Adam = step `step_t` (1-based) on master/m/v (fp32, the op order of reading
 * D18), shard = RNE_bf16(master).  Every mode then posts "consumed" to every
 * rank.  DC_EINVAL for micro outside [0, n).
 * ------------------------------------------------------------------------ */
dc_status dc_grad_slot(const dc_ctx* ctx, int32_t layer, void** grad_full_bf16);
dc_status dc_grad_slot_acquire(dc_ctx* ctx, int32_t layer, cudaStream_t compute_stream);
dc_status dc_grad_slot_publish(dc_ctx* ctx, int32_t layer, cudaStream_t compute_stream);
dc_status dc_reduce_scatter_step(dc_ctx* ctx, int32_t layer, int32_t step_t, int32_t micro,
                                 cudaStream_t rs_stream);

/* ------------------------------------------------------------------------
 * Offload: fragment f = a contiguous slice of the fp32 m or v
 * store (dc_offload_fragments).  op: DC_D2H_START (async cudaMemcpyAsync to
 * the pinned host slot on copy_stream), DC_D2H_SYNC_FREE (compute stream waits
 * for that copy; the device slice may then be reused), DC_H2D_START,
 * DC_H2D_SYNC (the stream passed waits for the reload).
 *
 * Host-resident states (reading D28, dc_model_bind_host_states): the device
 * copy of an offloaded fragment exists only in a ring slot of a device pool,
 * from its reload (DC_H2D_START: host -> slot) through its layer's update
 * (rs_adam reads and writes the slot) to DC_WRITEBACK (slot -> host, issued
 * by the executor right after that update); DC_D2H_START / DC_D2H_SYNC_FREE
 * are then no-ops because the host copy is already current.  The device m / v
 * arrays hold only the fragments the plan keeps resident, so the offloaded
 * bytes are really free for activations.  DC_WRITEBACK outside host-state mode
 * is DC_ESTATE.
 * ------------------------------------------------------------------------ */
typedef struct { int32_t layer; int32_t state; /* 0 = m, 1 = v */ int64_t offset_elems, elems; } dc_fragment;
dc_status dc_offload_fragments(dc_ctx* ctx, int64_t max_fragment_bytes, dc_fragment* out,
                               int32_t* n_inout);
dc_status dc_offload(dc_ctx* ctx, int32_t fragment, int32_t op, cudaStream_t stream);

/* ------------------------------------------------------------------------
 * Synthetic Llama-shaped layer stack — the "user model"
 * that exercises the path.  GEMMs are tcgen05/TMEM/TMA kernels (bf16 in,
 * fp32 accumulate); glue kernels are fused elementwise/row kernels.
 * ------------------------------------------------------------------------ */
typedef struct {
  int32_t hidden, ffn, n_heads, n_kv, head_dim, layers, tokens;
  int32_t checkpoint;            /* 1: layer-level activation checkpointing (*/
                                 /* "recomputing each layer as a block"): only each */
                                 /* layer's output is kept; the backward of a layer */
                                 /* re-runs its forward ops (all but down) first    */
  int32_t n_experts;             /* 0: Llama-shaped MLP; 2..8: Mixtral-shaped MoE  */
                                 /* MLP: router [E, hidden], */
                                 /* fixed balanced top-2 routing t -> t mod E,       */
                                 /* (t+1) mod E, gates = softmax of the two logits;  */
                                 /* per layer 7 + 3E params in the order attn_norm,  */
                                 /* wq, wk, wv, wo, mlp_norm, router, then w1_e,     */
                                 /* w3_e, w2_e per expert.  tokens % (4E) == 0.      */
} dc_model_dims;

/* Plain GEMM entry (tests, comparators): C[M,N] (bf16, row-major, ldc) =
 * A_op[M,K] * B_op[K,N] (+ R[M,N] if R != NULL), fp32 accumulation.
 * a_mn_major = 0: A stored [M][lda] (K contiguous); 1: A stored [K][lda]
 * (M contiguous).  b_mn_major = 0: B stored [N][ldb] (K contiguous, i.e. the
 * nn.Linear weight layout for x W^T); 1: B stored [K][ldb] (N contiguous).
 * Up to 4 B segments split along N (b_split_k = 0; seg_end in units of
 * 256 columns) or along K (b_split_k = 1; seg_end in units of 64). */
typedef struct {
  int32_t M, N, K;
  const void* A; int64_t lda; int32_t a_mn_major;
  int32_t n_bseg; const void* B[4]; int64_t ldb[4]; int32_t bseg_end[4];
  int32_t b_mn_major, b_split_k;
  void* C; int64_t ldc;
  const void* R; int64_t ldr;
  int32_t num_sms;               /* 0 = all SMs                                 */
  int32_t kernel;                /* 0 auto (CTA pairs), 1 one-CTA tiles, 2 pairs */
  int32_t stream_k;              /* 1: split the last waves' k-blocks evenly over */
                                 /* the pairs (fp32 partials through `workspace`, */
                                 /* deterministic); ignored when workspace is    */
                                 /* NULL.  Only when no other persistent GEMM can */
                                 /* run concurrently on the device (it spins on  */
                                 /* another pair's partial).                     */
  int32_t epilogue;              /* 0 plain; CTA pairs only, N = F (SwiGLU width): */
                                 /* 2 GLU forward: B = {W_gate, W_up} (2 K-major  */
                                 /*   segments, bseg_end ignored), C = gate half  */
                                 /*   of gu, C + glu_off = up half (ldc = 2F),    */
                                 /*   aux[row * ld_aux + j] = SiLU(g) * u (bf16)  */
                                 /* 3 GLU backward: acc = dact, aux = gu (ld_aux  */
                                 /*   = 2F, up half at + glu_off), C = d(gate),   */
                                 /*   C + glu_off = d(up); same values as the     */
                                 /*   separate act / act_bwd kernels, bit for bit */
  void* aux; int64_t ld_aux, glu_off;
  /* stream-K workspace: caller-owned device memory of at least
   * dc_gemm_workspace_bytes() bytes, zero-filled before its first use and
   * used by launches on ONE stream at a time (they are ordered, so they may
   * share it; the library keeps a per-workspace launch epoch, so stale flags
   * of earlier launches are harmless).  NULL: no stream-K. */
  void* workspace; uint64_t workspace_bytes;
  /* persistent tile order (pair kernel): 0 auto (groups of 2 m-tiles when
   * m_tiles >= 2 n_tiles, else m-fastest over the whole grid); g > 0: groups
   * of g m-tiles (the last group may be partial); -1: never group. */
  int32_t tile_group_m;
  /* fused all-gather -> GEMM (CTA-pair kernel only): for a B
   * segment s with chunk_flags[s] != NULL the producer, before loading B
   * elements of that segment (flat row-major index into the segment's tensor
   * of chunk_numel[s] elements), waits until every chunk overlapping them
   * holds a value >= chunk_value[s] (serial-number compare): chunk (q, j) is
   * the flat range [q S + j E, min(q S + (j + 1) E, (q + 1) S)), its word
   * chunk_flags[s][q * 64 + j], S = chunk_S[s] (shard elements), E =
   * chunk_E[s].  Acquire loads, then fence.proxy.async before the TMA loads.
   * A wait longer than chunk_timeout_ns writes the device error record at
   * chunk_err (the ctx's, reported by dc_poll as DC_ETIMEOUT) and proceeds. */
  const uint32_t* chunk_flags[4]; int64_t chunk_S[4], chunk_E[4], chunk_numel[4]; uint32_t chunk_value[4];
  uint32_t* chunk_err; uint64_t chunk_timeout_ns;
} dc_gemm_args;
dc_status dc_gemm(const dc_gemm_args* g, cudaStream_t stream);
/* Bytes of a stream-K workspace (fp32 partial tiles + flags). */
uint64_t dc_gemm_workspace_bytes(void);
/* CTA pairs the default pair kernel keeps co-resident on this device
 * (cudaOccupancyMaxActiveClusters; the persistent grid never exceeds it);
 * -1 on a CUDA error. */
int32_t dc_gemm_pair_slots(void);

dc_status dc_model_create(dc_ctx* ctx, const dc_model_dims* d, dc_model** out);
dc_status dc_model_destroy(dc_model* m);
/* Bytes of the activation + workspace buffer the caller must provide. */
dc_status dc_model_act_bytes(const dc_model* m, uint64_t* bytes);
/* x, target: bf16 [n][tokens][hidden] device buffers: this rank's n =
 * micro_steps (dc_init) micro-batches, contiguous. */
dc_status dc_model_bind(dc_model* m, void* act_buf, uint64_t act_bytes, const void* x,
                        const void* target);
/* The S_0 schedule of the model as a profile skeleton (p_mem/transient/dur
 * filled from the last profiled step if any, else 0). */
dc_status dc_model_profile_json(const dc_model* m, char* buf, size_t* len);
/* One training step through the bound schedule: per micro-step forward,
 * loss, backward with gathers / releases / reduce-scatter (+ Adam on the last
 * micro-step) / offload ops interleaved as planned.  Streams: compute, ag, rs, copy.  profile: 0 off; 1 record per-op
 * CUDA events around every compute / RS op and read them now (synchronises);
 * 2 record only (read by the next dc_model_profile_json, no sync). */
dc_status dc_model_step(dc_model* m, int32_t step_t, int32_t profile, cudaStream_t compute,
                        cudaStream_t ag, cudaStream_t rs, cudaStream_t copy);
/* Device pointer to fp32 [n]: the loss (mean 1/2 (y-t)^2) of every
 * micro-step of the last step. */
dc_status dc_model_loss_ptr(const dc_model* m, float** loss);
/* Pointers into the activation buffer of layer l (tests): which = 0 h1, 1 qkv,
 * 2 a, 3 x2, 4 h2, 5 gate|up, 6 act, 7 y (layer output), 8 / 9 the two
 * backward gradient ping-pong buffers. */
dc_status dc_model_act_ptr(const dc_model* m, int32_t layer, int32_t which, void** ptr);
/* Options: "fused_adam" (default 0; N = 1 only) — the reduce-scatter is the
 * identity at N = 1, so each weight's Adam update (the rs_adam arithmetic on
 * fp32(bf16(grad)), bit-identical) can run in the epilogue of its dW GEMM,
 * leaving only the norm gains to rs_adam.  Ignored for a step whose schedule
 * offloads optimizer state (the reload lands after the dW GEMMs) and with
 * gradient accumulation (micro_steps > 1).
 * "side_adam" (default 0; N = 1 only): layer l's reduce-scatter + Adam (the
 * rs_adam arithmetic, bit-identical) is sliced across layer l-1's backward
 * GEMM launches and streamed by idle warps of the CTA-pair GEMM, so the
 * HBM-bound update overlaps tensor-bound work instead of competing for SMs;
 * layer 0's update stays an rs_adam launch.  Same offload exclusion.
 * "stream_k" (default 1 unless N > 1 virtual ranks share the GPU): the layer
 * GEMMs split their last waves with stream-K (dc_gemm_args.stream_k).
 * "rs_overlap" (default 1 at N > 1, 0 at N = 1): reduce-scatter + Adam on the rs stream beside the
 * backward GEMMs; 0 runs it in compute-stream order.
 * "dw_stream" / "wb_stream" (value = a cudaStream_t, caller-owned, must outlive
 * the model): the stream of the concurrent dW GEMMs / of the host-state
 * write-backs instead of one the model creates (DC_EINVAL for 0, DC_ESTATE
 * after graph capture).  Virtual ranks sharing one GPU pass streams from one
 * pool so that no two ranks share a hardware queue. */
dc_status dc_model_set_option(dc_model* m, const char* key, int64_t value);
/* Host-resident optimizer states (reading D28; §4.4 P:370-408 with
 * the update fused per layer, D17).  After dc_bind_schedule of a plan whose
 * offloaded fragments (dc_offload_fragments) are whole (layer, m|v) slices
 * forming a prefix of the fragment order:
 *   query: m_first / v_first = first element of m / v that stays device
 *     resident (every element below is offloaded; shard_elems when all are,
 *     0 without offload); pool_bytes = ring of slots the reloads land in
 *     (slots * the largest offloaded fragment; a slot is reused once the
 *     fragment in it was written back, in schedule order on the copy stream).
 *   bind: m_dev / v_dev = fp32 device arrays of shard_elems - m_first /
 *     v_first elements (NULL if 0), pool = at least the queried pool_bytes of
 *     device memory (NULL if 0); whole extra slots are used round-robin so
 *     a reload need not wait for the write-back just issued.  host_bytes (query) = pinned host bytes the offloaded fragments'
 *     slots span (fragments are packed in id order); host_pinned (bind), if
 *     not NULL, replaces dc_init's host_pinned buffer.  Caller-owned.  States
 *     are reset to zero (device arrays and the offloaded fragments' pinned
 *     host slots): bind before the first step.
 * DC_EINVAL if the plan's offload set is not such a prefix, DC_ESTATE without
 * a bound schedule or with micro_steps > 1. */
dc_status dc_model_host_states_query(dc_model* m, int64_t* m_first, int64_t* v_first, uint64_t* pool_bytes,
                                     uint64_t* host_bytes);
dc_status dc_model_bind_host_states(dc_model* m, float* m_dev, float* v_dev, void* pool, uint64_t pool_bytes,
                                    void* host_pinned, uint64_t host_bytes);
/* CUDA graph of the scheduled step (context option
 * "graph_mode" set before dc_bind_schedule; no offload / host states / side or
 * fused Adam / SM partition).  In graph mode every step restarts the whole
 * flag protocol (gather ready / done, grad-slot and reduce-scatter counters,
 * stream-K flags) from zero — at N > 1 between two rounds of a barrier on a
 * device step counter (A: every rank finished the previous step; B: every
 * rank cleared its table) — and rs_adam reads the step's Adam scalars from
 * device memory, so one captured step is valid for every later step.  Each
 * rank (process or virtual rank) captures and replays its own graph.
 * capture: records one dc_model_step on `compute` (the other streams fork from
 *   and join it) into a graph WITHOUT executing it; step_t only has to be >= 1.
 * launch: writes step_t's Adam scalars (same host arithmetic as the eager path)
 *   and replays the graph on `compute` (asynchronous).  Bit-identical to eager
 *   steps.  DC_ESTATE without graph_mode / a captured graph. */
dc_status dc_model_graph_capture(dc_model* m, int32_t step_t, cudaStream_t compute, cudaStream_t ag,
                                 cudaStream_t rs, cudaStream_t copy);
dc_status dc_model_graph_launch(dc_model* m, int32_t step_t, cudaStream_t compute);
/* Host-resident states (reading D28): dc_model_step does not join the
 * write-back stream into the compute stream — the write-backs of the step's
 * last updated fragments overlap the next step's forward, whose reloads wait
 * for them.  This enqueues on `stream` a wait for every write-back issued so
 * far (call before reading the host copies from the stream, or before the
 * end event of a timed region); DC_OK and nothing enqueued otherwise. */
dc_status dc_model_join_states(dc_model* m, cudaStream_t stream);
/* Number of kernels the last dc_model_step launched. */
dc_status dc_model_launch_count(const dc_model* m, int64_t* n);

#ifdef __cplusplus
}
#endif
#endif /* DC_H */
