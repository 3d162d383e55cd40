/* dh — the B200 device layer of the SI framework, as a C ABI.
 *
 * Everything the host planner (include/weft/ headers) needs from the GPU crosses
 * here: plain pointers, sizes and an opaque CUDA stream (void*); no C++ or
 * torch types. Every call returns a dh status; dh_last_error() gives the
 * message (thread-local).
 *
 * Reference interfaces replaced (the reference has no device code):
 *   - the lane model's "one op per lane" (reference core.hpp:29-33) becomes one
 *     CUDA stream per lane inside a dh_ctx;
 *   - each DAG template node (reference op_model.cpp:79-113, our
 *     op_model.cpp kDenseNodes) becomes dh_node_launch(..., node_id) whose
 *     kernels are the ones below;
 *   - the solo / pair time tables the reference reads from JSON
 *     (overlap_profile.cpp:227-259) are produced by dh_profile_*.
 *
 * Layout conventions: all matrices row-major; activations bf16; weights bf16
 * with fp32 master copies and fp32 gradient accumulators.
 */
#ifndef DH_CAPI_H
#define DH_CAPI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum dh_status {
    DH_OK = 0,
    DH_ERR_OTHER = 1,
    DH_ERR_CONFIG = 2,     /* == weft ConfigError exit code      */
    DH_ERR_INFEASIBLE = 3, /* == weft InfeasibleError exit code  */
    DH_ERR_MISSING = 4,    /* == weft MissingProfileEntry code   */
    DH_ERR_INVALID = 5,    /* bad argument                       */
    DH_ERR_CUDA = 6,       /* CUDA runtime / driver failure      */
    DH_ERR_NCCL = 7,       /* NCCL failure                       */
    DH_ERR_OOM = 8         /* memory pool exhausted              */
};

const char* dh_last_error(void);
int dh_version(void);

/* ---------------------------------------------------------------- kernels */

/* D(m,n) (+)= sum_k A(m,k) B(n,k) on tcgen05 (gemm_tcgen05.cu).
 * a_mn = 0: A(m,k) = a[m*lda + k]  (K-major)     a_mn = 1: A(m,k) = a[k*lda + m]
 * b_mn = 0: B(n,k) = b[n*ldb + k]  (K-major)     b_mn = 1: B(n,k) = b[k*ldb + n]
 * d_fp32 = 0: D bf16, d_fp32 = 1: D fp32; accumulate = 1 adds into D (fp32 exact
 * sum; bf16: D = bf16(D + bf16(acc)) on the CTA-pair path, bf16(D + acc) otherwise).
 * max_ctas caps the persistent grid (0 = every SM). tile_n: 0 = auto; 128/192/256 = one
 * CTA per 128 x tile_n tile; 512 = CTA pair (cta_group::2) per 256 x 256 tile;
 * -128/-192/-256 = CTA pair per 256 x abs(tile_n) tile (-192 needs a K-major B). */
typedef struct dh_gemm_args {
    const void* a;
    long long lda;
    int a_mn;
    const void* b;
    long long ldb;
    int b_mn;
    void* d;
    long long ldd;
    int d_fp32;
    int m, n, k;
    int accumulate;
    int max_ctas;
    int tile_n;
    /* Fused SwiGLU epilogues (bf16 d, no accumulate; d2 and aux share d's row pitch ld_aux):
     *   DH_EPI_SWIGLU_FWD     d = up = bf16(acc), d2 = act = silu(aux0 = gate) * up
     *   DH_EPI_SWIGLU_FWD_UP  d = gate = bf16(acc), d2 = act = silu(gate) * (aux0 = up)
     *   DH_EPI_SWIGLU_BWD     acc = d_act (rounded to bf16); d = d_gate, d2 = d_up from
     *                         aux0 = gate, aux1 = up (d_act itself is not stored) */
    int epilogue;
    void* d2;
    const void* aux0;
    const void* aux1;
    long long ld_aux;
    /* Two-segment GEMMs in one launch (CTA-pair kernel; otherwise two launches, same result
     * up to summation order), not with the SwiGLU epilogues:
     *   K-concatenation (k2 > 0): D (+)= A B^T + A2 B2^T, A2 / B2 with A's / B's majors and K = k2
     *     (k % 64 == 0), accumulated in one pass (one rounding of D).
     *   M-concatenation (m2 > 0): rows [0, m) of the result from A into D, rows [0, m2) from A2
     *     into d_m2 (same B, same epilogue; m % 256 == 0). */
    const void* a2;
    long long lda2;
    const void* b2;
    long long ldb2;
    int k2;
    void* d_m2;
    long long ldd_m2;
    int m2;
} dh_gemm_args;
/* DH_EPI_SWIGLU_PAIR: mlp_gate and mlp_up as one GEMM (K-major A, B = Wg, B2 = Wu, both [n, k]):
 * d = gate = bf16(A Wg^T), d2 = up = bf16(A Wu^T), d_m2 = act = silu(gate) * up (all [m, n], pitch ldd). */
enum { DH_EPI_NONE = 0, DH_EPI_SWIGLU_FWD = 1, DH_EPI_SWIGLU_FWD_UP = 2, DH_EPI_SWIGLU_BWD = 3,
       DH_EPI_SWIGLU_PAIR = 4 };
int dh_gemm(const dh_gemm_args* args, void* stream);

/* RMSNorm over the last dim (elementwise.cu). y = x * rstd * gamma, rstd fp32 [rows]. */
int dh_rmsnorm_fwd(const void* x, const void* gamma, void* y, float* rstd, int rows, int cols,
                   float eps, void* stream);
/* Fused residual add + RMSNorm (bda0 + ln1): x_out = bf16(x + resid), y = RMSNorm(x_out);
 * bitwise dh_add followed by dh_rmsnorm_fwd. resid NULL = dh_rmsnorm_fwd. */
int dh_add_rmsnorm_fwd(const void* x, const void* resid, void* x_out, const void* gamma, void* y,
                       float* rstd, int rows, int cols, float eps, void* stream);
/* dx = RMSNorm'(dy) (+ resid if non-null); dgamma_acc[cols] += sum_rows dy*x*rstd,
 * reduced deterministically through `partial` (fp32, >= 1184*cols floats). */
int dh_rmsnorm_bwd(const void* x, const void* gamma, const float* rstd, const void* dy,
                   const void* resid, void* dx, float* dgamma_acc, float* partial, int rows,
                   int cols, void* stream);
/* out = a + b (bf16, n elements). */
int dh_add(const void* a, const void* b, void* out, long long n, void* stream);
/* act = silu(gate) * up */
int dh_swiglu_fwd(const void* gate, const void* up, void* act, long long n, void* stream);
/* dgate = dact * up * silu'(gate), dup = dact * silu(gate) */
int dh_swiglu_bwd(const void* gate, const void* up, const void* dact, void* dgate, void* dup,
                  long long n, void* stream);
/* Rotary embedding in place on the q and k heads of a packed qkv row block:
 * row t holds [q heads | k heads | v heads], head_dim each, row pitch `ld`.
 * inverse = 1 applies the transpose rotation (the backward). Position = t + pos0. */
int dh_rope(void* qkv, long long ld, int tokens, int n_q_heads, int n_kv_heads, int head_dim,
            float theta, int pos0, int inverse, void* stream);
/* Causal GQA flash attention (attention.cu). q/k/v/o are [tokens, heads*head_dim]
 * views with row pitches; lse fp32 [n_q_heads, tokens]. head_dim 64 or 128.
 * `scratch` (fp32, may be NULL) enables splitting long causal rows into KV
 * chunks when the grid is too small to balance the SMs (few heads per GPU);
 * it is used only if scratch_floats >= dh_attn_fwd_scratch_floats(...). */
long long dh_attn_fwd_scratch_floats(int tokens, int n_q_heads, int n_kv_heads, int head_dim);
int dh_attn_fwd(const void* q, const void* k, const void* v, long long ldq, long long ldkv,
                void* o, long long ldo, float* lse, float* scratch, long long scratch_floats,
                int tokens, int n_q_heads, int n_kv_heads, int head_dim, float scale, void* stream);
/* Context-parallel form (the cp_kv_exchange path): `tokens` query rows at
 * global positions [q_offset, q_offset + tokens) attend causally to
 * `tokens_kv` key rows (q_offset a multiple of 256, q_offset + tokens <=
 * tokens_kv). dh_attn_fwd is the case tokens_kv == tokens, q_offset == 0. */
long long dh_attn_fwd_scratch_floats_ex(int tokens, int n_q_heads, int n_kv_heads, int head_dim, int tokens_kv,
                                        int q_offset);
int dh_attn_fwd_ex(const void* q, const void* k, const void* v, long long ldq, long long ldkv, void* o,
                   long long ldo, float* lse, float* scratch, long long scratch_floats, int tokens, int tokens_kv,
                   int q_offset, int n_q_heads, int n_kv_heads, int head_dim, float scale, void* stream);
/* dq/dk/dv written (not accumulated); `scratch` fp32 of dh_attn_bwd_scratch_floats_ex floats for
 * this shape (the backward's work plan: rowsum(dO*O) plus the partial slots of GQA groups and of
 * items split across SMs; dh_attn_bwd_scratch_floats covers any n_kv_heads at q_offset 0). The _ex
 * form: dk/dv cover all tokens_kv key rows, each the gradient from this call's queries only. */
long long dh_attn_bwd_scratch_floats(int tokens, int n_q_heads, int head_dim, int tokens_kv);
/* exact scratch of dh_attn_bwd_ex for this GQA shape and query offset */
long long dh_attn_bwd_scratch_floats_ex(int tokens, int n_q_heads, int n_kv_heads, int head_dim, int tokens_kv,
                                        int q_offset);
int dh_attn_bwd_ex(const void* q, const void* k, const void* v, long long ldq, long long ldkv, const void* o,
                   long long ldo, const float* lse, const void* dout, void* dq, void* dk, void* dv, long long lddq,
                   long long lddkv, float* scratch, int tokens, int tokens_kv, int q_offset, int n_q_heads,
                   int n_kv_heads, int head_dim, float scale, void* stream);
int dh_attn_bwd(const void* q, const void* k, const void* v, long long ldq, long long ldkv,
                const void* o, long long ldo, const float* lse, const void* dout,
                void* dq, void* dk, void* dv, long long lddq, long long lddkv, float* scratch,
                int tokens, int n_q_heads, int n_kv_heads, int head_dim, float scale,
                void* stream);
/* AdamW on fp32 master weights; refreshes the bf16 copy; zeroes grad if zero_grad. */
int dh_adamw(float* master, void* weight_bf16, float* grad, float* m, float* v, long long n,
             float lr, float beta1, float beta2, float eps, float weight_decay, int step,
             float grad_scale, int zero_grad, void* stream);
/* AdamW whose hyperparameters live in device memory (9 floats written by
 * dh_adamw_set_hparams): capturable in a CUDA graph that replays every step.
 * enabled == 0 turns the launch into a no-op. Gradients are zeroed after use.
 * Same per-element math as dh_adamw with the same (lr, betas, eps, wd, step). */
typedef struct dh_adamw_hparams {
    float lr, beta1, beta2, eps, weight_decay;
    float bc1, bc2;    /* 1 - beta^step, computed on the host as dh_adamw does */
    float grad_scale;
    int enabled;
} dh_adamw_hparams;
int dh_adamw_set_hparams(float* hp_dev, const dh_adamw_hparams* v, void* stream);
int dh_adamw_dev(float* master, void* weight_bf16, float* grad, float* m, float* v, long long n,
                 const float* hp_dev, void* stream);
/* Deterministic normal(0, std) init of bf16 (and optional fp32 master) from (seed, offset). */
int dh_init_normal(void* bf16_out, float* f32_out, long long n, unsigned long long seed,
                   float std_dev, void* stream);
/* Holds `stream` for `ns` nanoseconds (one thread, globaltimer): a launch gate
 * so ops queued behind it start together, free of host launch latency. */
int dh_spin_ns(long long ns, void* stream);
int dh_fill_bf16(void* out, float value, long long n, void* stream);
int dh_copy(void* dst, const void* src, long long bytes, void* stream);
/* Single-GPU stand-in for one rank's collective (mode 0 AllGather of `count`
 * bf16 per rank, 1 ReduceScatter to `count`, 2 AllToAll of a `count`-element
 * buffer): same HBM traffic on `ctas` CTAs, held for the wire bytes ((tp-1)*count*2,
 * a2a (tp-1)/tp*count*2) / link_gbs. Not numerically a collective. */
int dh_comm_proxy(const void* src, void* dst, long long count, int tp, int mode, int ctas,
                  double link_gbs, void* stream);
/* *loss = sum(y * r) in fp32, deterministic two-pass reduction through
 * partial (>= 1024 floats). One micro-batch, this rank's SP shard. */
int dh_dot_loss(const void* y, const void* r, long long n, float* partial, float* loss,
                void* stream);

/* ---------------------------------------------------------------- MoE (moe.cu)
 * Nodes of the moe_ep template (reference op_model.cpp:121-169). Slot layout:
 * expert e owns rows [e*C, (e+1)*C) of a [E*C, hidden] block (C = capacity per
 * expert per source rank); assignment a = t*topk + k. Empty slots are zero rows. */
/* router (9): probs fp32 [T,E] = softmax(x wr^T) (the logits GEMM on tcgen05, fp32
 * out), ids int32 [T,K] = top-k by probability (ties: lower expert), wts fp32 [T,K]
 * = top / sum(top). E <= 64 and a multiple of 4, K <= 8. */
int dh_moe_router_fwd(const void* x, const void* wr, float* probs, int* ids, float* wts, int tokens,
                      int hidden, int experts, int topk, void* stream);
/* permute (10), part 1: slot[a] = e*C + (rank of a among expert e's assignments in
 * (t, k) order) or -1 past capacity; slot_src[e*C + j] = a or -1 (empty). */
int dh_moe_assign(const int* ids, int tokens, int topk, int experts, int capacity, int* slot,
                  int* slot_src, void* stream);
/* permute (10), part 2: xp[s] = x[slot_src[s] / topk] (zero row when empty). */
int dh_moe_permute(const void* x, const int* slot_src, void* xp, int n_slots, int topk, int hidden,
                   void* stream);
/* unpermute (15): out[t] = bf16(sum_k wts[t,k] * y[slot[t,k]]), k ascending, fp32. */
int dh_moe_unpermute(const void* y, const int* slot, const float* wts, void* out, int tokens, int topk,
                     int hidden, void* stream);
/* unpermute_bwd (21): dys[s] = bf16(wts[a] * dy[t]); dw[a] = <y[s], dy[t]> (a = slot_src[s]). */
int dh_moe_unpermute_bwd(const void* dy, const void* y, const int* slot_src, const float* wts, void* dys,
                         float* dw, int n_slots, int topk, int hidden, void* stream);
/* permute_bwd (28): dx[t] = bf16(sum_k dxp[slot[t,k]]). */
int dh_moe_permute_bwd(const void* dxp, const int* slot, void* dx, int tokens, int topk, int hidden,
                       void* stream);
/* router_bwd (29): through the top-k renormalisation and the softmax (dropped
 * assignments carry no weight gradient); dlogits (bf16) then feeds two tcgen05
 * GEMMs: dx_out = dx_in + dlogits wr (bf16 accumulate; dx_out may equal dx_in),
 * dwr[E,H] += dlogits^T x (fp32). scratch: fp32, at least
 * dh_moe_router_bwd_scratch_floats(tokens, hidden, experts). */
long long dh_moe_router_bwd_scratch_floats(int tokens, int hidden, int experts);
int dh_moe_router_bwd(const float* probs, const int* ids, const int* slot, const float* dw, const void* x,
                      const void* wr, const void* dx_in, void* dx_out, float* dwr, float* scratch, int tokens,
                      int hidden, int experts, int topk, void* stream);
/* ---------------------------------------------------------------- runtime */

typedef struct dh_ctx dh_ctx;
typedef struct dh_model dh_model;

/* One context per GPU / TP rank. nccl_unique_id: the 128-byte ncclUniqueId
 * shared by the TP group (NULL when tp_size == 1; with tp_size == 1 and an id,
 * a one-rank communicator that only dh_comm_run uses). nccl_max_ctas caps the SMs
 * NCCL kernels occupy (0 = NCCL default) so they coexist with the other
 * strand's GEMMs (north star (2)). Streams: one per weft::Lane. */
int dh_ctx_create(int device, int tp_rank, int tp_size, const void* nccl_unique_id,
                  int nccl_max_ctas, dh_ctx** out);
/* One W-pipeline stage on one GPU (weft SendRecv between stages, reference
 * folding_pipeline.cpp:157-192): a dh_ctx_create context for this stage's TP
 * group plus a stage group of pp_size ranks over NCCL (pp_unique_id shared by
 * the stage group; NULL when pp_size == 1). Activations and gradients travel
 * on two communicators split from the stage group, each on its own stream,
 * so a stage's sends never block its compute stream. Not graph-capturable. */
int dh_ctx_create_pp(int device, int tp_rank, int tp_size, const void* tp_unique_id, int pp_rank, int pp_size,
                     const void* pp_unique_id, int nccl_max_ctas, dh_ctx** out);
/* Single-process pipeline group on ONE device (test backend): pp_size stage
 * contexts (TP = 1) whose point-to-point activation / gradient transfers are
 * staged device copies matched in program order (never blocking the sender). */
int dh_loopback_pp_group_create(int device, int pp_size, dh_ctx** ctxs_out);
/* Single-process multi-rank "loopback" group on ONE device (test backend):
 * creates tp_size contexts whose AllGather / ReduceScatter are device copies
 * plus a fixed-order sum. Each context must be driven by its own host thread
 * (collectives rendezvous like real ranks). Not graph-capturable. */
int dh_loopback_group_create(int device, int tp_size, dh_ctx** ctxs_out);
/* Emulated TP group on ONE GPU (performance studies only): this context has
 * the per-rank shapes of tp_size ranks, but its collectives are dh_comm_proxy
 * kernels (comm_ctas CTAs, NVLink-time link_gbs) — numerically meaningless,
 * timing- and SM-footprint-faithful. Graph-capturable. */
int dh_ctx_create_emulated(int device, int tp_size, int comm_ctas, double link_gbs, dh_ctx** out);
int dh_ctx_destroy(dh_ctx* ctx);
/* One collective of the context's TP / EP group on lane stream `lane`,
 * enqueue-only (the same backend call the SI executor issues for an ag / rs /
 * a2a node; reference comm bytes op_model.cpp:290-301). bf16 elements, except
 * DH_COMM_ALL_REDUCE_F32 (fp32; recv may equal send):
 *   ALL_GATHER      recv[r*count + i] = send_r[i]
 *   REDUCE_SCATTER  recv[i] = sum_r send_r[rank*count + i]
 *   ALL_TO_ALL      recv[src*count + i] = send_src[rank*count + i]
 * Used to time each collective alone (bench.py: NVLink bus GB/s) and to test
 * the backends against their definitions. */
enum { DH_COMM_ALL_GATHER = 0, DH_COMM_REDUCE_SCATTER = 1, DH_COMM_ALL_REDUCE_F32 = 2, DH_COMM_ALL_TO_ALL = 3 };
int dh_comm_run(dh_ctx* ctx, int op, const void* send, void* recv, long long count, int lane);
void* dh_ctx_stream(dh_ctx* ctx, int lane);
int dh_nccl_unique_id(void* out128);

typedef struct dh_model_cfg {
    int hidden, ffn, n_heads, n_kv_heads, head_dim, layers, seq_len;
    int micro_batches;
    float rope_theta, norm_eps;
    unsigned long long seed;
    float init_std;
    /* Pipeline stage (zero = single stage, the defaults): `layers` are this
     * stage's layers of the U-fold (weft fold_layers), `split_layer` the local
     * index where the way-back half starts (its input arrives from the next
     * stage, 0 = contiguous), `slots` the activation slots (0 = layers + 1;
     * pipelined micro-batches need more), pp_rank / pp_size the stage. */
    int slots, split_layer, pp_rank, pp_size;
    /* MoE (moe_ep template, zero = dense): experts > 1 makes the MLP a top-`topk`
     * mixture of `experts` SwiGLU experts with `capacity` slots per expert per
     * source rank (0 = ceil(1.25 * seq * topk / experts) rounded up to 32).
     * The context's group is then the EP group (attention runs data-parallel,
     * TP = 1) and each rank holds experts / group_size experts. */
    int experts, topk, capacity;
    /* Context parallelism (dense only, zero = off): with context_parallel = 1
     * the context's group is the CP group (TP = 1). Each rank holds seq_len /
     * group_size consecutive tokens (a multiple of 256) at global positions
     * rank * seq_len / group_size onward; cp_kv_exchange all-gathers the
     * layer's K/V over the group before attn (and again before attn_bwd, which
     * reduce-scatters the dK/dV partials back to their owners). Weights are
     * replicated: their gradients are summed over the group before AdamW. */
    int context_parallel;
} dh_model_cfg;

typedef struct dh_optim_cfg {
    float lr, beta1, beta2, eps, weight_decay;
    int enabled; /* 0: skip the optimizer (tests) */
} dh_optim_cfg;

/* Llama-style TP+SP layer stack on this rank: allocates ONE pool for weights,
 * fp32 master / grad / Adam state, L+1 activation slots shared by the strands
 * and one forward + one backward transient set. */
int dh_model_create(dh_ctx* ctx, const dh_model_cfg* cfg, dh_model** out);
int dh_model_destroy(dh_model* m);

/* Load an SI plan (weft plan_to_json text) and lower it to lane-stream launches.
 * profile_json (weft Profile schema, may be NULL) supplies the solo times the
 * lowering replays the lane dispatch rule with; cluster_json the ClusterSpec used
 * to rebuild the DAG (may be NULL = a B200 default). mode 0 = SI (W schedule:
 * F1, SI(F_{i+1}, B_i) ..., B_m), 1 = sequential (F1 B1 F2 B2 ...), both with
 * the plan's per-strand operator orders; 2 = SI with relaxed steps (same per-lane
 * issue order, lanes joined only at layer-pair boundaries). plan_json NULL =
 * template order, one segment per pass (valid for mode 1 and as a trivial SI plan). */
/* mode 3: W pipeline stage (weft schedule_w_pipeline(micro_batches, pp_size) blocks of
 * this pp_rank; SI visits pair the plan's steps as mode 0).
 * mode 4: as mode 2, with the backward layer's trailing attention weight gradients
 * issued after the next layer pair's first step (needs cfg.slots >= layers + 2).
 * Every mode computes bitwise the same losses and gradients. */
int dh_model_set_plan(dh_model* m, const char* plan_json, const char* profile_json,
                      const char* cluster_json, int mode);
/* Host-only lowering (no GPU needed): the launch program dh_model_set_plan would
 * build for (cfg, tp, rank, plan, mode), as JSON {"ops": [{strand, layer, node,
 * lane, slot, prev_slot, first_dx, waits}], "slots", "fwd_seq", "bwd_seq"}.
 * Every rank of a TP group must obtain the same collective order from it. */
int dh_lower_json(const dh_model_cfg* cfg, int tp, int rank, const char* plan_json,
                  const char* profile_json, int mode, char** out);
/* Cap the SMs of GEMMs that co-run with a collective (0 = no cap). */
/* In-program optimizer (default on): per-layer AdamW ops on the cross lane
 * overlap the last strand's backward; only the LN gammas are updated after the
 * program. Off: one AdamW over all parameters after the program (bitwise the
 * same weights). Takes effect at the next dh_model_set_plan. */
int dh_model_set_fuse_optimizer(dh_model* m, int on);
int dh_model_set_overlap_ctas(dh_model* m, int gemm_ctas);

/* Run one training step: every micro-batch forward + backward per the lowered
 * program, then (optionally) AdamW over all parameters. use_graph = 1 captures
 * the program once as a CUDA graph and replays it. Asynchronous: returns after
 * enqueueing on the compute lane stream. */
int dh_model_step(dh_model* m, const dh_optim_cfg* optim, int use_graph);
/* Only the forward/backward program (no optimizer, no grad zeroing). */
int dh_model_run_program(dh_model* m, int use_graph);
int dh_model_zero_grads(dh_model* m);
int dh_model_sync(dh_model* m);

/* Named device buffer access for tests / IO: name in {"x_in","dy","y","loss",
 * "w.<tensor>","grad.<tensor>","master.<tensor>","act.<field>"}, tensor in
 * {g0,g1,wqkv,wo,wg,wu,wd}. layer/strand select the instance.
 * dtype out: 0 bf16, 1 fp32. */
int dh_model_tensor(dh_model* m, const char* name, int layer, int strand, void** ptr,
                    long long* numel, int* dtype);
/* JSON with pool accounting, the lowered program and launch counts. Caller frees
 * with dh_free_string. */
int dh_model_info_json(dh_model* m, char** out);
void dh_free_string(char* s);
/* Timing probes: CUDA events around every launch of template node `node` in
 * the lowered program, on the launching lane stream. Each call adds a node to
 * the probed set (-1 = clear all). After a run, dh_model_probe_read_node
 * returns one node's summed time and launch count (dh_model_probe_read: the
 * first probed node). Re-arm after dh_model_set_plan (the program changed). */
int dh_model_probe(dh_model* m, int node);
int dh_model_probe_read_node(dh_model* m, int node, double* total_ms, int* count);
/* Measurement mode: re-lower the current plan without its collective nodes
 * (compute order and step barriers unchanged) so T_SI - T_compute_only gives
 * the exposed communication. */
int dh_model_set_skip_comm(dh_model* m, int skip);
int dh_model_probe_read(dh_model* m, double* total_ms, int* count);

/* ---------------------------------------------------------------- profiler */

/* On-device operator-pair overlap profiler (north star (4)): times every node
 * solo, and every cross-lane (forward node, backward node) pair co-running on
 * two streams, with CUDA events; aggregates P_ij into class-pair OEF via weft
 * Eq. 1 and emits a weft Profile JSON (solo keyed by node name, slowdown and
 * launch-overhead terms 0 because measured P_ij already include them). */
int dh_profile_json(dh_model* m, int iters, char** out);

#ifdef __cplusplus
}
#endif

#endif /* DH_CAPI_H */
