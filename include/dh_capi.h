/* dh — the B200 device layer of the SI framework, as a C ABI.
 *
 * Everything the host planner (include/weft/*.hpp) needs from the GPU crosses
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
 * d_fp32 = 0: D bf16, d_fp32 = 1: D fp32; accumulate = 1 adds into D.
 * max_ctas caps the persistent grid (0 = every SM); tile_n 0 = auto, 128, 256. */
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
} dh_gemm_args;
int dh_gemm(const dh_gemm_args* args, void* stream);

/* RMSNorm over the last dim (elementwise.cu). y = x * rstd * gamma, rstd fp32 [rows]. */
int dh_rmsnorm_fwd(const void* x, const void* gamma, void* y, float* rstd, int rows, int cols,
                   float eps, void* stream);
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
 * views with row pitches; lse fp32 [n_q_heads, tokens]. head_dim 64 or 128. */
int dh_attn_fwd(const void* q, const void* k, const void* v, long long ldq, long long ldkv,
                void* o, long long ldo, float* lse, int tokens, int n_q_heads, int n_kv_heads,
                int head_dim, float scale, void* stream);
/* dq/dk/dv written (not accumulated); `scratch` fp32 >= tokens*n_q_heads*(2*head_dim+1) floats. */
int dh_attn_bwd(const void* q, const void* k, const void* v, long long ldq, long long ldkv,
                const void* o, long long ldo, const float* lse, const void* dout,
                void* dq, void* dk, void* dv, long long lddq, long long lddkv, float* scratch,
                int tokens, int n_q_heads, int n_kv_heads, int head_dim, float scale,
                void* stream);
/* AdamW on fp32 master weights; refreshes the bf16 copy; zeroes grad if zero_grad. */
int dh_adamw(float* master, void* weight_bf16, float* grad, float* m, float* v, long long n,
             float lr, float beta1, float beta2, float eps, float weight_decay, int step,
             float grad_scale, int zero_grad, void* stream);
/* Deterministic normal(0, std) init of bf16 (and optional fp32 master) from (seed, offset). */
int dh_init_normal(void* bf16_out, float* f32_out, long long n, unsigned long long seed,
                   float std_dev, void* stream);
int dh_fill_bf16(void* out, float value, long long n, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DH_CAPI_H */
