// Internal C++ runtime behind include/dh_capi.h: device context (lane streams,
// collective backend), the Llama TP+SP model (memory pool, weights, activation
// slot ring), per-template-node launchers and the SI executor.
//
// Ownership: dh_ctx owns streams, events and the communicator; dh_model owns
// one device slab (the pool) carved into model state, L+1 activation slots and
// one forward + one backward transient set. One host thread drives one ctx.
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "dh_capi.h"
#include "weft/op_model.hpp"
#include "weft/overlap_profile.hpp"
#include "weft/pairing_search.hpp"

namespace dh {

int set_error(int code, const char* msg);
inline int set_error(int code, const std::string& msg) { return set_error(code, msg.c_str()); }
int cuda_fail(cudaError_t e, const char* what);

#define RT_CUDA(expr)                                            \
    do {                                                         \
        cudaError_t rt_e_ = (expr);                              \
        if (rt_e_ != cudaSuccess) return ::dh::cuda_fail(rt_e_, #expr); \
    } while (0)
#define RT_TRY(expr)                 \
    do {                             \
        int rt_rc_ = (expr);         \
        if (rt_rc_ != DH_OK) return rt_rc_; \
    } while (0)

constexpr int kLanes = 3;  // weft::Lane: compute, local_comm, cross_comm

// ------------------------------------------------------------------ collectives

class Comm {
public:
    virtual ~Comm() = default;
    // recv[r*count .. (r+1)*count) = send of rank r (bf16 elements)
    virtual int all_gather(const void* send, void* recv, size_t count, cudaStream_t s) = 0;
    // recv = sum over ranks of send[rank*count .. (rank+1)*count) (bf16)
    virtual int reduce_scatter(const void* send, void* recv, size_t count, cudaStream_t s) = 0;
    virtual int all_reduce_f32(float* buf, size_t count, cudaStream_t s) = 0;
    // MoE all-to-all of bf16 chunks (`chunk` elements), `groups` chunks per peer:
    //   dispatch (combine = false): send [dst][g][chunk] -> recv [g][src][chunk]
    //   combine  (combine = true):  send [g][dst][chunk] -> recv [src][g][chunk]
    virtual int all_to_all(const void* send, void* recv, size_t chunk, int groups, bool combine,
                           cudaStream_t s) {
        return set_error(DH_ERR_CONFIG, std::string(name()) + ": no all-to-all");
    }
    // point-to-point (pipeline stages): a recv matches the send with the same
    // (peer pair, tag); the two stages may issue different tags in different orders
    virtual int send(const void* buf, size_t bytes, int peer, int tag, cudaStream_t s) {
        return set_error(DH_ERR_CONFIG, std::string(name()) + ": no point-to-point transfers");
    }
    virtual int recv(void* buf, size_t bytes, int peer, int tag, cudaStream_t s) {
        return set_error(DH_ERR_CONFIG, std::string(name()) + ": no point-to-point transfers");
    }
    // wait until every transfer this backend issued on its own streams is done
    virtual int sync() { return DH_OK; }
    // device-side rank alignment on stream s (the profiler's per-iteration start)
    virtual int barrier(cudaStream_t s) { return DH_OK; }
    virtual bool capturable() const = 0;
    virtual const char* name() const = 0;
};

std::unique_ptr<Comm> make_nccl_comm(int rank, int size, const void* unique_id, int max_ctas,
                                     int* rc);
std::unique_ptr<Comm> make_nccl_p2p(int rank, int size, const void* unique_id, int* rc);
struct LoopbackGroup;
std::unique_ptr<Comm> make_loopback_comm(LoopbackGroup* group, int rank, int* rc);

struct Ctx {
    int device = 0;
    int tp_rank = 0, tp_size = 1;
    int comm_ctas = 0;
    std::array<cudaStream_t, kLanes> lane{};
    std::unique_ptr<Comm> comm;
    std::unique_ptr<Comm> pp;  // pipeline-stage transfers (weft SendRecv, cross lane)
    int pp_rank = 0, pp_size = 1;
    int sm_count = 148;
};

// ------------------------------------------------------------------ model

struct ModelCfg {
    int hidden = 0, ffn = 0, n_heads = 0, n_kv_heads = 0, head_dim = 0, layers = 0, seq = 0;
    int micro_batches = 2;
    int slots = 0, split = 0, pp_rank = 0, pp_size = 1;  // pipeline stage (dh_model_cfg)
    float rope_theta = 500000.f, eps = 1e-5f;
    unsigned long long seed = 1234;
    float init_std = 0.02f;
    // MoE (moe_ep template): experts > 1; the context group is the EP group
    int experts = 0, topk = 0, capacity = 0;
    bool moe = false;
    int ep = 1, ep_rank = 0, e_loc = 0;  // EP group, experts held by this rank
    int moe_rows = 0;                    // experts * capacity: slot rows on either side of the a2a
    // context parallelism (the context group is the CP group; TP = 1): `seq` is
    // this rank's token chunk, starting at global position cp_rank * seq
    int cp = 1, cp_rank = 0, seq_full = 0;
    // derived (per TP rank)
    int tp = 1, rank = 0;
    int tok_loc = 0;  // seq / tp (sequence-parallel shard)
    int nq_l = 0, nkv_l = 0, qkv_n = 0, ffn_l = 0, attn_n = 0;
};

// Byte-offset view into the pool.
struct Buf {
    size_t off = 0, bytes = 0;
};

// Saved activations of one (strand, layer): lifetime = forward of that layer
// to its backward. L+1 of these form the ring shared by both strands.
// MoE layers add the routing state and the expert-side rows (gate / up / act
// then hold moe_rows rows: the slot rows of this rank's experts).
struct Slot {
    Buf out, rstd0, ln0_full, qkv, o, lse, x1, rstd1, ln1_full, gate, up, act;
    Buf probs, ids, wts, mslot, slot_src, xe, y;  // MoE: router outputs, slot maps, expert in / out
};

struct FwdScratch {
    Buf ln_loc, part, rs_out;
    Buf kv_loc, kv_full;  // CP: this rank's K|V rows packed, and the group's gathered
    Buf xp, ye;  // MoE with ep > 1: a2a send buffer of the permuted rows, expert outputs
};

struct BwdScratch {
    // dy_full: the gathered output gradient, double-buffered by layer parity so that a
    // deferred mlp_down_wgrad (mode 4) can still read it while the next layer gathers
    Buf grad[2], d_x1, dy_full[2], d_gate, d_up, d_act, dx_part, dx1_full, d_o, dqkv, attn_scratch,
        ln_partial, rs_out;
    Buf dys, dys_e, dxe, dxp, dw, router_scratch;  // MoE
    Buf kv_loc, kv_full, dkv_full, dkv_loc;        // CP: re-gathered K|V, dK|dV partials and sums
};

struct LayerParams {
    // offsets in elements into the flat parameter arrays
    // (MoE: wg / wu / wd are the e_loc stacked expert w1g / w1u / w2, wr the router)
    size_t g0, g1, wqkv, wo, wr, wg, wu, wd;
};

struct Model;

// Pseudo node of the lowered program: AdamW of one layer's matrices, issued on
// the cross lane right after the last strand's backward of that layer, so the
// optimizer overlaps the rest of the backward pass (device-side hyperparameters,
// a no-op unless dh_model_step armed them).
constexpr int kOptNode = 100;
// Pipeline transfers of one (strand, layer): the activation leaving / entering
// a visit and the gradient leaving / entering it (peer = Op::peer).
constexpr int kSendAct = 101, kRecvAct = 102, kSendGrad = 103, kRecvGrad = 104;

// One launch of the lowered schedule.
struct Op {
    int strand = 0;   // micro-batch index
    int layer = 0;
    int node = 0;     // template node id (op_model.cpp kDenseNodes)
    int lane = 0;     // stream
    int slot = 0;     // activation slot of (strand, layer)
    int prev_slot = -1;  // slot holding this layer's input (layer - 1), -1 = strand input
    bool first_dx = true;  // mlp_gate_dgrad/mlp_up_dgrad: whether this one overwrites dx_part
    bool fuse_swiglu = false;  // mlp_gate/mlp_up: the later of the two computes act in its epilogue
    std::vector<int> waits;  // indices of ops whose completion this op waits for
    bool barrier = false;    // step barrier before this op (all lanes joined)
    bool capped = true;      // GEMMs may co-run with a collective: limit them to gemm_ctas_overlap SMs
    int peer = -1;           // pipeline transfers: the other stage
    int part = -1;           // mlp_fc1_wgrad issued as two launches: 0 gate rows, 1 up rows (-1: both)
};

struct Program {
    std::vector<Op> ops;
    int mode = 0;  // 0 SI, 1 sequential
    std::vector<std::string> phases;
};

struct Model {
    Ctx* ctx = nullptr;
    ModelCfg cfg;
    // pool
    void* base = nullptr;
    size_t pool_bytes = 0;
    std::map<std::string, size_t> usage;  // bytes per category
    // flat model state
    size_t n_params = 0;
    Buf w_bf16, w_master, w_grad, adam_m, adam_v;
    std::vector<LayerParams> lp;
    size_t gamma_elems = 0;  // LN gammas live at [0, gamma_elems) of the flat arrays
    // activations
    std::vector<Slot> slots;  // layers + 1
    FwdScratch fs;
    BwdScratch bs;
    std::vector<Buf> mb_in, mb_dy;  // per micro-batch: input x0 and dL/dy (SP shards)
    std::vector<Buf> mid_in, mid_dy;  // split stage: input of the way-back half / dy of the way-down half
    Buf loss;                       // fp32 [micro_batches]
    // schedule
    weft::LayerDag fwd_dag, bwd_dag;
    weft::BestPlan plan;
    bool have_plan = false;
    Program prog;
    std::vector<cudaEvent_t> events;
    cudaGraphExec_t graph = nullptr;
    int adam_step = 0;
    int gemm_ctas_overlap = 0;  // SM cap for GEMMs that co-run with a collective
    bool fuse_optimizer = true;  // per-layer AdamW ops inside the program (kOptNode)
    // SwiGLU in the mlp GEMM epilogues (fwd: the later of mlp_gate / mlp_up; bwd:
    // mlp_down_dgrad) when the GEMM has enough waves to hide the epilogue;
    // otherwise standalone kernels after plain GEMMs (decided at model create)
    bool swiglu_in_epilogue = true;
    // mlp_gate | mlp_up as one GEMM (SwiGLU pair epilogue) and the gate / up dgrads as one
    // K-concatenated GEMM (DH_MLP_MERGE; default at TP = 1 only, see model.cpp). The fc1
    // wgrads are always one M-concatenated GEMM (one node either way).
    bool mlp_merge = true;
    bool prog_has_opt = false;   // the lowered program contains them
    int peak_slots = 0;          // activation slots the lowered program holds at once
    Buf opt_hp;                   // dh_adamw_hparams as 9 floats
    std::map<int, double> solo_us;  // node id -> solo time used for lowering
    weft::OverlapTable plan_overlap;  // table the lowering replays the lane model with
    std::array<cudaEvent_t, kLanes> fork_join{};
    std::vector<int> y_slot;  // slot holding each strand's last-layer output
    // timing probes: events around every launch of the probed template nodes
    std::vector<int> probe_nodes;
    bool skip_comm = false;  // measurement mode: collectives become no-ops (compute-only time)
    std::map<int, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>> probe_events;  // node -> per launch

    template <class T = void>
    T* ptr(const Buf& b) const {
        return reinterpret_cast<T*>(static_cast<char*>(base) + b.off);
    }
};

int derive_cfg(const dh_model_cfg* c, int tp, int rank, ModelCfg* out);
weft::ClusterSpec default_cluster();
int build_dags(Model& m, const weft::ClusterSpec& cl, const weft::SoloTimeTable* solo);
int configure_plan(Model& m, const char* plan_json, const char* profile_json, const char* cluster_json);
int lower_ops(Model& m, int mode);
int model_create(Ctx* ctx, const dh_model_cfg* c, Model** out);
void model_destroy(Model* m);
int launch_node(Model& m, const Op& op, cudaStream_t s);
// MoE-only nodes of the moe_ep template (moe.cpp); `dense_id` gets the
// dense_tp_sp id of a shared (attention / norm / residual) node, else -1.
int launch_moe_node(Model& m, const Op& op, cudaStream_t s, void* dy, int* dense_id);
int moe_dense_id(int moe_node);
int moe_capacity(int tokens, int experts, int topk);
int lower_program(Model& m, int mode);
int kernels_per_node(const Model& m, int node, int layer);
int run_program(Model& m, bool use_graph);
int run_optimizer(Model& m, const dh_optim_cfg* oc, cudaStream_t s);
int arm_optimizer(Model& m, const dh_optim_cfg* oc, cudaStream_t s);
int set_probe(Model& m, int node);
int read_probe(Model& m, int node, double* total_ms, int* count);

}  // namespace dh

struct dh_ctx : dh::Ctx {};
struct dh_model : dh::Model {};
