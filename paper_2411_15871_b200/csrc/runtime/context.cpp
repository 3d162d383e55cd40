// Device context: lane streams and the collective backend.
//
// Lanes (weft::Lane, reference core.hpp:29-33) map 1:1 to CUDA streams; the
// communication lanes get the highest stream priority so a collective's CTAs
// are scheduled ahead of the co-running strand's GEMM tiles.
//
// Backends:
//   * NcclComm     — one communicator per TP group (ncclCommInitRankConfig with
//                    maxCTAs = the SM budget left to NCCL), bf16 AllGather /
//                    ReduceScatter, fp32 AllReduce. Graph-capturable.
//   * LoopbackComm — tp_size ranks inside one process on ONE device, each driven
//                    by its own host thread. Collectives rendezvous on the host,
//                    exchange readiness through CUDA events and move data with
//                    device copies / a fixed-order sum kernel. Exists so that
//                    TP=2/4/8 numerics and the SI executor's collective ordering
//                    can be tested on a single GPU. Not capturable.
#include <nccl.h>

#include <array>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <tuple>

#include "runtime.hpp"

extern "C" int dh_sum_bf16_ptrs(const void* const* srcs, int nsrc, void* dst, long long n,
                                void* stream);
extern "C" int dh_comm_proxy(const void* src, void* dst, long long count, int tp, int mode,
                             int ctas, double link_gbs, void* stream);
extern "C" int dh_sum_f32_ptrs(const float* const* srcs, int nsrc, float* dst, long long n,
                               void* stream);

namespace dh {

int cuda_fail(cudaError_t e, const char* what) {
    return set_error(DH_ERR_CUDA, std::string(cudaGetErrorString(e)) + " at " + what);
}

namespace {

#define RT_NCCL(expr)                                                                   \
    do {                                                                                \
        ncclResult_t rt_n_ = (expr);                                                    \
        if (rt_n_ != ncclSuccess)                                                       \
            return set_error(DH_ERR_NCCL, std::string(ncclGetErrorString(rt_n_)) + " at " #expr); \
    } while (0)

class NcclComm final : public Comm {
public:
    ncclComm_t comm = nullptr;
    float* one = nullptr;  // barrier operand
    ~NcclComm() override {
        if (comm) ncclCommDestroy(comm);
        if (one) cudaFree(one);
    }
    int barrier(cudaStream_t s) override {
        if (!one) RT_CUDA(cudaMalloc(&one, sizeof(float)));
        RT_NCCL(ncclAllReduce(one, one, 1, ncclFloat32, ncclSum, comm, s));
        return DH_OK;
    }
    int all_gather(const void* send, void* recv, size_t count, cudaStream_t s) override {
        RT_NCCL(ncclAllGather(send, recv, count, ncclBfloat16, comm, s));
        return DH_OK;
    }
    int reduce_scatter(const void* send, void* recv, size_t count, cudaStream_t s) override {
        RT_NCCL(ncclReduceScatter(send, recv, count, ncclBfloat16, ncclSum, comm, s));
        return DH_OK;
    }
    int all_reduce_f32(float* buf, size_t count, cudaStream_t s) override {
        RT_NCCL(ncclAllReduce(buf, buf, count, ncclFloat32, ncclSum, comm, s));
        return DH_OK;
    }
    // Grouped point-to-point: per (peer, group) one chunk each way; messages
    // between a pair match in issue order (group ascending on both sides).
    int all_to_all(const void* send, void* recv, size_t chunk, int groups, bool combine,
                   cudaStream_t s) override {
        int size = 0;
        RT_NCCL(ncclCommCount(comm, &size));
        const auto* sb = static_cast<const char*>(send);
        auto* rb = static_cast<char*>(recv);
        const size_t bytes = chunk * 2;
        RT_NCCL(ncclGroupStart());
        for (int p = 0; p < size; ++p) {
            for (int g = 0; g < groups; ++g) {
                const size_t so = combine ? static_cast<size_t>(g) * size + p : static_cast<size_t>(p) * groups + g;
                const size_t ro = combine ? static_cast<size_t>(p) * groups + g : static_cast<size_t>(g) * size + p;
                RT_NCCL(ncclSend(sb + so * bytes, chunk, ncclBfloat16, p, comm, s));
                RT_NCCL(ncclRecv(rb + ro * bytes, chunk, ncclBfloat16, p, comm, s));
            }
        }
        RT_NCCL(ncclGroupEnd());
        return DH_OK;
    }
    bool capturable() const override { return true; }
    const char* name() const override { return "nccl"; }
};

class EmulatedComm final : public Comm {
public:
    int tp, ctas;
    double link_gbs;  // bytes per ns == GB/s
    EmulatedComm(int t, int c, double bw) : tp(t), ctas(c), link_gbs(bw) {}
    int all_gather(const void* send, void* recv, size_t count, cudaStream_t s) override {
        return dh_comm_proxy(send, recv, static_cast<long long>(count), tp, 0, ctas, link_gbs, s);
    }
    int reduce_scatter(const void* send, void* recv, size_t count, cudaStream_t s) override {
        return dh_comm_proxy(send, recv, static_cast<long long>(count), tp, 1, ctas, link_gbs, s);
    }
    int all_reduce_f32(float*, size_t, cudaStream_t) override { return DH_OK; }
    // the a2a's HBM traffic (every byte read and written once) held for the
    // (ep-1)/ep of the buffer that crosses NVLink; the copy keeps layouts fixed
    int all_to_all(const void* send, void* recv, size_t chunk, int groups, bool,
                   cudaStream_t s) override {
        return dh_comm_proxy(send, recv, static_cast<long long>(chunk) * groups * tp, tp, 2, ctas, link_gbs, s);
    }
    bool capturable() const override { return true; }
    const char* name() const override { return "emulated"; }
};

// Pipeline-stage transfers over NCCL (weft SendRecv between W-pipeline
// stages, one GPU each). NCCL matches point-to-point messages per direction
// in issue order, not by tag, and a stage may send a micro-batch's activation
// before it receives an earlier one's gradient (the W schedule does, see
// tests/test_executor_lowering.py). So activations and gradients travel on
// two communicators split from the stage group, each with its own stream:
// within one kind, sender and receiver issue in micro-batch order. A send
// first copies the payload into a staging buffer on the issuing (compute)
// stream, so the next op may overwrite the source, and the NCCL send then
// runs on the kind's stream; it never blocks the compute stream. A receive
// runs on the kind's stream and the compute stream waits for it.
class NcclP2P final : public Comm {
public:
    ncclComm_t base = nullptr;
    std::array<ncclComm_t, 2> kind_comm{};
    std::array<cudaStream_t, 2> kind_stream{};
    std::array<cudaEvent_t, 2> to_kind{}, from_kind{};  // re-recorded per transfer
    ~NcclP2P() override {
        for (auto c : kind_comm)
            if (c) ncclCommDestroy(c);
        if (base) ncclCommDestroy(base);
        for (auto st : kind_stream)
            if (st) cudaStreamDestroy(st);
        for (auto e : to_kind)
            if (e) cudaEventDestroy(e);
        for (auto e : from_kind)
            if (e) cudaEventDestroy(e);
    }
    int init(int rank, int size, const void* unique_id) {
        ncclUniqueId id;
        std::memcpy(&id, unique_id, sizeof(id));
        ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
        RT_NCCL(ncclCommInitRankConfig(&base, size, id, rank, &cfg));
        int lo = 0, hi = 0;
        RT_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        for (int k = 0; k < 2; ++k) {
            ncclConfig_t c2 = NCCL_CONFIG_INITIALIZER;
            RT_NCCL(ncclCommSplit(base, 0, rank, &kind_comm[k], &c2));
            RT_CUDA(cudaStreamCreateWithPriority(&kind_stream[k], cudaStreamNonBlocking, hi));
            RT_CUDA(cudaEventCreateWithFlags(&to_kind[k], cudaEventDisableTiming));
            RT_CUDA(cudaEventCreateWithFlags(&from_kind[k], cudaEventDisableTiming));
        }
        return DH_OK;
    }
    int all_gather(const void*, void*, size_t, cudaStream_t) override { return unsupported(); }
    int reduce_scatter(const void*, void*, size_t, cudaStream_t) override { return unsupported(); }
    int all_reduce_f32(float*, size_t, cudaStream_t) override { return unsupported(); }
    int send(const void* buf, size_t bytes, int peer, int tag, cudaStream_t s) override {
        const int k = tag & 1;  // xfer_tag: 0 activation, 1 gradient (+ 2 * micro-batch)
        void* staging = nullptr;
        RT_CUDA(cudaMallocAsync(&staging, bytes, s));
        RT_CUDA(cudaMemcpyAsync(staging, buf, bytes, cudaMemcpyDeviceToDevice, s));
        RT_CUDA(cudaEventRecord(to_kind[k], s));
        RT_CUDA(cudaStreamWaitEvent(kind_stream[k], to_kind[k], 0));
        RT_NCCL(ncclSend(staging, bytes, ncclChar, peer, kind_comm[k], kind_stream[k]));
        RT_CUDA(cudaFreeAsync(staging, kind_stream[k]));
        return DH_OK;
    }
    int recv(void* buf, size_t bytes, int peer, int tag, cudaStream_t s) override {
        const int k = tag & 1;
        // the destination is free once the compute stream got here
        RT_CUDA(cudaEventRecord(to_kind[k], s));
        RT_CUDA(cudaStreamWaitEvent(kind_stream[k], to_kind[k], 0));
        RT_NCCL(ncclRecv(buf, bytes, ncclChar, peer, kind_comm[k], kind_stream[k]));
        RT_CUDA(cudaEventRecord(from_kind[k], kind_stream[k]));
        RT_CUDA(cudaStreamWaitEvent(s, from_kind[k], 0));
        return DH_OK;
    }
    int sync() override {
        for (auto st : kind_stream) RT_CUDA(cudaStreamSynchronize(st));
        return DH_OK;
    }
    bool capturable() const override { return false; }
    const char* name() const override { return "nccl_p2p"; }

private:
    int unsupported() { return set_error(DH_ERR_CONFIG, "nccl_p2p: pipeline transfers only"); }
};

}  // namespace

std::unique_ptr<Comm> make_nccl_p2p(int rank, int size, const void* unique_id, int* rc) {
    auto c = std::make_unique<NcclP2P>();
    *rc = c->init(rank, size, unique_id);
    if (*rc != DH_OK) return nullptr;
    return c;
}

std::unique_ptr<Comm> make_nccl_comm(int rank, int size, const void* unique_id, int max_ctas,
                                     int* rc) {
    auto c = std::make_unique<NcclComm>();
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    if (max_ctas > 0) {
        cfg.maxCTAs = max_ctas;
        cfg.minCTAs = std::min(max_ctas, 2);
    }
    const ncclResult_t r = ncclCommInitRankConfig(&c->comm, size, id, rank, &cfg);
    if (r != ncclSuccess) {
        *rc = set_error(DH_ERR_NCCL, std::string("ncclCommInitRankConfig: ") + ncclGetErrorString(r));
        c->comm = nullptr;
        return nullptr;
    }
    *rc = DH_OK;
    return c;
}

// ------------------------------------------------------------------ loopback

struct LoopbackGroup {
    int size = 1;
    int device = 0;
    std::mutex mu;
    std::condition_variable cv;
    // current collective: pointers / events posted by each rank
    std::vector<const void*> send;
    std::vector<cudaEvent_t> ready, done;
    int posted_ready = 0, posted_done = 0;
    long long gen_ready = 0, gen_done = 0;
    int refs = 0;
};

namespace {

class LoopbackComm final : public Comm {
public:
    LoopbackGroup* g;
    int rank;
    LoopbackComm(LoopbackGroup* grp, int r) : g(grp), rank(r) {}
    ~LoopbackComm() override {
        std::lock_guard<std::mutex> lk(g->mu);
        cudaEventDestroy(g->ready[rank]);
        cudaEventDestroy(g->done[rank]);
        if (--g->refs == 0) {
            // last rank out frees the group
            delete_group_ = true;
        }
    }
    bool delete_group_ = false;

    // Phase 1: publish send buffer + readiness event, wait for every rank.
    int rendezvous_ready(const void* send, cudaStream_t s) {
        RT_CUDA(cudaEventRecord(g->ready[rank], s));
        std::unique_lock<std::mutex> lk(g->mu);
        g->send[rank] = send;
        const long long gen = g->gen_ready;
        if (++g->posted_ready == g->size) {
            g->posted_ready = 0;
            ++g->gen_ready;
            g->cv.notify_all();
        } else {
            g->cv.wait(lk, [&] { return g->gen_ready != gen; });
        }
        return DH_OK;
    }
    // Phase 2: after pulling, publish completion and make this stream wait for
    // every peer's pulls (peers read our send buffer).
    int rendezvous_done(cudaStream_t s) {
        RT_CUDA(cudaEventRecord(g->done[rank], s));
        std::unique_lock<std::mutex> lk(g->mu);
        const long long gen = g->gen_done;
        if (++g->posted_done == g->size) {
            g->posted_done = 0;
            ++g->gen_done;
            g->cv.notify_all();
        } else {
            g->cv.wait(lk, [&] { return g->gen_done != gen; });
        }
        lk.unlock();
        for (int p = 0; p < g->size; ++p) {
            if (p != rank) RT_CUDA(cudaStreamWaitEvent(s, g->done[p], 0));
        }
        return DH_OK;
    }

    int all_gather(const void* send, void* recv, size_t count, cudaStream_t s) override {
        RT_TRY(rendezvous_ready(send, s));
        for (int p = 0; p < g->size; ++p) {
            if (p != rank) RT_CUDA(cudaStreamWaitEvent(s, g->ready[p], 0));
            RT_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + p * count * 2, g->send[p], count * 2,
                                    cudaMemcpyDeviceToDevice, s));
        }
        return rendezvous_done(s);
    }
    int reduce_scatter(const void* send, void* recv, size_t count, cudaStream_t s) override {
        RT_TRY(rendezvous_ready(send, s));
        std::vector<const void*> srcs(g->size);
        for (int p = 0; p < g->size; ++p) {
            if (p != rank) RT_CUDA(cudaStreamWaitEvent(s, g->ready[p], 0));
            srcs[p] = static_cast<const char*>(g->send[p]) + rank * count * 2;
        }
        RT_TRY(dh_sum_bf16_ptrs(srcs.data(), g->size, recv, static_cast<long long>(count), s));
        return rendezvous_done(s);
    }
    int all_reduce_f32(float* buf, size_t count, cudaStream_t s) override {
        // Sum into a private copy first so no rank reads a partially reduced peer.
        float* tmp = nullptr;
        RT_CUDA(cudaMallocAsync(&tmp, count * 4, s));
        RT_TRY(rendezvous_ready(buf, s));
        std::vector<const float*> srcs(g->size);
        for (int p = 0; p < g->size; ++p) {
            if (p != rank) RT_CUDA(cudaStreamWaitEvent(s, g->ready[p], 0));
            srcs[p] = static_cast<const float*>(g->send[p]);
        }
        RT_TRY(dh_sum_f32_ptrs(srcs.data(), g->size, tmp, static_cast<long long>(count), s));
        RT_TRY(rendezvous_done(s));
        RT_CUDA(cudaMemcpyAsync(buf, tmp, count * 4, cudaMemcpyDeviceToDevice, s));
        RT_CUDA(cudaFreeAsync(tmp, s));
        // A second barrier: peers must not read our buffer after we overwrite it.
        RT_TRY(rendezvous_ready(buf, s));
        return rendezvous_done(s);
    }
    int all_to_all(const void* send, void* recv, size_t chunk, int groups, bool combine,
                   cudaStream_t s) override {
        RT_TRY(rendezvous_ready(send, s));
        const size_t bytes = chunk * 2;
        const int size = g->size;
        for (int p = 0; p < size; ++p) {
            if (p != rank) RT_CUDA(cudaStreamWaitEvent(s, g->ready[p], 0));
            for (int q = 0; q < groups; ++q) {
                // pull peer p's chunk addressed to this rank
                const size_t so = combine ? static_cast<size_t>(q) * size + rank : static_cast<size_t>(rank) * groups + q;
                const size_t ro = combine ? static_cast<size_t>(p) * groups + q : static_cast<size_t>(q) * size + p;
                RT_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + ro * bytes,
                                        static_cast<const char*>(g->send[p]) + so * bytes, bytes,
                                        cudaMemcpyDeviceToDevice, s));
            }
        }
        return rendezvous_done(s);
    }
    bool capturable() const override { return false; }
    const char* name() const override { return "loopback"; }
};

}  // namespace

// ------------------------------------------------------------------ loopback pipeline transfers

// One mailbox per (src stage, dst stage, tag). A send copies the payload into
// a private staging buffer on the sender's stream and posts it with an event;
// the matching recv (program order) waits for that event, copies out and frees
// the staging buffer on its own stream. Sends never wait for the receiver, so
// any schedule whose transfers follow its data dependencies cannot deadlock.
struct P2PGroup {
    std::mutex mu;
    std::condition_variable cv;
    struct Msg {
        void* staging;
        size_t bytes;
        cudaEvent_t ready;
    };
    std::map<std::tuple<int, int, int>, std::deque<Msg>> box;  // (src, dst, tag)
};

namespace {

class LoopbackP2P final : public Comm {
public:
    LoopbackP2P(std::shared_ptr<P2PGroup> g, int r) : g_(std::move(g)), rank_(r) {}
    int all_gather(const void*, void*, size_t, cudaStream_t) override { return unsupported(); }
    int reduce_scatter(const void*, void*, size_t, cudaStream_t) override { return unsupported(); }
    int all_reduce_f32(float*, size_t, cudaStream_t) override { return unsupported(); }
    int send(const void* buf, size_t bytes, int peer, int tag, cudaStream_t s) override {
        P2PGroup::Msg msg{nullptr, bytes, nullptr};
        RT_CUDA(cudaMallocAsync(&msg.staging, bytes, s));
        RT_CUDA(cudaMemcpyAsync(msg.staging, buf, bytes, cudaMemcpyDeviceToDevice, s));
        RT_CUDA(cudaEventCreateWithFlags(&msg.ready, cudaEventDisableTiming));
        RT_CUDA(cudaEventRecord(msg.ready, s));
        std::lock_guard<std::mutex> lk(g_->mu);
        g_->box[{rank_, peer, tag}].push_back(msg);
        g_->cv.notify_all();
        return DH_OK;
    }
    int recv(void* buf, size_t bytes, int peer, int tag, cudaStream_t s) override {
        P2PGroup::Msg msg;
        {
            std::unique_lock<std::mutex> lk(g_->mu);
            auto& q = g_->box[{peer, rank_, tag}];
            g_->cv.wait(lk, [&] { return !q.empty(); });
            msg = q.front();
            q.pop_front();
        }
        if (msg.bytes != bytes) return set_error(DH_ERR_OTHER, "pipeline transfer: size mismatch between stages");
        RT_CUDA(cudaStreamWaitEvent(s, msg.ready, 0));
        RT_CUDA(cudaEventDestroy(msg.ready));
        RT_CUDA(cudaMemcpyAsync(buf, msg.staging, bytes, cudaMemcpyDeviceToDevice, s));
        RT_CUDA(cudaFreeAsync(msg.staging, s));
        return DH_OK;
    }
    bool capturable() const override { return false; }
    const char* name() const override { return "loopback_p2p"; }

private:
    int unsupported() { return set_error(DH_ERR_CONFIG, "loopback_p2p: pipeline transfers only"); }
    std::shared_ptr<P2PGroup> g_;
    int rank_;
};

}  // namespace

std::unique_ptr<Comm> make_loopback_comm(LoopbackGroup* group, int rank, int* rc) {
    auto c = std::make_unique<LoopbackComm>(group, rank);
    if (cudaEventCreateWithFlags(&group->ready[rank], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&group->done[rank], cudaEventDisableTiming) != cudaSuccess) {
        *rc = set_error(DH_ERR_CUDA, "loopback: event creation failed");
        return nullptr;
    }
    *rc = DH_OK;
    return c;
}

}  // namespace dh

// ------------------------------------------------------------------ C ABI

namespace {

int init_streams(dh::Ctx* c) {
    RT_CUDA(cudaSetDevice(c->device));
    int lo = 0, hi = 0;
    RT_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    for (int l = 0; l < dh::kLanes; ++l) {
        // hi is the numerically smallest = highest priority
        RT_CUDA(cudaStreamCreateWithPriority(&c->lane[l], cudaStreamNonBlocking, l == 0 ? lo : hi));
    }
    RT_CUDA(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, c->device));
    return DH_OK;
}

}  // namespace

extern "C" {

int dh_nccl_unique_id(void* out128) {
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return dh::set_error(DH_ERR_NCCL, ncclGetErrorString(r));
    std::memcpy(out128, &id, sizeof(id));
    return DH_OK;
}

int dh_ctx_create(int device, int tp_rank, int tp_size, const void* nccl_unique_id,
                  int nccl_max_ctas, dh_ctx** out) {
    if (!out || tp_size < 1 || tp_rank < 0 || tp_rank >= tp_size)
        return dh::set_error(DH_ERR_INVALID, "dh_ctx_create: bad rank/size");
    auto* c = new dh_ctx();
    c->device = device;
    c->tp_rank = tp_rank;
    c->tp_size = tp_size;
    c->comm_ctas = nccl_max_ctas;
    int rc = init_streams(c);
    // tp_size == 1 with an id: a one-rank NCCL communicator (the model issues no
    // collectives at TP = 1; dh_comm_run exercises the NCCL path on one GPU)
    if (rc == DH_OK && (tp_size > 1 || nccl_unique_id)) {
        if (!nccl_unique_id) {
            rc = dh::set_error(DH_ERR_INVALID, "dh_ctx_create: tp_size > 1 needs an ncclUniqueId");
        } else {
            c->comm = dh::make_nccl_comm(tp_rank, tp_size, nccl_unique_id, nccl_max_ctas, &rc);
        }
    }
    if (rc != DH_OK) {
        dh_ctx_destroy(c);
        return rc;
    }
    *out = c;
    return DH_OK;
}

int dh_ctx_create_pp(int device, int tp_rank, int tp_size, const void* tp_unique_id, int pp_rank, int pp_size,
                     const void* pp_unique_id, int nccl_max_ctas, dh_ctx** out) {
    if (!out || pp_size < 1 || pp_rank < 0 || pp_rank >= pp_size || (pp_size > 1 && !pp_unique_id))
        return dh::set_error(DH_ERR_INVALID, "dh_ctx_create_pp: bad stage rank/size or missing ncclUniqueId");
    dh_ctx* c = nullptr;
    RT_TRY(dh_ctx_create(device, tp_rank, tp_size, tp_unique_id, nccl_max_ctas, &c));
    c->pp_rank = pp_rank;
    c->pp_size = pp_size;
    if (pp_size > 1) {
        int rc = DH_OK;
        c->pp = dh::make_nccl_p2p(pp_rank, pp_size, pp_unique_id, &rc);
        if (rc != DH_OK) {
            dh_ctx_destroy(c);
            return rc;
        }
    }
    *out = c;
    return DH_OK;
}

int dh_ctx_create_emulated(int device, int tp_size, int comm_ctas, double link_gbs, dh_ctx** out) {
    if (!out || tp_size < 2) return dh::set_error(DH_ERR_INVALID, "emulated: tp_size >= 2 required");
    auto* c = new dh_ctx();
    c->device = device;
    c->tp_rank = 0;
    c->tp_size = tp_size;
    c->comm_ctas = comm_ctas;
    const int rc = init_streams(c);
    if (rc != DH_OK) {
        dh_ctx_destroy(c);
        return rc;
    }
    c->comm = std::make_unique<dh::EmulatedComm>(tp_size, comm_ctas > 0 ? comm_ctas : 16, link_gbs);
    *out = c;
    return DH_OK;
}

int dh_loopback_pp_group_create(int device, int pp_size, dh_ctx** ctxs_out) {
    if (pp_size < 1 || !ctxs_out) return dh::set_error(DH_ERR_INVALID, "loopback pp: bad size");
    auto g = std::make_shared<dh::P2PGroup>();
    for (int r = 0; r < pp_size; ++r) {
        auto* c = new dh_ctx();
        c->device = device;
        c->pp_rank = r;
        c->pp_size = pp_size;
        const int rc = init_streams(c);
        if (rc != DH_OK) return rc;
        if (pp_size > 1) c->pp = std::make_unique<dh::LoopbackP2P>(g, r);
        ctxs_out[r] = c;
    }
    return DH_OK;
}

int dh_loopback_group_create(int device, int tp_size, dh_ctx** ctxs_out) {
    if (tp_size < 1 || !ctxs_out) return dh::set_error(DH_ERR_INVALID, "loopback: bad size");
    auto* g = new dh::LoopbackGroup();
    g->size = tp_size;
    g->device = device;
    g->send.assign(tp_size, nullptr);
    g->ready.assign(tp_size, nullptr);
    g->done.assign(tp_size, nullptr);
    g->refs = tp_size;
    for (int r = 0; r < tp_size; ++r) {
        auto* c = new dh_ctx();
        c->device = device;
        c->tp_rank = r;
        c->tp_size = tp_size;
        int rc = init_streams(c);
        if (rc == DH_OK && tp_size > 1) c->comm = dh::make_loopback_comm(g, r, &rc);
        if (rc != DH_OK) return rc;
        ctxs_out[r] = c;
    }
    if (tp_size == 1) delete g;
    return DH_OK;
}

int dh_ctx_destroy(dh_ctx* c) {
    if (!c) return DH_OK;
    cudaSetDevice(c->device);
    dh::LoopbackGroup* grp = nullptr;
    bool last = false;
    if (c->comm && std::strcmp(c->comm->name(), "loopback") == 0) {
        auto* lb = static_cast<dh::LoopbackComm*>(c->comm.get());
        grp = lb->g;
        c->comm.reset();  // destructor decrements refs
        std::lock_guard<std::mutex> lk(grp->mu);
        last = grp->refs == 0;
    }
    c->comm.reset();
    for (auto& s : c->lane) {
        if (s) cudaStreamDestroy(s);
    }
    delete c;
    if (last) delete grp;
    return DH_OK;
}

int dh_comm_run(dh_ctx* c, int op, const void* send, void* recv, long long count, int lane) {
    if (!c || lane < 0 || lane >= dh::kLanes || count < 0)
        return dh::set_error(DH_ERR_INVALID, "dh_comm_run: bad context, lane or count");
    if (!c->comm) return dh::set_error(DH_ERR_CONFIG, "dh_comm_run: the context has no TP/EP communicator");
    RT_CUDA(cudaSetDevice(c->device));
    cudaStream_t s = c->lane[lane];
    const auto n = static_cast<size_t>(count);
    switch (op) {
        case DH_COMM_ALL_GATHER: return c->comm->all_gather(send, recv, n, s);
        case DH_COMM_REDUCE_SCATTER: return c->comm->reduce_scatter(send, recv, n, s);
        case DH_COMM_ALL_REDUCE_F32:
            if (send != recv) RT_CUDA(cudaMemcpyAsync(recv, send, n * 4, cudaMemcpyDeviceToDevice, s));
            return c->comm->all_reduce_f32(static_cast<float*>(recv), n, s);
        case DH_COMM_ALL_TO_ALL: return c->comm->all_to_all(send, recv, n, 1, false, s);
        default: return dh::set_error(DH_ERR_INVALID, "dh_comm_run: unknown op");
    }
}

void* dh_ctx_stream(dh_ctx* c, int lane) {
    if (!c || lane < 0 || lane >= dh::kLanes) return nullptr;
    return c->lane[lane];
}

}  // extern "C"
