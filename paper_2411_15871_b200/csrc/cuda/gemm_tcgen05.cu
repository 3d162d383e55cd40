// Persistent, warp-specialised bf16 GEMM for sm_100a on tcgen05 / TMEM / TMA.
//
//   D(m, n) (+)= sum_k A(m, k) * B(n, k)
//
// A and B are each either K-major (row-major [rows, K]: the forward GEMMs) or
// MN-major (K rows of contiguous M / N: the dgrad B operand and both wgrad
// operands), so every GEMM of the Megatron TP+SP layer — forward, dgrad and
// wgrad — runs without a transpose pass. D is bf16 (optionally accumulated,
// beta = 1) or fp32 (accumulated: the fp32 main-grad of wgrad).
//
// CTA = 6 warps:  warp 0  TMA producer (one lane)
//                 warp 1  TMEM allocator + tcgen05.mma issuer (one elected lane)
//                 warps 2-5 epilogue: tcgen05.ld TMEM -> registers -> swizzled smem
//                           staging (2 x 16 KB) -> TMA store (bf16) or TMA
//                           reduce-add (fp32 main-grad accumulation); the legacy
//                           register path remains for bf16 accumulate.
// Tile BM=128 x BN (128, 192 or 256, picked per shape for wave quantisation) x
// BK=64, SWIZZLE_128B smem operands, a 4-6 stage TMA ring (full/empty
// mbarriers) and a double-buffered TMEM accumulator (2 x BN fp32 columns) so
// the epilogue of tile i overlaps the main loop of tile i+1. The grid is persistent: min(tiles, SMs allowed), which
// is how the SI executor caps a GEMM's SM footprint next to NCCL kernels.
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "dh_capi.h"

#ifdef DH_GEMM_TRACE
// per-CTA globaltimer stamps of the last pair-kernel launch (tools/gemm_trace.py):
// [0] entry [1] prologue done [2] first stage consumed by the MMA [3] last
// accumulator ready [4] last store issued and drained [5] exit
__device__ unsigned long long g_gemm_trace[512 * 8];
extern "C" int dh_gemm_trace_read(unsigned long long* out, int n) {
    return cudaMemcpyFromSymbol(out, g_gemm_trace, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : 1;
}
#define GTR(i, cond)                                                                     \
    do {                                                                                 \
        if (cond) {                                                                      \
            unsigned long long t_;                                                       \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                       \
            g_gemm_trace[blockIdx.x * 8 + (i)] = t_;                                     \
        }                                                                                \
    } while (0)
#else
#define GTR(i, cond) do { } while (0)
#endif

namespace dh {
namespace {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kThreads = 192;

enum Epi {
    kEpiStoreBf16 = 0,
    kEpiAddF32 = 1,
    kEpiDirect = 2,
    kEpiAddBf16 = 3,
    kEpiSwiGLUFwd = 4,  // D = bf16(acc), D2 = swiglu(aux0, D) or swiglu(D, aux0) (aux_is_up)
    kEpiSwiGLUBwd = 5,  // acc = d_act: D = d_gate, D2 = d_up from (aux0 = gate, aux1 = up)
    kEpiSwiGLUPair = 6, // mlp_gate | mlp_up in one GEMM: the CTA pair's two B halves are Wg and Wu rows
                        // of the same 128 features, so the accumulator holds gate | up side by side;
                        // D = gate, D2 = up, X0 (a store map here) = act = silu(gate) * up
};

template <int BN>
struct GemmCfg {
    static constexpr int kStageA = BM * BK * 2;
    static constexpr int kStageB = BN * BK * 2;
    static constexpr int kStageBytes = kStageA + kStageB;
    static constexpr int kStages = BN == 128 ? 6 : 4;
    static constexpr int kTmemCols = BN == 128 ? 256 : 512;
    static constexpr int kStaging = 2 * 16384;
    static constexpr int kSmemBytes = kStages * kStageBytes + kStaging + 1024 /*align*/ + 256 /*barriers*/;
};

struct KParams {
    void* d;
    long long ldd;
    int m, n, k;
    int accumulate;
    int tiles_m, tiles_n;
    const __nv_bfloat16* aux0;  // fused SwiGLU epilogues: [m, n] bf16 operands, row pitch ld_aux
    const __nv_bfloat16* aux1;
    long long ld_aux;
    int aux_is_up;  // kEpiSwiGLUFwd: acc is the gate projection and aux0 holds up
    // Raster order of the persistent tile loop (tile_coords): groups of `group`
    // m-tiles (b_resident == 0: their A panels stay in L2 while every n-tile
    // streams past) or of `group` n-tiles (b_resident == 1), the grouped
    // dimension fastest inside a group.
    int b_resident, group;
    // two-segment launches of the CTA-pair kernel (maps tma_x0 / tma_x1 / tma_d2,
    // otherwise the fused epilogues' aux maps): k-blocks >= kb_split read A2 / B2
    // (K-concatenation); 256-row m-tiles >= mt_split read A2 and store to D2
    // (M-concatenation). Past the end = one segment.
    int kb_split, mt_split;
};

void raster_for(KParams& p, int bm, int bn, int k);

// Tile index -> (m-tile, n-tile) in the raster order chosen by the host
// (raster_for): the operand panels a group touches stay L2-resident while the
// other operand's panels stream through once per group.
__device__ __forceinline__ void tile_coords(int tile, const KParams& p, int* mi, int* ni) {
    const int fast = p.b_resident ? p.tiles_n : p.tiles_m;  // grouped dimension
    const int slow = p.b_resident ? p.tiles_m : p.tiles_n;
    const int per_group = p.group * slow;
    const int g = tile / per_group, r = tile - g * per_group;
    const int width = min(p.group, fast - g * p.group);
    const int f = g * p.group + r % width, sl = r / width;
    *mi = p.b_resident ? sl : f;
    *ni = p.b_resident ? f : sl;
}

template <int BN, bool A_MN, bool B_MN, int EPI, bool D_F32>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tcgen05_kernel(const __grid_constant__ CUtensorMap tma_a,
                        const __grid_constant__ CUtensorMap tma_b,
                        const __grid_constant__ CUtensorMap tma_d, const KParams p) {
    using Cfg = GemmCfg<BN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + Cfg::kStages * Cfg::kStageA;
    uint8_t* staging = smem + Cfg::kStages * Cfg::kStageBytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(staging + Cfg::kStaging);
    uint64_t* empty = full + Cfg::kStages;
    uint64_t* tfull = empty + Cfg::kStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const int num_tiles = p.tiles_m * p.tiles_n;
    const int num_kb = (p.k + BK - 1) / BK;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tma_a);
        tma_prefetch(&tma_b);
        if constexpr (EPI != kEpiDirect) tma_prefetch(&tma_d);
        for (int s = 0; s < Cfg::kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 128);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, Cfg::kTmemCols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                int mi, ni;
                tile_coords(tile, p, &mi, &ni);
                const int m0 = mi * BM;
                const int n0 = ni * BN;
                for (int kb = 0; kb < num_kb; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_expect_tx(&full[stage], Cfg::kStageBytes);
                    uint8_t* a_dst = sA + stage * Cfg::kStageA;
                    uint8_t* b_dst = sB + stage * Cfg::kStageB;
                    const int k0 = kb * BK;
                    if constexpr (A_MN) {
#pragma unroll
                        for (int i = 0; i < BM / 64; ++i)
                            tma_load_2d(a_dst + i * (BK * 128), &tma_a, &full[stage], m0 + 64 * i, k0);
                    } else {
                        tma_load_2d(a_dst, &tma_a, &full[stage], k0, m0);
                    }
                    if constexpr (B_MN) {
#pragma unroll
                        for (int i = 0; i < BN / 64; ++i)
                            tma_load_2d(b_dst + i * (BK * 128), &tma_b, &full[stage], n0 + 64 * i, k0);
                    } else {
                        tma_load_2d(b_dst, &tma_b, &full[stage], k0, n0);
                    }
                    if (++stage == Cfg::kStages) stage = 0, phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        constexpr uint32_t idesc = umma_idesc_bf16(BM, BN, A_MN, B_MN);
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            mbar_wait(&tempty[acc], acc_phase ^ 1);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + acc * BN;
            for (int kb = 0; kb < num_kb; ++kb) {
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t a_addr = smem_u32(sA + stage * Cfg::kStageA);
                    const uint32_t b_addr = smem_u32(sB + stage * Cfg::kStageB);
#pragma unroll
                    for (int kk = 0; kk < BK / 16; ++kk) {
                        // K-major: advance 16 elements = 32 B inside the swizzled row.
                        // MN-major: advance two 8-row k atoms = 2048 B.
                        const uint64_t a_desc =
                            A_MN ? umma_desc_sw128(a_addr + kk * 2048, BK * 128, 1024)
                                 : umma_desc_sw128(a_addr + kk * 32, 16, 1024);
                        const uint64_t b_desc =
                            B_MN ? umma_desc_sw128(b_addr + kk * 2048, BK * 128, 1024)
                                 : umma_desc_sw128(b_addr + kk * 32, 16, 1024);
                        tc_mma_bf16(d_tmem, a_desc, b_desc, idesc, (kb | kk) != 0);
                    }
                    tc_commit(&empty[stage]);
                    if (kb == num_kb - 1) tc_commit(&tfull[acc]);
                }
                __syncwarp();
                if (++stage == Cfg::kStages) stage = 0, phase ^= 1;
            }
            if (++acc == 2) acc = 0, acc_phase ^= 1;
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const int quad = warp & 3;  // TMEM lane quadrant this warp may access
        const int r = quad * 32 + lane;        // row within the tile
        const bool leader = warp == 4 && lane == 0;  // issues the TMA stores
        const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
        int acc = 0;
        uint32_t acc_phase = 0;
        int chunk = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            int mi, ni;
            tile_coords(tile, p, &mi, &ni);
            const int m0 = mi * BM;
            const int n0 = ni * BN;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            if constexpr (EPI == kEpiStoreBf16) {
                // 64-column chunks: 128 rows x 128 B, SW128-swizzled, TMA-stored.
#pragma unroll 1
                for (int c = 0; c < BN / 64; ++c, ++chunk) {
                    uint8_t* stg = staging + (chunk & 1) * 16384;
                    if (leader) bulk_wait_read<1>();  // store from 2 chunks ago has left stg
                    named_barrier(2, 128);
                    uint32_t v0[32], v1[32];
                    tmem_ld32(tmem_base + lane_off + acc * BN + c * 64, v0);
                    tmem_ld32(tmem_base + lane_off + acc * BN + c * 64 + 32, v1);
                    tmem_ld_wait();
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        float f[8];
#pragma unroll
                        for (int t = 0; t < 8; ++t)
                            f[t] = __uint_as_float(u < 4 ? v0[u * 8 + t] : v1[(u - 4) * 8 + t]);
                        *reinterpret_cast<uint4*>(stg + r * 128 + ((u ^ (r & 7)) << 4)) = pack8(f);
                    }
                    fence_async_shared();
                    named_barrier(2, 128);
                    if (leader) {
                        tma_store_2d(&tma_d, stg, n0 + c * 64, m0);
                        bulk_commit();
                    }
                }
            } else if constexpr (EPI == kEpiAddF32) {
                // 32-column fp32 chunks, TMA reduce-add into the fp32 main grad.
#pragma unroll 1
                for (int c = 0; c < BN / 32; ++c, ++chunk) {
                    uint8_t* stg = staging + (chunk & 1) * 16384;
                    if (leader) bulk_wait_read<1>();
                    named_barrier(2, 128);
                    uint32_t v[32];
                    tmem_ld32(tmem_base + lane_off + acc * BN + c * 32, v);
                    tmem_ld_wait();
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        *reinterpret_cast<uint4*>(stg + r * 128 + ((u ^ (r & 7)) << 4)) =
                            make_uint4(v[u * 4], v[u * 4 + 1], v[u * 4 + 2], v[u * 4 + 3]);
                    }
                    fence_async_shared();
                    named_barrier(2, 128);
                    if (leader) {
                        tma_reduce_add_2d(&tma_d, stg, n0 + c * 32, m0);
                        bulk_commit();
                    }
                }
            } else {
                const int row = m0 + r;
                const bool row_ok = row < p.m;
#pragma unroll 1
                for (int c = 0; c < BN / 32; ++c) {
                    uint32_t rr[32];
                    tmem_ld32(tmem_base + lane_off + acc * BN + c * 32, rr);
                    tmem_ld_wait();
                    const int col0 = n0 + c * 32;
                    if (!row_ok || col0 >= p.n) continue;
                    const bool full_chunk = col0 + 32 <= p.n;
                    if constexpr (D_F32) {
                        float* drow = reinterpret_cast<float*>(p.d) + static_cast<long long>(row) * p.ldd + col0;
                        for (int j = 0; j < 32 && col0 + j < p.n; ++j) {
                            float x = __uint_as_float(rr[j]);
                            if (p.accumulate) x += drow[j];
                            drow[j] = x;
                        }
                    } else {
                        __nv_bfloat16* drow =
                            reinterpret_cast<__nv_bfloat16*>(p.d) + static_cast<long long>(row) * p.ldd + col0;
                        if (full_chunk) {
#pragma unroll
                            for (int j = 0; j < 32; j += 8) {
                                float f[8];
#pragma unroll
                                for (int t = 0; t < 8; ++t) f[t] = __uint_as_float(rr[j + t]);
                                if (p.accumulate) {
                                    float o[8];
                                    unpack8(*reinterpret_cast<const uint4*>(drow + j), o);
#pragma unroll
                                    for (int t = 0; t < 8; ++t) f[t] += o[t];
                                }
                                *reinterpret_cast<uint4*>(drow + j) = pack8(f);
                            }
                        } else {
                            for (int j = 0; j < 32 && col0 + j < p.n; ++j) {
                                float x = __uint_as_float(rr[j]);
                                if (p.accumulate) x += __bfloat162float(drow[j]);
                                drow[j] = __float2bfloat16(x);
                            }
                        }
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(&tempty[acc]);
            if (++acc == 2) acc = 0, acc_phase ^= 1;
        }
        if constexpr (EPI != kEpiDirect) {
            if (leader) bulk_wait<0>();
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem_base, Cfg::kTmemCols);
    }
}

// ---------------------------------------------------------------------------
// CTA-pair variant (tcgen05 cta_group::2): a 256 x PBN tile per pair of SMs
// (PBN 256, 192 or 128: the narrower pair tiles fill the SMs on the skinny
// TP-sharded GEMMs). Each CTA stages its own 128 rows of A and its half
// (PBN/2 rows) of B per 64-wide k block (32 KB/stage for PBN 256 instead of
// 48 KB for 128 x 256 on one SM: 1.5x less L2->SM traffic per FLOP); the even
// CTA issues M256 N<PBN> MMAs that read both CTAs' smem and write both CTAs'
// TMEM (128 lanes x PBN columns each). TMA loads of both CTAs complete on the
// leader's full barrier; MMA commits multicast to both CTAs' empty /
// accumulator-full barriers; both epilogues release the accumulator on the
// leader's tempty barrier.

template <int PBN, bool FUSED = false>
struct PairCfg {
    static constexpr int kHalfB = PBN / 2;                    // B rows per CTA
    static constexpr int kStageA = BM * BK * 2;               // 16 KB
    static constexpr int kStageB = kHalfB * BK * 2;           // 16 / 12 / 8 KB
    static constexpr int kStage = kStageA + kStageB;
    static constexpr int kStaging = (FUSED ? 4 : 2) * 16384;  // fused: two outputs per chunk
    static constexpr int kBudget = 232448 - kStaging - 1024 - 256;  // 227 KB opt-in smem per CTA
    static constexpr int kStages = kBudget / kStage < 8 ? kBudget / kStage : 8;
    static constexpr int kSmem = kStages * kStage + kStaging + 1024 + 256;
};

// Fused SwiGLU epilogues run 8 epilogue warps (two per TMEM lane quadrant, each
// on half of a 64-column chunk): their element math would otherwise be slower
// than the main loop it has to hide behind.
template <int EPI>
constexpr int pair_threads() {
    return EPI == kEpiSwiGLUFwd || EPI == kEpiSwiGLUBwd || EPI == kEpiSwiGLUPair ? 320 : kThreads;
}

template <int PBN, bool A_MN, bool B_MN, int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(pair_threads<EPI>(), 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                     const __grid_constant__ CUtensorMap tma_d, const __grid_constant__ CUtensorMap tma_d2,
                     const __grid_constant__ CUtensorMap tma_x0, const __grid_constant__ CUtensorMap tma_x1,
                     const KParams p) {
    constexpr bool kFused = EPI == kEpiSwiGLUFwd || EPI == kEpiSwiGLUBwd;
    constexpr bool kPairEpi = EPI == kEpiSwiGLUPair;
    static_assert(!kPairEpi || PBN == 256, "the gate | up pair epilogue uses 256-wide pair tiles");
    using C = PairCfg<PBN, kFused || kPairEpi>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + C::kStages * C::kStageA;
    uint8_t* staging = smem + C::kStages * C::kStage;
    uint64_t* full = reinterpret_cast<uint64_t*>(staging + C::kStaging);
    uint64_t* empty = full + C::kStages;
    uint64_t* tfull = empty + C::kStages;
    uint64_t* tempty = tfull + 2;
    uint64_t* xfull = tempty + 2;  // [2] fused epilogues: aux tiles of a staging set landed
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xfull + 2);

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int tiles_m = p.tiles_m;  // in units of 256 rows
    const int num_tiles = tiles_m * p.tiles_n;
    const int num_kb = (p.k + BK - 1) / BK;
    GTR(0, threadIdx.x == 0);

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tma_a);
        tma_prefetch(&tma_b);
        tma_prefetch(&tma_d);
        if constexpr (kFused) tma_prefetch(&tma_d2);
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 2 * (pair_threads<EPI>() - 64));  // every epilogue thread of both CTAs
            mbar_init(&xfull[b], 1);
        }
        if constexpr (kFused || kPairEpi) {
            tma_prefetch(&tma_x0);
            if constexpr (EPI != kEpiSwiGLUFwd) tma_prefetch(&tma_x1);
        } else if (p.kb_split < num_kb || p.mt_split < tiles_m) {
            tma_prefetch(&tma_x0);
            tma_prefetch(&tma_x1);
            tma_prefetch(&tma_d2);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc_pair(tmem_slot, 512);
    tc_fence_before();
    cluster_sync();  // barriers of both CTAs initialised before any remote arrive
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    GTR(1, threadIdx.x == 0);

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = pair; tile < num_tiles; tile += npairs) {
                int mi, ni;
                tile_coords(tile, p, &mi, &ni);
                const int m0 = mi * 256 + rank * BM;             // this CTA's A rows
                // this CTA's B half (pair epilogue: Wg / Wu rows of the tile's 128 features)
                const int n0 = kPairEpi ? ni * 128 : ni * PBN + rank * C::kHalfB;
                for (int kb = 0; kb < num_kb; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (leader) mbar_expect_tx(&full[stage], 2 * C::kStage);
                    const uint32_t bar = leader_addr(&full[stage]);
                    uint8_t* a_dst = sA + stage * C::kStageA;
                    uint8_t* b_dst = sB + stage * C::kStageB;
                    // second segment: K-concatenation (A2, B2) or M-concatenation (A2)
                    const bool ks2 = kb >= p.kb_split, ms2 = mi >= p.mt_split;
                    const CUtensorMap* ta = ks2 || ms2 ? &tma_x0 : &tma_a;
                    const CUtensorMap* tb = ks2 || (kPairEpi && rank) ? &tma_x1 : &tma_b;
                    const int k0 = (ks2 ? kb - p.kb_split : kb) * BK;
                    const int ma = ms2 ? m0 - p.mt_split * 256 : m0;
                    if constexpr (A_MN) {
                        tma_load_2d_pair(a_dst, ta, bar, ma, k0);
                        tma_load_2d_pair(a_dst + BK * 128, ta, bar, ma + 64, k0);
                    } else {
                        tma_load_2d_pair(a_dst, ta, bar, k0, ma);
                    }
                    if constexpr (B_MN) {
#pragma unroll
                        for (int i = 0; i < C::kHalfB / 64; ++i)
                            tma_load_2d_pair(b_dst + i * BK * 128, tb, bar, n0 + i * 64, k0);
                    } else {
                        tma_load_2d_pair(b_dst, tb, bar, k0, n0);
                    }
                    if (++stage == C::kStages) stage = 0, phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        if (leader) {
            constexpr uint32_t idesc = umma_idesc_bf16(256, PBN, A_MN, B_MN);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int tile = pair; tile < num_tiles; tile += npairs) {
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * PBN;
                for (int kb = 0; kb < num_kb; ++kb) {
                    mbar_wait(&full[stage], phase);
                    GTR(2, lane == 0 && tile == pair && kb == 0);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t a_addr = smem_u32(sA + stage * C::kStageA);
                        const uint32_t b_addr = smem_u32(sB + stage * C::kStageB);
#pragma unroll
                        for (int kk = 0; kk < BK / 16; ++kk) {
                            const uint64_t a_desc = A_MN ? umma_desc_sw128(a_addr + kk * 2048, BK * 128, 1024)
                                                         : umma_desc_sw128(a_addr + kk * 32, 16, 1024);
                            const uint64_t b_desc = B_MN ? umma_desc_sw128(b_addr + kk * 2048, BK * 128, 1024)
                                                         : umma_desc_sw128(b_addr + kk * 32, 16, 1024);
                            tc_mma_bf16_pair(d_tmem, a_desc, b_desc, idesc, (kb | kk) != 0);
                        }
                        tc_commit_pair_mc(&empty[stage]);
                        if (kb == num_kb - 1) tc_commit_pair_mc(&tfull[acc]);
                    }
                    __syncwarp();
                    if (++stage == C::kStages) stage = 0, phase ^= 1;
                }
                if (++acc == 2) acc = 0, acc_phase ^= 1;
            }
        }
    } else {
        const int quad = warp & 3;
        const int r = quad * 32 + lane;
        const bool store_leader = warp == 4 && lane == 0;
        const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
        const uint32_t tempty_leader[2] = {leader_addr(&tempty[0]), leader_addr(&tempty[1])};
        int acc = 0;
        uint32_t acc_phase = 0;
        int chunk = 0;
        for (int tile = pair; tile < num_tiles; tile += npairs) {
            int mi, ni;
            tile_coords(tile, p, &mi, &ni);
            const int m0 = mi * 256 + rank * BM;
            const int n0 = ni * PBN;
            mbar_wait(&tfull[acc], acc_phase);
            GTR(3, store_leader);
            tc_fence_after();
            if constexpr (kPairEpi) {
                // gate | up of 128 features: per 64-feature chunk, each thread takes 32
                // features of its row (half), rounds gate and up to bf16 (the stored
                // values) and forms act from them; three staging buffers are TMA-stored
                const int half = (warp - 2) >> 2;
                const int f0 = ni * 128;
#pragma unroll 1
                for (int c = 0; c < 2; ++c, ++chunk) {
                    uint32_t vg[32], vu[32];
                    tmem_ld32(tmem_base + lane_off + acc * PBN + c * 64 + half * 32, vg);
                    tmem_ld32(tmem_base + lane_off + acc * PBN + 128 + c * 64 + half * 32, vu);
                    if (store_leader) bulk_wait_read<0>();  // the previous chunk's stores have read staging
                    named_barrier(2, 256);
                    tmem_ld_wait();
#pragma unroll
                    for (int uu = 0; uu < 4; ++uu) {
                        const int u = half * 4 + uu;
                        const int sw = r * 128 + ((u ^ (r & 7)) << 4);
                        float gg[8], up[8], a[8];
#pragma unroll
                        for (int t = 0; t < 8; ++t) {
                            gg[t] = __bfloat162float(__float2bfloat16(__uint_as_float(vg[uu * 8 + t])));
                            up[t] = __bfloat162float(__float2bfloat16(__uint_as_float(vu[uu * 8 + t])));
                            a[t] = swiglu_fwd_elem(gg[t], up[t]);
                        }
                        *reinterpret_cast<uint4*>(staging + sw) = pack8(gg);
                        *reinterpret_cast<uint4*>(staging + 16384 + sw) = pack8(up);
                        *reinterpret_cast<uint4*>(staging + 32768 + sw) = pack8(a);
                    }
                    fence_async_shared();
                    named_barrier(2, 256);
                    if (store_leader) {
                        tma_store_2d(&tma_d, staging, f0 + c * 64, m0);
                        tma_store_2d(&tma_d2, staging + 16384, f0 + c * 64, m0);
                        tma_store_2d(&tma_x0, staging + 32768, f0 + c * 64, m0);
                        bulk_commit();
                    }
                }
                tc_fence_before();
                mbar_arrive_cluster(tempty_leader[acc]);
                if (++acc == 2) acc = 0, acc_phase ^= 1;
                continue;
            } else if constexpr (kFused) {
                // SwiGLU fused into the epilogue. Per 64-column chunk, one staging
                // set (2 x 16 KB) first receives the aux tiles by TMA (issued one
                // chunk ahead), each thread turns its row's aux + accumulator values
                // into the two outputs in place, and the set is TMA-stored.
                constexpr int kChunks = PBN / 64;
                constexpr uint32_t kAuxBytes = (EPI == kEpiSwiGLUBwd ? 2 : 1) * 16384;
                auto load_aux = [&](int ch, int t_m0, int col) {  // leader thread only
                    uint8_t* set = staging + (ch & 1) * 32768;
                    mbar_expect_tx(&xfull[ch & 1], kAuxBytes);
                    tma_load_2d(set, &tma_x0, &xfull[ch & 1], col, t_m0);
                    if constexpr (EPI == kEpiSwiGLUBwd) tma_load_2d(set + 16384, &tma_x1, &xfull[ch & 1], col, t_m0);
                };
                const int half = (warp - 2) >> 2;  // which 32 columns of each chunk
                if (store_leader && chunk == 0) load_aux(0, m0, n0);
#pragma unroll 1
                for (int c = 0; c < kChunks; ++c, ++chunk) {
                    const int col = n0 + c * 64;
                    uint8_t* stg0 = staging + (chunk & 1) * 32768;
                    uint8_t* stg1 = stg0 + 16384;
                    uint32_t v0[32];
                    tmem_ld32(tmem_base + lane_off + acc * PBN + c * 64 + half * 32, v0);
                    mbar_wait(&xfull[chunk & 1], (chunk >> 1) & 1);
                    tmem_ld_wait();
#pragma unroll
                    for (int uu = 0; uu < 4; ++uu) {
                        const int u = half * 4 + uu;
                        const int sw = r * 128 + ((u ^ (r & 7)) << 4);
                        float f[8], x[8], o0[8], o1[8];
#pragma unroll
                        for (int t = 0; t < 8; ++t) {
                            // the GEMM output as the unfused path stores it (bf16)
                            f[t] = __bfloat162float(__float2bfloat16(__uint_as_float(v0[uu * 8 + t])));
                        }
                        unpack8(*reinterpret_cast<const uint4*>(stg0 + sw), x);
                        if constexpr (EPI == kEpiSwiGLUFwd) {
#pragma unroll
                            for (int t = 0; t < 8; ++t) {
                                o0[t] = f[t];
                                o1[t] = p.aux_is_up ? swiglu_fwd_elem(f[t], x[t]) : swiglu_fwd_elem(x[t], f[t]);
                            }
                        } else {
                            float y[8];
                            unpack8(*reinterpret_cast<const uint4*>(stg1 + sw), y);
#pragma unroll
                            for (int t = 0; t < 8; ++t) swiglu_bwd_elem(x[t], y[t], f[t], o0[t], o1[t]);
                        }
                        *reinterpret_cast<uint4*>(stg0 + sw) = pack8(o0);
                        *reinterpret_cast<uint4*>(stg1 + sw) = pack8(o1);
                    }
                    fence_async_shared();
                    named_barrier(2, 256);
                    if (store_leader) {
                        tma_store_2d(&tma_d, stg0, col, m0);
                        tma_store_2d(&tma_d2, stg1, col, m0);
                        bulk_commit();
                        // prefetch the next chunk's aux tiles into the other set once
                        // the stores that last used it have read their data
                        int nt = tile, nc = c + 1;
                        if (nc == kChunks) nt += npairs, nc = 0;
                        if (nt < num_tiles) {
                            bulk_wait_read<1>();
                            int nmi, nni;
                            tile_coords(nt, p, &nmi, &nni);
                            load_aux(chunk + 1, nmi * 256 + rank * BM, nni * PBN + nc * 64);
                        }
                    }
                }
                tc_fence_before();
                mbar_arrive_cluster(tempty_leader[acc]);
                if (++acc == 2) acc = 0, acc_phase ^= 1;
                continue;
            }
            constexpr bool kBf16 = EPI == kEpiStoreBf16 || EPI == kEpiAddBf16;
            constexpr int CW = kBf16 ? 64 : 32;
#pragma unroll 1
            for (int c = 0; c < PBN / CW; ++c, ++chunk) {
                uint8_t* stg = staging + (chunk & 1) * 16384;
                if (store_leader) bulk_wait_read<1>();
                named_barrier(2, 128);
                if constexpr (kBf16) {
                    uint32_t v0[32], v1[32];
                    tmem_ld32(tmem_base + lane_off + acc * PBN + c * 64, v0);
                    tmem_ld32(tmem_base + lane_off + acc * PBN + c * 64 + 32, v1);
                    tmem_ld_wait();
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        float f[8];
#pragma unroll
                        for (int t = 0; t < 8; ++t) f[t] = __uint_as_float(u < 4 ? v0[u * 8 + t] : v1[(u - 4) * 8 + t]);
                        *reinterpret_cast<uint4*>(stg + r * 128 + ((u ^ (r & 7)) << 4)) = pack8(f);
                    }
                } else {
                    uint32_t v[32];
                    tmem_ld32(tmem_base + lane_off + acc * PBN + c * 32, v);
                    tmem_ld_wait();
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        *reinterpret_cast<uint4*>(stg + r * 128 + ((u ^ (r & 7)) << 4)) =
                            make_uint4(v[u * 4], v[u * 4 + 1], v[u * 4 + 2], v[u * 4 + 3]);
                }
                fence_async_shared();
                named_barrier(2, 128);
                if (store_leader) {
                    const bool ms2 = mi >= p.mt_split;  // M-concatenation: rows of the second output
                    const CUtensorMap* td = ms2 ? &tma_d2 : &tma_d;
                    const int mrow = ms2 ? m0 - p.mt_split * 256 : m0;
                    if constexpr (EPI == kEpiStoreBf16) tma_store_2d(td, stg, n0 + c * CW, mrow);
                    else tma_reduce_add_2d(td, stg, n0 + c * CW, mrow);  // f32 or bf16 add
                    bulk_commit();
                }
            }
            tc_fence_before();
            mbar_arrive_cluster(tempty_leader[acc]);
            if (++acc == 2) acc = 0, acc_phase ^= 1;
        }
        if (store_leader) bulk_wait<0>();
        GTR(4, store_leader);
    }

    tc_fence_before();
    cluster_sync();  // no CTA leaves while its peer may still signal its barriers
    GTR(5, threadIdx.x == 0);
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_pair(tmem_base, 512);
    }
}

// --------------------------------------------------------------------------- host side

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess) {
            fn = reinterpret_cast<EncodeTiledFn>(p);
        }
    });
    return fn;
}

}  // namespace

// 2D bf16 tensor map: `inner` contiguous elements per row, `outer` rows,
// `ld` elements between rows, box = box_inner x box_rows, 128-byte swizzle.
int make_tma_2d(CUtensorMap* map, const void* base, long long inner, long long outer, long long ld,
                int box_inner, int box_rows, bool f32) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return set_error(DH_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const int esz = f32 ? 4 : 2;
    if ((reinterpret_cast<uintptr_t>(base) & 15) || (ld * esz) % 16) {
        return set_error(DH_ERR_INVALID, "TMA operand must be 16-byte aligned with 16-byte row pitch");
    }
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * esz)};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_inner), static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = fn(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                          const_cast<void*>(base), dims,
                          strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_error(DH_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    return DH_OK;
}

namespace {

int make_map(CUtensorMap* map, const void* base, long long inner, long long outer, long long ld,
             int box_rows) {
    return make_tma_2d(map, base, inner, outer, ld, 64, box_rows);
}

int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

template <int BN, bool A_MN, bool B_MN, int EPI, bool D_F32>
int launch(const dh_gemm_args* g, cudaStream_t stream) {
    using Cfg = GemmCfg<BN>;
    CUtensorMap ma, mb, md;
    int rc = A_MN ? make_map(&ma, g->a, g->m, g->k, g->lda, BK) : make_map(&ma, g->a, g->k, g->m, g->lda, BM);
    if (rc) return rc;
    rc = B_MN ? make_map(&mb, g->b, g->n, g->k, g->ldb, BK) : make_map(&mb, g->b, g->k, g->n, g->ldb, BN);
    if (rc) return rc;
    if constexpr (EPI == kEpiStoreBf16) {
        rc = make_tma_2d(&md, g->d, g->n, g->m, g->ldd, 64, BM, false);
    } else if constexpr (EPI == kEpiAddF32) {
        rc = make_tma_2d(&md, g->d, g->n, g->m, g->ldd, 32, BM, true);
    } else {
        md = ma;  // unused
    }
    if (rc) return rc;
    KParams p{};
    p.kb_split = p.mt_split = 1 << 30;
    p.d = g->d;
    p.ldd = g->ldd;
    p.m = g->m;
    p.n = g->n;
    p.k = g->k;
    p.accumulate = g->accumulate;
    p.tiles_m = (g->m + BM - 1) / BM;
    p.tiles_n = (g->n + BN - 1) / BN;
    raster_for(p, BM, BN, g->k);
    const int tiles = p.tiles_m * p.tiles_n;
    int ctas = g->max_ctas > 0 ? std::min(g->max_ctas, sm_count()) : sm_count();
    ctas = std::min(ctas, tiles);
    auto kern = gemm_tcgen05_kernel<BN, A_MN, B_MN, EPI, D_F32>;
    static bool configured = false;  // per template instance
    if (!configured) {
        DH_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           Cfg::kSmemBytes));
        configured = true;
    }
    kern<<<ctas, kThreads, Cfg::kSmemBytes, stream>>>(ma, mb, md, p);
    DH_CUDA_CHECK(cudaGetLastError());
    return DH_OK;
}

// Raster order for the tile loop: estimate the DRAM bytes of each order and
// group size (the grouped operand's panels read once, the other operand's once
// per group; a group's panels must fit an L2 budget that leaves room for the
// streamed operand and the output) and keep the cheapest. The all-of-M group
// (b_resident 0, group tiles_m) is the plain m-fastest order.
void raster_for(KParams& p, int bm, int bn, int k) {
    constexpr double kBudget = 40.0 * (1 << 20);
    const double pa = static_cast<double>(bm) * k * 2, pb = static_cast<double>(bn) * k * 2;  // panel bytes
    const double A = pa * p.tiles_m, B = pb * p.tiles_n;
    double best = -1.0;
    for (int br = 0; br < 2; ++br) {
        const int fast = br ? p.tiles_n : p.tiles_m;
        const double panel = br ? pb : pa;
        for (int gsz = fast; gsz >= 1; --gsz) {
            if (gsz * panel > kBudget && gsz > 1) continue;
            const int groups = (fast + gsz - 1) / gsz;
            const double bytes = br ? B + A * groups : A + B * groups;
            if (best < 0 || bytes < best * 0.999) {
                best = bytes;
                p.b_resident = br;
                p.group = gsz;
            }
            break;  // the largest group within the budget is the cheapest for this order
        }
    }
    // DH_GEMM_RASTER=m: the plain m-fastest order (A/B comparisons)
    static const bool plain = [] {
        const char* e = std::getenv("DH_GEMM_RASTER");
        return e && e[0] == 'm';
    }();
    if (plain) {
        p.b_resident = 0;
        p.group = p.tiles_m;
    }
}

template <int PBN, bool A_MN, bool B_MN, int EPI>
int launch_pair(const dh_gemm_args* g, cudaStream_t stream, int ctas) {
    constexpr bool kFused = EPI == kEpiSwiGLUFwd || EPI == kEpiSwiGLUBwd;
    constexpr bool kPairEpi = EPI == kEpiSwiGLUPair;
    using C = PairCfg<PBN, kFused || kPairEpi>;
    CUtensorMap ma, mb, md, md2;
    int rc = A_MN ? make_map(&ma, g->a, g->m, g->k, g->lda, BK) : make_map(&ma, g->a, g->k, g->m, g->lda, BM);
    if (rc) return rc;
    rc = B_MN ? make_map(&mb, g->b, g->n, g->k, g->ldb, BK) : make_map(&mb, g->b, g->k, g->n, g->ldb, C::kHalfB);
    if (rc) return rc;
    rc = EPI == kEpiAddF32 ? make_tma_2d(&md, g->d, g->n, g->m, g->ldd, 32, BM, true)
                           : make_tma_2d(&md, g->d, g->n, g->m, g->ldd, 64, BM, false);
    if (rc) return rc;
    CUtensorMap mx0, mx1;
    const bool kcat = g->k2 > 0, mcat = g->m2 > 0;
    if (kPairEpi) {  // B halves: Wg (b) and Wu (b2) rows; outputs gate (d), up (d2), act (d_m2)
        rc = make_map(&mb, g->b, g->k, g->n, g->ldb, C::kHalfB);
        if (!rc) rc = make_map(&mx1, g->b2, g->k, g->n, g->ldb2, C::kHalfB);
        if (!rc) rc = make_tma_2d(&md2, g->d2, g->n, g->m, g->ldd, 64, BM, false);
        if (!rc) rc = make_tma_2d(&mx0, g->d_m2, g->n, g->m, g->ldd, 64, BM, false);
        if (rc) return rc;
    } else if (kcat) {  // second K segment: A2 [m, k2], B2 [n, k2] with A's / B's majors
        rc = A_MN ? make_map(&mx0, g->a2, g->m, g->k2, g->lda2, BK) : make_map(&mx0, g->a2, g->k2, g->m, g->lda2, BM);
        if (!rc) rc = B_MN ? make_map(&mx1, g->b2, g->n, g->k2, g->ldb2, BK)
                           : make_map(&mx1, g->b2, g->k2, g->n, g->ldb2, C::kHalfB);
        if (rc) return rc;
        md2 = md;
    } else if (mcat) {  // second M segment: A2 [m2, k] -> D2 [m2, n]
        rc = A_MN ? make_map(&mx0, g->a2, g->m2, g->k, g->lda2, BK) : make_map(&mx0, g->a2, g->k, g->m2, g->lda2, BM);
        if (!rc) rc = EPI == kEpiAddF32 ? make_tma_2d(&md2, g->d_m2, g->n, g->m2, g->ldd_m2, 32, BM, true)
                                        : make_tma_2d(&md2, g->d_m2, g->n, g->m2, g->ldd_m2, 64, BM, false);
        if (rc) return rc;
        mx1 = mb;
    } else if (kFused) {
        rc = make_tma_2d(&md2, g->d2, g->n, g->m, g->ldd, 64, BM, false);
        if (!rc) rc = make_tma_2d(&mx0, g->aux0, g->n, g->m, g->ld_aux, 64, BM, false);
        if (!rc) rc = make_tma_2d(&mx1, g->aux1 ? g->aux1 : g->aux0, g->n, g->m, g->ld_aux, 64, BM, false);
        if (rc) return rc;
    } else {
        md2 = mx0 = mx1 = md;  // unused
    }
    KParams p{};
    p.aux0 = static_cast<const __nv_bfloat16*>(g->aux0);
    p.aux1 = static_cast<const __nv_bfloat16*>(g->aux1);
    p.ld_aux = g->ld_aux;
    p.aux_is_up = g->epilogue == DH_EPI_SWIGLU_FWD_UP;
    p.d = g->d;
    p.ldd = g->ldd;
    p.m = g->m;
    p.n = g->n;
    p.k = g->k;
    p.accumulate = g->accumulate;
    p.tiles_m = (g->m + 255) / 256;
    p.tiles_n = kPairEpi ? (g->n + 127) / 128 : (g->n + PBN - 1) / PBN;
    p.kb_split = p.mt_split = 1 << 30;
    if (kcat) {
        p.kb_split = g->k / BK;
        p.k = g->k + g->k2;
    }
    if (mcat) {
        p.mt_split = g->m / 256;
        p.tiles_m = g->m / 256 + (g->m2 + 255) / 256;
    }
    raster_for(p, 256, PBN, p.k);
    const int tiles = p.tiles_m * p.tiles_n;
    const int grid = 2 * std::min(ctas / 2, tiles);
    auto kern = gemm_pair_kernel<PBN, A_MN, B_MN, EPI>;
    static bool configured = false;
    if (!configured) {
        DH_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
        configured = true;
    }
    kern<<<grid, pair_threads<EPI>(), C::kSmem, stream>>>(ma, mb, md, md2, mx0, mx1, p);
    DH_CUDA_CHECK(cudaGetLastError());
    return DH_OK;
}

template <int PBN, int EPI>
int dispatch_pair(const dh_gemm_args* g, cudaStream_t s, int ctas) {
    const int key = (g->a_mn ? 2 : 0) | (g->b_mn ? 1 : 0);
    switch (key) {
        case 0: return launch_pair<PBN, false, false, EPI>(g, s, ctas);
        case 1: return launch_pair<PBN, false, true, EPI>(g, s, ctas);
        case 2: return launch_pair<PBN, true, false, EPI>(g, s, ctas);
        default: return launch_pair<PBN, true, true, EPI>(g, s, ctas);
    }
}

template <int PBN>
int dispatch_pair_epi(const dh_gemm_args* g, cudaStream_t s, int ctas) {
    if constexpr (PBN == 256)
        if (g->epilogue == DH_EPI_SWIGLU_PAIR) return launch_pair<256, false, false, kEpiSwiGLUPair>(g, s, ctas);
    if (g->epilogue == DH_EPI_SWIGLU_BWD) return dispatch_pair<PBN, kEpiSwiGLUBwd>(g, s, ctas);
    if (g->epilogue) return dispatch_pair<PBN, kEpiSwiGLUFwd>(g, s, ctas);
    if (g->d_fp32) return dispatch_pair<PBN, kEpiAddF32>(g, s, ctas);
    // bf16 accumulate = TMA reduce-add: D = bf16(D + bf16(acc))
    return g->accumulate ? dispatch_pair<PBN, kEpiAddBf16>(g, s, ctas)
                         : dispatch_pair<PBN, kEpiStoreBf16>(g, s, ctas);
}

template <int BN, int EPI, bool D_F32>
int dispatch_major(const dh_gemm_args* g, cudaStream_t s) {
    const int key = (g->a_mn ? 2 : 0) | (g->b_mn ? 1 : 0);
    switch (key) {
        case 0: return launch<BN, false, false, EPI, D_F32>(g, s);
        case 1: return launch<BN, false, true, EPI, D_F32>(g, s);
        case 2: return launch<BN, true, false, EPI, D_F32>(g, s);
        default: return launch<BN, true, true, EPI, D_F32>(g, s);
    }
}

template <int BN>
int dispatch_epi(const dh_gemm_args* g, cudaStream_t s) {
    const bool aligned = (reinterpret_cast<uintptr_t>(g->d) & 15) == 0 &&
                         (g->ldd * (g->d_fp32 ? 4 : 2)) % 16 == 0;
    if (aligned && !g->d_fp32 && !g->accumulate) return dispatch_major<BN, kEpiStoreBf16, false>(g, s);
    if (aligned && g->d_fp32 && g->accumulate) return dispatch_major<BN, kEpiAddF32, true>(g, s);
    if (g->d_fp32) return dispatch_major<BN, kEpiDirect, true>(g, s);
    return dispatch_major<BN, kEpiDirect, false>(g, s);
}

}  // namespace

// Tile choice: per candidate tile, the fraction of issued tile area that is
// useful given the persistent grid's wave quantisation, times the tile's
// measured per-SM efficiency relative to the 256 x 256 CTA pair (B200, see
// profiles/: narrower tiles re-read more operand bytes per FLOP, one-CTA tiles
// stage both operands on one SM). Ties go to the earlier (wider) candidate.
struct TileCand {
    int pbn;      // > 0: CTA pair 256 x pbn; < 0: one CTA 128 x -pbn
    double eff;   // per-SM efficiency of the tile shape
};
constexpr TileCand kTiles[] = {{256, 1.0}, {192, 0.95}, {128, 0.85},
                               {-256, 0.92}, {-192, 0.80}, {-128, 0.70}};

double tile_score(const TileCand& t, long long m, long long n, int ctas) {
    const bool pair = t.pbn > 0;
    const long long bm = pair ? 256 : 128, bn = pair ? t.pbn : -t.pbn;
    const long long units = pair ? ctas / 2 : ctas;
    if (units < 1) return -1.0;
    const long long tiles = ((m + bm - 1) / bm) * ((n + bn - 1) / bn);
    const long long waves = (tiles + units - 1) / units;
    return static_cast<double>(m) * n / (static_cast<double>(waves) * units * bm * bn) * t.eff;
}

int gemm_pick_tile(int m, int n, int ctas, bool pair_ok, bool b_mn, bool pair_only = false) {
    int best = pair_only ? 256 : -256;
    double best_score = -1.0;
    for (const TileCand& t : kTiles) {
        if (t.pbn > 0 && !pair_ok) continue;
        if (t.pbn < 0 && pair_only) continue;
        if (t.pbn == 192 && b_mn) continue;  // 96-row MN-major B halves are not whole swizzle atoms
        const double sc = tile_score(t, m, n, ctas);
        if (sc > best_score + 1e-3) best_score = sc, best = t.pbn;
    }
    return best;
}

#define GEMM_TRY(expr)                   \
    do {                                  \
        const int rc_ = (expr);           \
        if (rc_ != DH_OK) return rc_;     \
    } while (0)

int gemm(const dh_gemm_args* g, cudaStream_t s);

// SwiGLU epilogues: fused into the CTA-pair kernel when the operands allow it,
// else the plain GEMM followed by the standalone SwiGLU kernel (same math).
int gemm_swiglu(const dh_gemm_args* g, cudaStream_t s) {
    if (g->epilogue == DH_EPI_SWIGLU_PAIR) {
        if (g->accumulate || g->d_fp32 || !g->d2 || !g->b2 || !g->d_m2 || g->a_mn || g->b_mn)
            return set_error(DH_ERR_INVALID, "gemm: SwiGLU pair epilogue needs K-major A / B, B2, bf16 d, d2, d_m2");
        const int ctas = g->max_ctas > 0 ? std::min(g->max_ctas, sm_count()) : sm_count();
        auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
        if (ctas >= 2 && g->n % 128 == 0 && g->ldd % 8 == 0 && al16(g->d) && al16(g->d2) && al16(g->d_m2))
            return dispatch_pair_epi<256>(g, s, ctas);
        // unfused: the two GEMMs, then the standalone SwiGLU
        dh_gemm_args a = *g;
        a.epilogue = DH_EPI_NONE;
        a.b2 = nullptr;
        GEMM_TRY(gemm(&a, s));
        a.b = g->b2;
        a.ldb = g->ldb2;
        a.d = g->d2;
        GEMM_TRY(gemm(&a, s));
        if (g->ldd != g->n) return set_error(DH_ERR_INVALID, "gemm: unfused SwiGLU pair needs dense [m, n] outputs");
        return dh_swiglu_fwd(g->d, g->d2, g->d_m2, static_cast<long long>(g->m) * g->n, s);
    }
    if (g->accumulate || g->d_fp32 || !g->d2 || !g->aux0 || (g->epilogue == DH_EPI_SWIGLU_BWD && !g->aux1))
        return set_error(DH_ERR_INVALID, "gemm: SwiGLU epilogue needs bf16 d, d2 and aux operands");
    const int ctas = g->max_ctas > 0 ? std::min(g->max_ctas, sm_count()) : sm_count();
    auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
    const bool fusable = ctas >= 2 && g->n % 64 == 0 && g->ldd % 8 == 0 && g->ld_aux % 8 == 0 && al16(g->d) &&
                         al16(g->d2) && al16(g->aux0) && (!g->aux1 || al16(g->aux1)) && g->ldd == g->ld_aux;
    if (!fusable) {
        dh_gemm_args plain = *g;
        plain.epilogue = DH_EPI_NONE;
        if (g->ldd != g->n || g->ld_aux != g->n)
            return set_error(DH_ERR_INVALID, "gemm: unfused SwiGLU fallback needs dense [m, n] operands");
        const long long count = static_cast<long long>(g->m) * g->n;
        if (g->epilogue == DH_EPI_SWIGLU_BWD) {
            plain.d = g->d2;  // d_act lands in d_up, then swiglu_bwd runs in place on it
            GEMM_TRY(gemm(&plain, s));
            return dh_swiglu_bwd(g->aux0, g->aux1, g->d2, g->d, g->d2, count, s);
        }
        GEMM_TRY(gemm(&plain, s));
        return g->epilogue == DH_EPI_SWIGLU_FWD_UP ? dh_swiglu_fwd(g->d, g->aux0, g->d2, count, s)
                                                   : dh_swiglu_fwd(g->aux0, g->d, g->d2, count, s);
    }
    int pick = g->tile_n < 0 ? -g->tile_n : g->tile_n == 512 ? 256 : 0;
    if (!pick) pick = gemm_pick_tile(g->m, g->n, ctas, true, g->b_mn, true);
    if (pick == 192 && !g->b_mn) return dispatch_pair_epi<192>(g, s, ctas);
    if (pick == 128) return dispatch_pair_epi<128>(g, s, ctas);
    return dispatch_pair_epi<256>(g, s, ctas);
}

int gemm(const dh_gemm_args* g, cudaStream_t s) {
    if (g->m <= 0 || g->n <= 0 || g->k <= 0) return set_error(DH_ERR_INVALID, "gemm: empty shape");
    if (g->k2 > 0 || g->m2 > 0) {
        if (g->epilogue || (g->k2 > 0 && g->m2 > 0) || !g->a2 || (g->k2 > 0 && !g->b2) || (g->m2 > 0 && !g->d_m2))
            return set_error(DH_ERR_INVALID, "gemm: one of k2 / m2 with a2 and b2 / d_m2, no SwiGLU epilogue");
        const int ctas = g->max_ctas > 0 ? std::min(g->max_ctas, sm_count()) : sm_count();
        const bool aligned = (reinterpret_cast<uintptr_t>(g->d) & 15) == 0 && (g->ldd * (g->d_fp32 ? 4 : 2)) % 16 == 0 &&
                             (!g->d_m2 || ((reinterpret_cast<uintptr_t>(g->d_m2) & 15) == 0 &&
                                           (g->ldd_m2 * (g->d_fp32 ? 4 : 2)) % 16 == 0));
        const bool one_launch = aligned && (g->accumulate || !g->d_fp32) && ctas >= 2 && g->tile_n == 0 &&
                                (g->k2 == 0 || g->k % BK == 0) && (g->m2 == 0 || g->m % 256 == 0);
        if (one_launch) return dispatch_pair_epi<256>(g, s, ctas);
        // two launches: the first segment, then the second (accumulated / into d_m2)
        dh_gemm_args a = *g, b = *g;
        a.a2 = b.a2 = nullptr;
        a.k2 = b.k2 = a.m2 = b.m2 = 0;
        b.a = g->a2;
        b.lda = g->lda2;
        if (g->k2 > 0) {
            b.b = g->b2;
            b.ldb = g->ldb2;
            b.k = g->k2;
            b.accumulate = 1;
        } else {
            b.m = g->m2;
            b.d = g->d_m2;
            b.ldd = g->ldd_m2;
        }
        GEMM_TRY(gemm(&a, s));
        return gemm(&b, s);
    }
    if (g->epilogue) return gemm_swiglu(g, s);
    const int ctas = g->max_ctas > 0 ? std::min(g->max_ctas, sm_count()) : sm_count();
    const bool aligned = (reinterpret_cast<uintptr_t>(g->d) & 15) == 0 &&
                         (g->ldd * (g->d_fp32 ? 4 : 2)) % 16 == 0;
    const bool pair_ok = aligned && (g->accumulate || !g->d_fp32) && ctas >= 2;
    // tile_n: 0 auto; 128/192/256 one CTA 128 x tile_n; 512 = CTA pair 256 x 256;
    // -128/-192/-256 = CTA pair 256 x |tile_n|
    int pick;
    if (g->tile_n == 0) pick = gemm_pick_tile(g->m, g->n, ctas, pair_ok, g->b_mn);
    else if (g->tile_n == 512) pick = 256;
    else if (g->tile_n < 0) pick = -g->tile_n;
    else pick = -g->tile_n;
    if (pick > 0 && !pair_ok) pick = -256;  // CTA pairs need an aligned bf16 or accumulated output
    if (pick > 0) {
        if (pick == 256) return dispatch_pair_epi<256>(g, s, ctas);
        if (pick == 192) {
            if (g->b_mn) return set_error(DH_ERR_INVALID, "gemm: pair tile 192 needs a K-major B");
            return dispatch_pair_epi<192>(g, s, ctas);
        }
        if (pick == 128) return dispatch_pair_epi<128>(g, s, ctas);
        return set_error(DH_ERR_INVALID, "gemm: pair tile_n must be 128, 192 or 256");
    }
    const int bn = -pick;
    if (bn == 256) return dispatch_epi<256>(g, s);
    if (bn == 192) return dispatch_epi<192>(g, s);
    if (bn == 128) return dispatch_epi<128>(g, s);
    return set_error(DH_ERR_INVALID, "gemm: tile_n must be 0, 128, 192, 256, 512 or -128/-192/-256");
}

}  // namespace dh

extern "C" int dh_gemm(const dh_gemm_args* args, void* stream) {
    if (!args) return dh::set_error(DH_ERR_INVALID, "dh_gemm: null args");
    return dh::gemm(args, static_cast<cudaStream_t>(stream));
}
