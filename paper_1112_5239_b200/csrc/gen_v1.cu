// gen_v1.cu -- V1: Alg. 4 "improved" kernel on sm_100a.
//
// Per stream (= paper thread): one 32-bit xor128 (Q5), the
// chaotic-iteration state x and the shared cell tp (the previous round's t,
// Q7/Q8).  Per round:  t = xor128() ^ tp[o1] ^ tp[o2];  tp = t;  x ^= t;
// emit x.  A combination group (C streams) never
// straddles a warp, so the exchange of shared cells is a register shuffle:
// no shared memory, no barrier, and the paper's unsynchronised shmem
// read/write becomes the two-phase semantics of reading Q7 by construction.
//
// Two kernels:
//  * v1_general_kernel -- any C | 32, any arrays: one lane per stream,
//    2 SHFL per number.
//  * v1_fast_kernel -- the default C = 32 arrays comb1 = l+1, comb2 = l+17
//    (Q6).  Because o2 = o1 + 16, lane j of a 16-lane half-warp owns streams
//    j and j+16 of a group; both need tp[j+1] ^ tp[j+17] = u[j+1] with
//    u[j] = tp[j] ^ tp[j+16] local to lane j, and u after a round is
//    g[j] ^ g[j+16] (the neighbour term cancels).  One SHFL per 2 numbers,
//    3 LOP3 per 2 numbers on top of the xor128 steps.  Stores either direct
//    (128-bit STG of 4-round buffers) or through a per-warp shared-memory
//    tile written to HBM by a 2-D TMA bulk tensor store.
#include <type_traits>

#include "device.cuh"
#include "kernels.h"
#include "sinks.cuh"

namespace ciprng {

// ===================================================================== general
template <class Sink>
__global__ void __launch_bounds__(256) v1_general_kernel(GenArgs a) {
    Sink sink(a);
    pdl_launch_dependents();
    pdl_wait();  // previous grid on the stream complete + visible
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t C = a.C;
    const uint32_t off = lane % C, gbase = lane - off;
    const uint32_t src1 = gbase + a.comb.t[0][off];
    const uint32_t src2 = gbase + a.comb.t[1][off];
    const uint64_t n_tiles = (a.s_count + 31) / 32;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    const StateIO sio(a);

    for (uint64_t tile = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); tile < n_tiles;
         tile += warps) {
        const uint64_t row = tile * 32 + lane;
        const bool valid = row < a.s_count;
        const uint64_t s = a.s_begin + row;
        uint32_t g0 = 0, g1 = 0, g2 = 0, g3 = 0, x = 0, tp = 0;
        if (valid) {
            g0 = sio.ld(0, s); g1 = sio.ld(1, s); g2 = sio.ld(2, s); g3 = sio.ld(3, s);
            x = sio.ld(4, s); tp = sio.ld(5, s);
        }
        sink.begin_row(0, row);
        uint64_t i = 0;
        for (; i + 4 <= a.n; i += 4) {
            uint32_t t, o0, o1, o2, o3;
            g0 = xor128_f(g0, g3);
            t = g0 ^ __shfl_sync(kFull, tp, src1) ^ __shfl_sync(kFull, tp, src2);
            tp = t; x ^= t; o0 = x;
            g1 = xor128_f(g1, g0);
            t = g1 ^ __shfl_sync(kFull, tp, src1) ^ __shfl_sync(kFull, tp, src2);
            tp = t; x ^= t; o1 = x;
            g2 = xor128_f(g2, g1);
            t = g2 ^ __shfl_sync(kFull, tp, src1) ^ __shfl_sync(kFull, tp, src2);
            tp = t; x ^= t; o2 = x;
            g3 = xor128_f(g3, g2);
            t = g3 ^ __shfl_sync(kFull, tp, src1) ^ __shfl_sync(kFull, tp, src2);
            tp = t; x ^= t; o3 = x;
            sink.put4(0, i, o0, o1, o2, o3, valid);
        }
        for (; i < a.n; ++i) {  // ragged tail: plain step with register moves
            uint32_t g = xor128_f(g0, g3);
            g0 = g1; g1 = g2; g2 = g3; g3 = g;
            uint32_t t = g ^ __shfl_sync(kFull, tp, src1) ^ __shfl_sync(kFull, tp, src2);
            tp = t; x ^= t;
            sink.put1(0, i, x, valid);
        }
        sink.end_rows(valid ? 1u : 0u);
        if (valid) {
            sio.st(0, s, g0); sio.st(1, s, g1); sio.st(2, s, g2); sio.st(3, s, g3);
            sio.st(4, s, x); sio.st(5, s, tp);
        }
    }
    sink.finish(a);
}

// ======================================================================== fast
// Tile = 64 streams (2 groups) per warp; lane L: half h = L >> 4 (group),
// j = L & 15, owns rows rA = 32h + j and rB = rA + 16 of the tile.
constexpr int kFastTileRows = 64;

// xor128 step of the fast kernel: the fused consumer takes the all-ALU-shift
// form (device.cuh xor128_f_alu), the store and battery kernels the balanced one
template <class Sink>
__device__ __forceinline__ uint32_t v1_x128(uint32_t xk, uint32_t wk3) {
    if constexpr (std::is_same<Sink, StatsSink>::value || std::is_same<Sink, StatsSinkCta>::value)
        return xor128_f_alu(xk, wk3);
    else return xor128_f(xk, wk3);
}
// the lane's second stream (experiment CIPRNG_CTA_X128B_HI: the CTA-histogram
// consumer's B stream in the balanced form, w >> 19 on the heavy pipe)
template <class Sink>
__device__ __forceinline__ uint32_t v1_x128b(uint32_t xk, uint32_t wk3) {
#if defined(CIPRNG_CTA_X128B_HI)
    if constexpr (std::is_same<Sink, StatsSinkCta>::value) return xor128_f(xk, wk3);
#endif
    return v1_x128<Sink>(xk, wk3);
}


// kCols == 0: direct stores through the Sink (StoreSink: 128-bit STG per
// 4 rounds per stream; StatsSink: fused consumer).  kCols in {8, 16, 32}:
// TMA tile store of kCols rounds x 64 streams per box, double-buffered.
// kStg: SURVEY s7 store path (b) -- the same swizzled shared-memory box as
// the TMA path, written back by the warp itself with coalesced 128-bit STG
// (8 lanes per 128-byte row piece, 4 rows per instruction) instead of a TMA
// bulk tensor store; kept for the three-way store-path comparison.
// The staged-STG instantiation takes the relaxed budget too: at ptxas'
// default 64 registers it spilled 8 bytes (80 registers, no spill).
template <class Sink, int kCols, bool kStg>
constexpr int v1_fast_min_blocks() {
    return (kLbForceMin1 || (std::is_same<Sink, StoreSink>::value && kCols > 0)) ? 1 : 0;
}

// experiment: launch bounds of the consumer instantiation (threads, min CTAs).
// Measured (profiles/experiments/s45_v1_consumer_bounds.jsonl): the default
// (256, 0) = 72 registers 1.69e12; (128, 8) = 64 registers, 8 CTAs/SM -5 %;
// (128, 0) = 80 registers -1.2 %.
#ifndef CIPRNG_EXP_V1C_THREADS
#define CIPRNG_EXP_V1C_THREADS 256
#endif
#ifndef CIPRNG_EXP_V1C_MINB
#define CIPRNG_EXP_V1C_MINB 0
#endif
template <class Sink>
constexpr int v1_fast_max_threads() {
    return Sink::kCtaHist ? 32 * cta_hist_warps<Sink>()
           : (std::is_same<Sink, StatsSink>::value || std::is_same<Sink, StatsSinkLane>::value) ? CIPRNG_EXP_V1C_THREADS
                                                                                                : 256;
}
template <class Sink, int kCols, bool kStg>
constexpr int v1_fast_min_blocks_x() {
    return Sink::kCtaHist                                                ? cta_hist_min_blocks<Sink>()
           : std::is_same<Sink, StatsSink>::value && CIPRNG_EXP_V1C_MINB > 0 ? CIPRNG_EXP_V1C_MINB
                                                                            : v1_fast_min_blocks<Sink, kCols, kStg>();
}

template <class Sink, int kCols, int kBufs = 2, bool kStg = false>
__global__ void __launch_bounds__((v1_fast_max_threads<Sink>()), (v1_fast_min_blocks_x<Sink, kCols, kStg>())) v1_fast_kernel(GenArgs a, const __grid_constant__ CUtensorMap tmap) {
    constexpr bool kTma = kCols > 0;
    constexpr uint32_t kTileBytes = kFastTileRows * (kCols > 0 ? kCols : 4) * 4;
    Sink sink(a);
    pdl_launch_dependents();
    pdl_wait();  // previous grid on the stream complete + visible
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t h = lane >> 4, j = lane & 15u;
    const uint32_t src = (j + 1u) & 15u;  // width-16 shuffle source
    const uint64_t n_tiles = (a.s_count + kFastTileRows - 1) / kFastTileRows;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    uint32_t *P = a.state;
    const uint64_t L = a.n_local;
    const uint32_t rA_t = 32u * h + j, rB_t = rA_t + 16u;  // rows within the tile

    uint32_t wsmem = 0;
    if constexpr (kTma) {
        extern __shared__ __align__(1024) uint8_t smem_dyn[];
        // swizzled TMA boxes need 1 KiB-aligned shared addresses
        const uint32_t base = (smem_u32(smem_dyn) + 1023u) & ~1023u;
        wsmem = base + (threadIdx.x >> 5) * (kBufs * kTileBytes);
    }
    uint32_t tma_issued = 0;  // boxes issued by this warp

    // State of the warp's NEXT tile is loaded into registers while the current
    // one computes (ncu r1e: the first use of freshly loaded state was 18 % of
    // all warp stall samples when every tile waited for its own loads).
    // Experiment CIPRNG_EXP_V1C_NOPF: consumers load each tile's state when it
    // starts (their tiles run n >= 2^10 rounds) to save the look-ahead's 12
    // registers -- per-warp-histogram consumer 77 -> 72 registers, 6 -> 7
    // CTAs/SM, but 1.849 -> 1.801e12 numbers/s (profiles/experiments/s56); off.
#if defined(CIPRNG_EXP_V1C_NOPF)
    constexpr bool kLookAhead = !Sink::kStats;
#else
    constexpr bool kLookAhead = true;
#endif
    uint64_t tile = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    uint32_t pa[6] = {0, 0, 0, 0, 0, 0}, pb[6] = {0, 0, 0, 0, 0, 0};
    const StateIO sio(a);
    auto prefetch = [&](uint64_t t) {
        if (t < n_tiles && t * kFastTileRows + 32u * h < a.s_count) {
            const uint64_t sA = a.s_begin + t * kFastTileRows + rA_t, sB = sA + 16u;
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                pa[k] = sio.ld(k, sA);
                pb[k] = sio.ld(k, sB);
            }
        } else if constexpr (std::is_same<Sink, StatsSinkCta>::value) {
            // an invalid half-warp runs on an all-zero state (StatsSinkCta::bin)
#pragma unroll
            for (int k = 0; k < 6; ++k) pa[k] = pb[k] = 0u;
        }
    };
    if constexpr (kLookAhead) prefetch(tile);
    for (; tile < n_tiles; tile += warps) {
        if constexpr (!kLookAhead) prefetch(tile);
        const uint64_t row0 = tile * kFastTileRows;
        const bool valid = row0 + 32u * h < a.s_count;  // s_count % 32 == 0
        const uint64_t rA = row0 + rA_t, rB = row0 + rB_t;
        const uint64_t sA = a.s_begin + rA, sB = a.s_begin + rB;
        // warm L2 with the state of the tile a warp of the next wave will take
        // (one wave = pf_ahead resident warps), so its first loads hit L2
        if (a.pf_ahead && lane == 0) {
            const uint64_t t2 = tile + a.pf_ahead;
            if (t2 * kFastTileRows + kFastTileRows <= a.s_count)
#pragma unroll
                for (int k = 0; k < 6; ++k)
                    bulk_prefetch_l2(P + k * L + a.s_begin + t2 * kFastTileRows, kFastTileRows * 4);
        }
        uint32_t a0 = pa[0], a1 = pa[1], a2 = pa[2], a3 = pa[3], xA = pa[4], tpA = pa[5];
        uint32_t b0 = pb[0], b1 = pb[1], b2 = pb[2], b3 = pb[3], xB = pb[4], tpB = pb[5];
        if constexpr (kLookAhead) prefetch(tile + warps);
        sink.begin_row(0, rA);
        sink.begin_row(1, rB);
        uint32_t u = tpA ^ tpB;  // u[j] = tp[j] ^ tp[j+16]
        uint32_t nb = 0;

#define CIPRNG_V1_ROUND(GA, GA3, GB, GB3, OA, OB)        \
    GA = v1_x128<Sink>(GA, GA3);                              \
    GB = v1_x128b<Sink>(GB, GB3);                             \
    nb = __shfl_sync(kFull, u, src, 16);                 \
    xA ^= GA ^ nb;                                       \
    xB ^= GB ^ nb;                                       \
    u = GA ^ GB;                                         \
    OA = xA;                                             \
    OB = xB;
#define CIPRNG_V1_BLOCK4(Q)                                                   \
    {                                                                         \
        uint32_t oA0, oA1, oA2, oA3, oB0, oB1, oB2, oB3;                      \
        CIPRNG_V1_ROUND(a0, a3, b0, b3, oA0, oB0)                             \
        CIPRNG_V1_ROUND(a1, a0, b1, b0, oA1, oB1)                             \
        CIPRNG_V1_ROUND(a2, a1, b2, b1, oA2, oB2)                             \
        CIPRNG_V1_ROUND(a3, a2, b3, b2, oA3, oB3)                             \
        st_shared_v4(buf + swz<kCols>(rA_t, (Q)), oA0, oA1, oA2, oA3);        \
        st_shared_v4(buf + swz<kCols>(rB_t, (Q)), oB0, oB1, oB2, oB3);        \
    }

        uint64_t i = 0;
        if constexpr (kTma) {
            // boxes of kCols rounds over the first nb4 rounds (TMA: n % 4 == 0
            // guaranteed by the host; staged STG: the last n % 4 rounds follow
            // as a scalar tail)
            const uint64_t nb4 = kStg ? (a.n & ~3ull) : a.n;
            for (uint64_t i0 = 0; i0 < nb4; i0 += kCols) {
                const uint32_t buf = wsmem + (tma_issued % kBufs) * kTileBytes;
                if (!kStg && tma_issued >= kBufs) {
                    if (lane == 0) bulk_wait_read<kBufs - 1>();
                    __syncwarp();
                }
                if (i0 + kCols <= nb4) {  // full box: no per-block bound checks
#pragma unroll
                    for (uint32_t q = 0; q < kCols / 4; ++q) CIPRNG_V1_BLOCK4(q)
                } else {
                    for (uint32_t q = 0; i0 + 4 * q < nb4; ++q) CIPRNG_V1_BLOCK4(q)
                }
                if constexpr (kStg) {
                    __syncwarp();
                    staged_writeback<kCols>(buf, a.out, row0, a.s_count, a.n, i0,
                                            (i0 + kCols <= nb4) ? kCols : nb4 - i0, a.vec != 0,
                                            a.evict_first != 0, lane);
                    __syncwarp();
                } else {
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        if (a.evict_first) tma_store_2d_hint(&tmap, buf, (int)i0, (int)row0, l2_evict_first_policy());
                        else tma_store_2d(&tmap, buf, (int)i0, (int)row0);
                        bulk_commit();
                    }
                }
                ++tma_issued;
            }
            i = nb4;
            if constexpr (kStg) {
                for (; i < a.n; ++i) {  // the last n % 4 rounds: scalar stores
                    uint32_t gA = v1_x128<Sink>(a0, a3), gB = v1_x128b<Sink>(b0, b3);
                    a0 = a1; a1 = a2; a2 = a3; a3 = gA;
                    b0 = b1; b1 = b2; b2 = b3; b3 = gB;
                    nb = __shfl_sync(kFull, u, src, 16);
                    xA ^= gA ^ nb;
                    xB ^= gB ^ nb;
                    u = gA ^ gB;
                    sink.put1(0, i, xA, valid);
                    sink.put1(1, i, xB, valid);
                }
            }
        } else {
#define CIPRNG_V1_DIRECT4(I)                              \
    {                                                     \
        uint32_t oA0, oA1, oA2, oA3, oB0, oB1, oB2, oB3;  \
        CIPRNG_V1_ROUND(a0, a3, b0, b3, oA0, oB0)         \
        CIPRNG_V1_ROUND(a1, a0, b1, b0, oA1, oB1)         \
        CIPRNG_V1_ROUND(a2, a1, b2, b1, oA2, oB2)         \
        CIPRNG_V1_ROUND(a3, a2, b3, b2, oA3, oB3)         \
        sink.put4(0, (I), oA0, oA1, oA2, oA3, valid);     \
        sink.put4(1, (I), oB0, oB1, oB2, oB3, valid);     \
    }
            // unroll 4 (8 rounds measured -1.5 %: 76 regs, 6 CTAs/SM, s20)
            if constexpr (Sink::kStats) {
                // consumers: n < 2^24 (host-checked), a 32-bit trip counter
                // and index (the u64 loop against a.n cost 8 instructions per 4 rounds)
                const uint32_t n4 = (uint32_t)a.n & ~3u;
#if defined(CIPRNG_EXP_V1C_UNROLL)  // experiment: unroll the 4-round body further
                constexpr int kUnroll = CIPRNG_EXP_V1C_UNROLL;
#pragma unroll kUnroll
#endif
                for (uint32_t i32 = 0; i32 != n4; i32 += 4) CIPRNG_V1_DIRECT4(i32)
                i = n4;
            } else {
                for (; i + 4 <= a.n; i += 4) CIPRNG_V1_DIRECT4(i)
            }
#undef CIPRNG_V1_DIRECT4
            for (; i < a.n; ++i) {  // ragged tail
                uint32_t gA = v1_x128<Sink>(a0, a3), gB = v1_x128b<Sink>(b0, b3);
                a0 = a1; a1 = a2; a2 = a3; a3 = gA;
                b0 = b1; b1 = b2; b2 = b3; b3 = gB;
                nb = __shfl_sync(kFull, u, src, 16);
                xA ^= gA ^ nb;
                xB ^= gB ^ nb;
                u = gA ^ gB;
                sink.put1(0, i, xA, valid);
                sink.put1(1, i, xB, valid);
            }
        }
#undef CIPRNG_V1_BLOCK4
#undef CIPRNG_V1_ROUND
        sink.end_rows(valid ? 2u : 0u);
        if (valid) {
            if (a.n > 0) {
                // last round's t = g ^ nb; g is the newest ring entry, a3 / b3
                tpA = a3 ^ nb;
                tpB = b3 ^ nb;
            }
            const uint32_t vA[6] = {a0, a1, a2, a3, xA, tpA}, vB[6] = {b0, b1, b2, b3, xB, tpB};
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                sio.st(k, sA, vA[k]);
                sio.st(k, sB, vB[k]);
            }
        }
    }
    if constexpr (kTma && !kStg) {
        if (lane == 0) bulk_wait_read<0>();  // smem must outlive the reads; global completion is ordered by the grid boundary
        __syncwarp();
    }
    sink.finish(a);
}

// ------------------------------------------------------------ band kernel
// The HBM-friendly store path.  A warp owns a 64-stream tile; its output is
// one contiguous slab of 64 rows x n words.  The tile is staged in shared
// memory as kBands "bands" of 32 rounds (128 bytes) per row and written by
// ONE 3-D TMA store per box: tensor map {32 words, rows (stride 4n bytes),
// bands (stride 128 bytes)}, box {32, 64, kBands}, 128-byte swizzle.  With
// kBands * 32 >= n a single bulk op writes the whole contiguous slab, so HBM
// sees long contiguous runs instead of 128-byte pieces 4n bytes apart
// (tools/pattern_bench: 7.16 TB/s vs 6.87 TB/s for 2-D 32-round boxes at
// n = 128, 7.27 TB/s for a plain contiguous fill).  Requires n % 32 == 0.
//
// Persistent: each warp walks tiles tile, tile + W, ...; the state of its
// next tile is prefetched into registers while the current one computes.
template <int kBands, int kBufs>
// launch-bounds minimum 1 = relaxed register budget (64 instead of 58):
// 2^20 x 256 1.562 -> 1.595e12, 2^20 x 1024 +0.5 %, 2^23 x 256 unchanged
// (profiles/experiments/s46_band_launch_bounds.jsonl)
#ifndef CIPRNG_EXP_BAND_MINB
#define CIPRNG_EXP_BAND_MINB 1
#endif
__global__ void __launch_bounds__(256, CIPRNG_EXP_BAND_MINB) v1_band_kernel(GenArgs a, const __grid_constant__ CUtensorMap tmap) {
    constexpr uint32_t kBoxRounds = 32 * kBands;
    constexpr uint32_t kBoxBytes = 64 * kBoxRounds * 4;
    pdl_launch_dependents();
    pdl_wait();  // previous grid on the stream complete + visible
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t h = lane >> 4, j = lane & 15u;
    const uint32_t src = (j + 1u) & 15u;
    const uint64_t n_tiles = (a.s_count + kFastTileRows - 1) / kFastTileRows;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    const StateIO sio(a);
    const uint32_t rA_t = 32u * h + j, rB_t = rA_t + 16u;
    // swizzled smem offsets of this lane's two rows (row r of a band lives at
    // band*8192 + r*128, 16-byte chunk c at (c ^ (r & 7)) * 16)
    const uint32_t offA = rA_t * 128u, offB = rB_t * 128u;
    const uint32_t swA = rA_t & 7u, swB = rB_t & 7u;

    extern __shared__ __align__(1024) uint8_t smem_dyn[];
    const uint32_t wsmem = ((smem_u32(smem_dyn) + 1023u) & ~1023u) + (threadIdx.x >> 5) * (kBufs * kBoxBytes);
    uint32_t issued = 0;

    uint64_t tile = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    // prefetched state of `tile`
    uint32_t pa[6] = {0, 0, 0, 0, 0, 0}, pb[6] = {0, 0, 0, 0, 0, 0};
    auto prefetch = [&](uint64_t t) {
        const uint64_t row0 = t * kFastTileRows;
        if (t < n_tiles && row0 + 32u * h < a.s_count) {
            const uint64_t sA = a.s_begin + row0 + rA_t, sB = sA + 16u;
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                pa[k] = sio.ld(k, sA);
                pb[k] = sio.ld(k, sB);
            }
        }
    };
    prefetch(tile);
    for (; tile < n_tiles; tile += warps) {
        const uint64_t row0 = tile * kFastTileRows;
        const bool valid = row0 + 32u * h < a.s_count;
        uint32_t a0 = pa[0], a1 = pa[1], a2 = pa[2], a3 = pa[3], xA = pa[4];
        uint32_t b0 = pb[0], b1 = pb[1], b2 = pb[2], b3 = pb[3], xB = pb[4];
        uint32_t u = pa[5] ^ pb[5];
        uint32_t nb = 0;
        prefetch(tile + warps);  // lands while this tile computes

#define CIPRNG_V1_ROUND(GA, GA3, GB, GB3, OA, OB) \
    GA = xor128_f(GA, GA3);                       \
    GB = xor128_f(GB, GB3);                       \
    nb = __shfl_sync(kFull, u, src, 16);          \
    xA ^= GA ^ nb;                                \
    xB ^= GB ^ nb;                                \
    u = GA ^ GB;                                  \
    OA = xA;                                      \
    OB = xB;
#define CIPRNG_V1_BLOCK4(Q)                                                                   \
    {                                                                                         \
        uint32_t oA0, oA1, oA2, oA3, oB0, oB1, oB2, oB3;                                      \
        CIPRNG_V1_ROUND(a0, a3, b0, b3, oA0, oB0)                                             \
        CIPRNG_V1_ROUND(a1, a0, b1, b0, oA1, oB1)                                             \
        CIPRNG_V1_ROUND(a2, a1, b2, b1, oA2, oB2)                                             \
        CIPRNG_V1_ROUND(a3, a2, b3, b2, oA3, oB3)                                             \
        const uint32_t band = (Q) >> 3, c = (Q) & 7u;                                         \
        st_shared_v4(buf + band * 8192u + offA + ((c ^ swA) << 4), oA0, oA1, oA2, oA3);       \
        st_shared_v4(buf + band * 8192u + offB + ((c ^ swB) << 4), oB0, oB1, oB2, oB3);       \
    }
        for (uint64_t i0 = 0; i0 < a.n; i0 += kBoxRounds) {
            const uint32_t buf = wsmem + (issued % kBufs) * kBoxBytes;
            if (issued >= kBufs) {
                if (lane == 0) bulk_wait_read<kBufs - 1>();
                __syncwarp();
            }
            if (i0 + kBoxRounds <= a.n) {
#pragma unroll 8
                for (uint32_t q = 0; q < kBoxRounds / 4; ++q) CIPRNG_V1_BLOCK4(q)
            } else {
                for (uint32_t q = 0; i0 + 4 * q < a.n; ++q) CIPRNG_V1_BLOCK4(q)
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
                asm volatile(
                    "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3, %4}], [%1], %5;" ::"l"(
                        reinterpret_cast<uint64_t>(&tmap)),
                    "r"(buf), "r"(0), "r"((int)row0), "r"((int)(i0 >> 5)),
                    "l"(a.evict_first ? l2_evict_first_policy() : l2_evict_normal_policy())
                    : "memory");
                bulk_commit();
            }
            ++issued;
        }
#undef CIPRNG_V1_BLOCK4
#undef CIPRNG_V1_ROUND
        if (valid) {
            const uint64_t sA = a.s_begin + row0 + rA_t, sB = sA + 16u;
            // n > 0 (the host never launches n == 0): last t = g ^ nb
            const uint32_t vA[6] = {a0, a1, a2, a3, xA, a3 ^ nb}, vB[6] = {b0, b1, b2, b3, xB, b3 ^ nb};
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                sio.st(k, sA, vA[k]);
                sio.st(k, sB, vB[k]);
            }
        }
    }
    if (lane == 0) bulk_wait_read<0>();  // smem must outlive the reads; global completion is ordered by the grid boundary
    __syncwarp();
}

// ===================================================================== launch
static int blocks_for(uint64_t warps_needed, int warps_per_block, int cap_blocks) {
    uint64_t b = (warps_needed + warps_per_block - 1) / warps_per_block;
    if (cap_blocks > 0 && b > (uint64_t)cap_blocks) b = cap_blocks;
    if (b == 0) b = 1;
    return (int)b;
}

template <int kBands, int kBufs>
static void launch_band(const GenArgs &a, const CUtensorMap &tm, uint64_t tiles, int wpb, int grid_mode,
                        cudaStream_t st) {
    const size_t smem = (size_t)wpb * kBufs * 64 * 32 * kBands * 4 + 1024;  // + alignment slack
    auto kern = v1_band_kernel<kBands, kBufs>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int grid = blocks_for(tiles, wpb, 0);
    if (grid_mode != 0) {
        int dev = 0, sms = 148, per_sm = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * wpb, smem);
        if (grid_mode > 0 && grid_mode < per_sm) per_sm = grid_mode;
        if (per_sm < 1) per_sm = 1;
        grid = blocks_for(tiles, wpb, per_sm * sms);
    }
    launch_k(kern, dim3(grid), dim3(32 * wpb), smem, st, a, tm);
}

template <int kCols, int kBufs = 2, bool kStg = false>
static void launch_fast_tma(const GenArgs &a0, const CUtensorMap &tm, int grid, int wpb, bool pf, cudaStream_t st) {
    const size_t smem = (size_t)wpb * kBufs * kFastTileRows * kCols * 4 + 1024;  // + alignment slack
    auto kern = v1_fast_kernel<StoreSink, kCols, kBufs, kStg>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    GenArgs a = a0;
    // one wave of resident warps ahead (non-persistent grid: the tile the
    // warp replacing this one in a later wave will take)
    a.pf_ahead = pf && grid > resident_blocks(reinterpret_cast<const void *>(kern), 32 * wpb, smem)
                     ? (uint32_t)(resident_blocks(reinterpret_cast<const void *>(kern), 32 * wpb, smem) * wpb)
                     : 0u;
    launch_k(kern, dim3(grid), dim3(32 * wpb), smem, st, a, tm);
}

static_assert(StatsSinkCta::kResv == (uint32_t)kCtaHistResvBytes, "reserved shared memory assumption");
static void launch_v1_consume_cta(const GenArgs &a, const CUtensorMap &tm, uint64_t tiles, cudaStream_t st) {
    launch_cta_hist(v1_fast_kernel<StatsSinkCta, 0>, StatsSinkCta::kWarps, StatsSinkCta::kSmemBytesExtra, tiles, a.n,
                    st, a, tm);
}

int launch_v1(const GenArgs &a, bool fast, int mode, const CUtensorMap *tmap, cudaStream_t st,
              const V1Tuning &tune) {
    // mode: 0 store-direct, 1 store-tma, 2 consume, 3 battery, 4 store staged (smem + coalesced STG)
    if (a.s_count == 0) return 0;
    if (fast) {
        const uint64_t tiles = (a.s_count + kFastTileRows - 1) / kFastTileRows;
        const int wpb = tune.wpb > 0 ? tune.wpb : 4;
        int cap = tune.grid_blocks > 0 ? tune.grid_blocks : 0;
        if (cap == 0 && tune.tiles_per_warp > 1)
            cap = (int)((tiles + (uint64_t)wpb * tune.tiles_per_warp - 1) / ((uint64_t)wpb * tune.tiles_per_warp));
        CUtensorMap dummy;
        if (tmap == nullptr) tmap = &dummy;
        if (mode == 4 || (mode == 0 && tune.smem_stg)) {
            // store path (b): shared-memory transpose + coalesced STG (any alignment, any n);
            // mode 4 = the AUTO fallback when no TMA descriptor applies
            launch_fast_tma<32, 1, true>(a, *tmap, blocks_for(tiles, wpb, cap), wpb, false, st);
        } else if (mode == 0) {
            launch_k(v1_fast_kernel<StoreSink, 0>, dim3(blocks_for(tiles, wpb, cap)), dim3(32 * wpb), 0, st, a, *tmap);
        } else if (mode == 1) {
            const int grid = blocks_for(tiles, wpb, cap);
            if (tune.cols == 64 && tune.bufs == 1) launch_band<2, 1>(a, *tmap, tiles, wpb, tune.grid_mode, st);
            else if (tune.cols == 64) launch_band<2, 2>(a, *tmap, tiles, wpb, tune.grid_mode, st);
            else if (tune.cols == 128) launch_band<4, 1>(a, *tmap, tiles, wpb, tune.grid_mode, st);
            else if (tune.cols == 8) launch_fast_tma<8>(a, *tmap, grid, wpb, tune.l2_prefetch, st);
            else if (tune.cols == 32 && tune.bufs == 1) launch_fast_tma<32, 1>(a, *tmap, grid, wpb, tune.l2_prefetch, st);
            else if (tune.cols == 32 && tune.bufs == 3) launch_fast_tma<32, 3>(a, *tmap, grid, wpb, tune.l2_prefetch, st);
            else if (tune.cols == 32) launch_fast_tma<32>(a, *tmap, grid, wpb, tune.l2_prefetch, st);
            else launch_fast_tma<16>(a, *tmap, grid, wpb, tune.l2_prefetch, st);
        } else {
            const uint64_t need = (tiles + 3) / 4;
            if (mode == 3) {
#if !defined(CIPRNG_BATTERY_HIST_WARP)
                if (cta_hist_ok()) {  // 4 byte-bin increments per word: the grid bound takes 4n
                    launch_cta_hist(v1_fast_kernel<BatterySinkCta, 0>, BatterySinkCta::kWarps,
                                    BatterySinkCta::kSmemBytesExtra, tiles, 4 * a.n, st, a, *tmap);
                    return 1;
                }
#endif
                auto kern = v1_fast_kernel<BatterySink, 0>;
                const size_t sm = 4 * BatterySink::kSmemBytesPerWarp + BatterySink::kSmemBytesExtra;
                launch_k(kern, dim3(persistent_grid(kern, 128, sm, need)), dim3(128), sm, st, a, *tmap);
            } else {
#if defined(CIPRNG_V1_HIST_PRIV)
                // experiment: per-lane private histogram columns (sinks.cuh StatsSinkLane)
                constexpr int kW = CIPRNG_V1_HIST_PRIV;  // warps per CTA
                auto kern = v1_fast_kernel<StatsSinkLane, 0>;
                const size_t sm = kW * StatsSinkLane::kSmemBytesPerWarp + StatsSinkLane::kSmemBytesExtra;
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
                const uint64_t needw = (tiles + kW - 1) / kW;
                launch_k(kern, dim3(persistent_grid(kern, 32 * kW, sm, needw)), dim3(32 * kW), sm, st, a, *tmap);
#else
                // default: one conflict-free histogram per CTA (StatsSinkCta);
                // the per-warp histograms (StatsSink) when the driver's reserved
                // shared memory is not the 1 KiB the CTA sink's addressing assumes,
                // or for the comparison build CIPRNG_V1_HIST_WARP
#if !defined(CIPRNG_V1_HIST_WARP)
                if (cta_hist_ok()) {
                    launch_v1_consume_cta(a, *tmap, tiles, st);
                    return 1;
                }
#endif
                auto kern = v1_fast_kernel<StatsSink, 0>;
                const size_t sm = 4 * StatsSink::kSmemBytesPerWarp + StatsSink::kSmemBytesExtra;
                launch_k(kern, dim3(persistent_grid(kern, 128, sm, need)), dim3(128), sm, st, a, *tmap);
#endif
            }
        }
    } else {
        const uint64_t tiles = (a.s_count + 31) / 32;
        const int wpb = 8;
        const uint64_t need = (tiles + wpb - 1) / wpb;
        if (mode == 2) {
            auto kern = v1_general_kernel<StatsSink>;
            const size_t sm = wpb * StatsSink::kSmemBytesPerWarp + StatsSink::kSmemBytesExtra;
            launch_k(kern, dim3(persistent_grid(kern, 32 * wpb, sm, need)), dim3(32 * wpb), sm, st, a);
        } else if (mode == 3) {
            auto kern = v1_general_kernel<BatterySink>;
            const size_t sm = wpb * BatterySink::kSmemBytesPerWarp + BatterySink::kSmemBytesExtra;
            launch_k(kern, dim3(persistent_grid(kern, 32 * wpb, sm, need)), dim3(32 * wpb), sm, st, a);
        } else {
            int grid = blocks_for(tiles, wpb, 0);
            launch_k(v1_general_kernel<StoreSink>, dim3(grid), dim3(32 * wpb), 0, st, a);
        }
    }
    return 1;
}

}  // namespace ciprng
