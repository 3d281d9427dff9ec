// gen_comb.cu -- V3: Alg. 4's neighbour combination
// with the xor64 source of the paper's "optimized versions" (P:1026-1028,
// "the optimized versions use the xor64 described in [Marsaglia2003]"),
// SURVEY s8(f) NEXT-1 (i).  Reading Q29: Alg. 4's t is a 32-bit word
// (P:950), so t = xor64() takes the low 32 bits of the 64-bit output.
//
// Per stream: xor64 state a (two u32 halves), x, the shared cell tp.  Per
// round:  t = lo(xor64(a)) ^ tp[o1] ^ tp[o2];  tp = t;  x ^= t;  emit x.
//
// The kernels are templated on the strategy source (`Src`): the exchange,
// store and consume machinery is the V1 design (gen_v1.cu) --
//  * comb_general_kernel: any C | 32 and any arrays, one lane per stream,
//    two SHFL.IDX per number;
//  * comb_fast_kernel: the default arrays comb1 = l+1, comb2 = l+17 (Q6):
//    lane j of a half-warp owns streams j and j+16, one width-16 SHFL per
//    two numbers (u[j] = tp[j] ^ tp[j+16] trick, see gen_v1.cu), and either
//    128-bit STG or 64-stream x 32-round TMA tiles (2-D bulk tensor store).
#include <cstdlib>

#include <type_traits>

#include "device.cuh"
#include "kernels.h"
#include "sinks.cuh"

namespace ciprng {

// Marsaglia xor64 (13, 7, 17) on (lo, hi) halves (device.cuh u64p helpers:
// plain halves as IMAD.SHL / IMAD.HI, funnel halves on SHF).
template <int kFun>
struct SrcXor64T {
    static constexpr int kPlanes = 2;  // a.lo, a.hi; then x, tp
    u64p a;
    __device__ __forceinline__ void load(const StateIO &io, uint64_t s) {
        a.lo = io.ld(0, s);
        a.hi = io.ld(1, s);
    }
    __device__ __forceinline__ void store(const StateIO &io, uint64_t s) const {
        io.st(0, s, a.lo);
        io.st(1, s, a.hi);
    }
    __device__ __forceinline__ void zero() { a = {0u, 0u}; }
    __device__ __forceinline__ uint32_t next() {
        a = xor64_step_p<kFun>(a);
        return a.lo;  // Q29
    }
};

// all three funnels on SHF: multiply funnels measured slower (L2 flushed:
// none 1.218e12, 13L 1.184e12, 13L+17L 1.083e12 numbers/s; profiles/experiments/s19)
constexpr int kV3FunnelDefault = 0;
using SrcXor64 = SrcXor64T<kV3FunnelDefault>;

// ===================================================================== general
template <class Src, class Sink>
__global__ void __launch_bounds__(256) comb_general_kernel(GenArgs a) {
    constexpr int X = Src::kPlanes, TP = Src::kPlanes + 1;
    Sink sink(a);
    pdl_launch_dependents();
    pdl_wait();
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
        Src g;
        uint32_t x = 0, tp = 0;
        g.zero();
        if (valid) {
            g.load(sio, s);
            x = sio.ld(X, s);
            tp = sio.ld(TP, s);
        }
        sink.begin_row(0, row);
        auto round = [&]() -> uint32_t {
            const uint32_t t = g.next() ^ __shfl_sync(kFull, tp, src1) ^ __shfl_sync(kFull, tp, src2);
            tp = t;
            x ^= t;
            return x;
        };
        uint64_t i = 0;
        for (; i + 4 <= a.n; i += 4) {
            const uint32_t o0 = round(), o1 = round(), o2 = round(), o3 = round();
            sink.put4(0, i, o0, o1, o2, o3, valid);
        }
        for (; i < a.n; ++i) sink.put1(0, i, round(), valid);
        sink.end_rows(valid ? 1u : 0u);
        if (valid) {
            g.store(sio, s);
            sio.st(X, s, x);
            sio.st(TP, s, tp);
        }
    }
    sink.finish(a);
}

// ======================================================================== fast
constexpr int kCombTileRows = 64;

template <class Sink, int kCols, bool kStg>
constexpr int comb_fast_min_blocks() {
    return (kLbForceMin1 || (std::is_same<Sink, StoreSink>::value && kCols > 0 && !kStg)) ? 1 : 0;
}

template <class Sink>
constexpr int comb_fast_max_threads() {
    return Sink::kCtaHist ? 32 * cta_hist_warps<Sink>() : 256;
}
template <class Sink, int kCols, bool kStg>
constexpr int comb_fast_min_blocks_x() {
    return Sink::kCtaHist ? cta_hist_min_blocks<Sink>() : comb_fast_min_blocks<Sink, kCols, kStg>();
}

template <class Src, class Sink, int kCols, bool kStg = false>
__global__ void __launch_bounds__((comb_fast_max_threads<Sink>()), (comb_fast_min_blocks_x<Sink, kCols, kStg>())) comb_fast_kernel(GenArgs a, const __grid_constant__ CUtensorMap tmap) {
    constexpr int X = Src::kPlanes, TP = Src::kPlanes + 1;
    constexpr bool kTma = kCols > 0;
    constexpr uint32_t kTileBytes = kCombTileRows * (kCols > 0 ? kCols : 4) * 4;
    Sink sink(a);
    pdl_launch_dependents();
    pdl_wait();
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t h = lane >> 4, j = lane & 15u;
    const uint32_t src = (j + 1u) & 15u;
    const uint64_t n_tiles = (a.s_count + kCombTileRows - 1) / kCombTileRows;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    const StateIO sio(a);
    const uint32_t rA_t = 32u * h + j, rB_t = rA_t + 16u;

    uint32_t wsmem = 0;
    if constexpr (kTma) {
        extern __shared__ __align__(1024) uint8_t smem_dyn[];
        const uint32_t base = (smem_u32(smem_dyn) + 1023u) & ~1023u;
        wsmem = base + (threadIdx.x >> 5) * (2 * kTileBytes);
    }
    uint32_t issued = 0;

    for (uint64_t tile = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); tile < n_tiles;
         tile += warps) {
        const uint64_t row0 = tile * kCombTileRows;
        const bool valid = row0 + 32u * h < a.s_count;
        const uint64_t rA = row0 + rA_t, rB = row0 + rB_t;
        const uint64_t sA = a.s_begin + rA, sB = a.s_begin + rB;
        Src gA, gB;
        uint32_t xA = 0, tpA = 0, xB = 0, tpB = 0;
        gA.zero();
        gB.zero();
        if (valid) {
            gA.load(sio, sA);
            gB.load(sio, sB);
            xA = sio.ld(X, sA); tpA = sio.ld(TP, sA);
            xB = sio.ld(X, sB); tpB = sio.ld(TP, sB);
        }
        sink.begin_row(0, rA);
        sink.begin_row(1, rB);
        uint32_t u = tpA ^ tpB, nb = 0, lastA = 0, lastB = 0;
        // one round for both of the lane's streams: u[j] = t[j] ^ t[j+16] of
        // the previous round; both streams need tp[j+1] ^ tp[j+17] = u[j+1]
        auto round2 = [&](uint32_t &oA, uint32_t &oB) {
            lastA = gA.next();
            lastB = gB.next();
            nb = __shfl_sync(kFull, u, src, 16);
            xA ^= lastA ^ nb;
            xB ^= lastB ^ nb;
            u = lastA ^ lastB;
            oA = xA;
            oB = xB;
        };
        uint64_t i = 0;
        if constexpr (kTma) {
            // staged store path (kStg): boxes over the first n - n%4 rounds,
            // scalar tail after; TMA: n % 4 == 0 (host)
            const uint64_t nb4 = kStg ? (a.n & ~3ull) : a.n;
            for (uint64_t i0 = 0; i0 < nb4; i0 += kCols) {
                const uint32_t buf = wsmem + (issued & 1u) * kTileBytes;
                if (!kStg && issued >= 2) {
                    if (lane == 0) bulk_wait_read<1>();
                    __syncwarp();
                }
                const uint32_t q_end = (i0 + kCols <= nb4) ? kCols / 4 : (uint32_t)((nb4 - i0) / 4);
#pragma unroll 8
                for (uint32_t q = 0; q < q_end; ++q) {
                    uint32_t oA0, oA1, oA2, oA3, oB0, oB1, oB2, oB3;
                    round2(oA0, oB0);
                    round2(oA1, oB1);
                    round2(oA2, oB2);
                    round2(oA3, oB3);
                    st_shared_v4(buf + swz<kCols>(rA_t, q), oA0, oA1, oA2, oA3);
                    st_shared_v4(buf + swz<kCols>(rB_t, q), oB0, oB1, oB2, oB3);
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
                ++issued;
            }
            i = nb4;
            if constexpr (kStg) {
                for (; i < a.n; ++i) {  // the last n % 4 rounds: scalar stores
                    uint32_t oA, oB;
                    round2(oA, oB);
                    sink.put1(0, i, oA, valid);
                    sink.put1(1, i, oB, valid);
                }
            }
        } else {
            auto block4 = [&](uint64_t i4) {
                uint32_t oA0, oA1, oA2, oA3, oB0, oB1, oB2, oB3;
                round2(oA0, oB0);
                round2(oA1, oB1);
                round2(oA2, oB2);
                round2(oA3, oB3);
                sink.put4(0, i4, oA0, oA1, oA2, oA3, valid);
                sink.put4(1, i4, oB0, oB1, oB2, oB3, valid);
            };
            if constexpr (Sink::kStats) {
                // consumers: n < 2^24 (host-checked), 32-bit trip counter and
                // index, as in the V1 consumer (gen_v1.cu)
                const uint32_t n4 = (uint32_t)a.n & ~3u;
                for (uint32_t i32 = 0; i32 != n4; i32 += 4) block4(i32);
                i = n4;
            } else {
                for (; i + 4 <= a.n; i += 4) block4(i);
            }
            for (; i < a.n; ++i) {
                uint32_t oA, oB;
                round2(oA, oB);
                sink.put1(0, i, oA, valid);
                sink.put1(1, i, oB, valid);
            }
        }
        sink.end_rows(valid ? 2u : 0u);
        if (valid) {
            if (a.n > 0) {  // last round's t = g ^ nb
                tpA = lastA ^ nb;
                tpB = lastB ^ nb;
            }
            gA.store(sio, sA);
            gB.store(sio, sB);
            sio.st(X, sA, xA); sio.st(TP, sA, tpA);
            sio.st(X, sB, xB); sio.st(TP, sB, tpB);
        }
    }
    if constexpr (kTma && !kStg) {
        if (lane == 0) bulk_wait_read<0>();
        __syncwarp();
    }
    sink.finish(a);
}

// ===================================================================== launch
static int comb_blocks(uint64_t warps_needed, int wpb, int cap) {
    uint64_t b = (warps_needed + wpb - 1) / wpb;
    if (cap > 0 && b > (uint64_t)cap) b = cap;
    return (int)(b ? b : 1);
}

template <class Src>
static int launch_comb(const GenArgs &a, bool fast, int mode, const CUtensorMap *tmap, cudaStream_t st) {
    // mode: 0 store-direct, 1 store-tma, 2 consume, 3 battery, 4 store staged
    if (a.s_count == 0) return 0;
    CUtensorMap dummy;
    if (tmap == nullptr) tmap = &dummy;
    if (fast) {
        const uint64_t tiles = (a.s_count + kCombTileRows - 1) / kCombTileRows;
        if (mode == 4) {  // staged shared-memory + coalesced STG (no TMA descriptor)
            constexpr int kCols = 32, wpb = 2;
            const size_t smem = (size_t)wpb * 2 * kCombTileRows * kCols * 4 + 1024;
            auto kern = comb_fast_kernel<Src, StoreSink, kCols, true>;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            launch_k(kern, dim3(comb_blocks(tiles, wpb, 0)), dim3(32 * wpb), smem, st, a, *tmap);
        } else if (mode == 1) {
            constexpr int kCols = CIPRNG_V3_COLS, wpb = CIPRNG_V3_WPB;  // kernels.h (s18, s41)
            const size_t smem = (size_t)wpb * 2 * kCombTileRows * kCols * 4 + 1024;
            auto kern = comb_fast_kernel<Src, StoreSink, kCols>;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            launch_k(kern, dim3(comb_blocks(tiles, wpb, 0)), dim3(32 * wpb), smem, st, a, *tmap);
        } else if (mode == 0) {
            launch_k(comb_fast_kernel<Src, StoreSink, 0>, dim3(comb_blocks(tiles, 4, 0)), dim3(128), 0, st, a, *tmap);
        } else if (mode == 2) {
#if !defined(CIPRNG_V3_HIST_WARP)
            // the CTA histogram (sinks.cuh StatsSinkCta): an invalid half-warp
            // runs on an all-zero xor64 state and emits zeros, as the sink needs
            if (cta_hist_ok()) {
                static_assert(StatsSinkCta::kResv == (uint32_t)kCtaHistResvBytes, "reserved shared memory");
                launch_cta_hist(comb_fast_kernel<Src, StatsSinkCta, 0>, StatsSinkCta::kWarps,
                                StatsSinkCta::kSmemBytesExtra, tiles, a.n, st, a, *tmap);
                return 1;
            }
#endif
            auto kern = comb_fast_kernel<Src, StatsSink, 0>;
            const size_t sm = 4 * StatsSink::kSmemBytesPerWarp + StatsSink::kSmemBytesExtra;
            launch_k(kern, dim3(persistent_grid(kern, 128, sm, (tiles + 3) / 4)), dim3(128), sm, st, a, *tmap);
        } else {
#if !defined(CIPRNG_BATTERY_HIST_WARP)
            if (cta_hist_ok()) {
                launch_cta_hist(comb_fast_kernel<Src, BatterySinkCta, 0>, BatterySinkCta::kWarps,
                                BatterySinkCta::kSmemBytesExtra, tiles, 4 * a.n, st, a, *tmap);
                return 1;
            }
#endif
            auto kern = comb_fast_kernel<Src, BatterySink, 0>;
            const size_t sm = 4 * BatterySink::kSmemBytesPerWarp + BatterySink::kSmemBytesExtra;
            launch_k(kern, dim3(persistent_grid(kern, 128, sm, (tiles + 3) / 4)), dim3(128), sm, st, a, *tmap);
        }
    } else {
        const uint64_t tiles = (a.s_count + 31) / 32;
        const int wpb = 8;
        if (mode == 2) {
            auto kern = comb_general_kernel<Src, StatsSink>;
            const size_t sm = wpb * StatsSink::kSmemBytesPerWarp + StatsSink::kSmemBytesExtra;
            launch_k(kern, dim3(persistent_grid(kern, 32 * wpb, sm, (tiles + wpb - 1) / wpb)), dim3(32 * wpb), sm, st, a);
        } else if (mode == 3) {
            auto kern = comb_general_kernel<Src, BatterySink>;
            const size_t sm = wpb * BatterySink::kSmemBytesPerWarp + BatterySink::kSmemBytesExtra;
            launch_k(kern, dim3(persistent_grid(kern, 32 * wpb, sm, (tiles + wpb - 1) / wpb)), dim3(32 * wpb), sm, st, a);
        } else {
            launch_k(comb_general_kernel<Src, StoreSink>, dim3(comb_blocks(tiles, wpb, 0)), dim3(32 * wpb), 0, st, a);
        }
    }
    return 1;
}

int launch_v3(const GenArgs &a, bool fast, int mode, const CUtensorMap *tmap, cudaStream_t st) {
    return launch_comb<SrcXor64>(a, fast, mode, tmap, st);
}

}  // namespace ciprng
