// gen_v0.cu -- V0: Listing 1 run by every thread = Alg. 3 "naive" kernel
// on sm_100a.
//
// Per stream: xor64 a (Q1-A), xor128 on u64 b0..b3 (Q2), xorwow on u64
// c0..c4 + Weyl d (Q2, Q3), and x.  Per round:
//   t1 = xorshift(); t2 = xor128(); t3 = xorwow();
//   x ^= lo(t1) ^ hi(t2) ^ hi(t3) ^ lo(t2) ^ hi(t1) ^ lo(t3);  emit x
// Streams are independent (no neighbour exchange).  64-bit shifts and XORs
// become SHF/LOP3 pairs; the xor128 (period-4 register ring) and xorwow
// (period-5 ring) recurrences are unrolled 20 rounds deep so the state never
// moves between registers.  Integer-issue bound, not HBM bound.
//
// kComb = true is V4 (reading Q30): the same fold
// f is Alg. 4's strategy source, t = f ^ tp[o1] ^ tp[o2]; tp = t; x ^= t
// (P:971-974), the group's shared cells exchanged by two SHFL.IDX per number
// (any C | 32 and any arrays; the draw, not the shuffle, is the cost here).
#include <cstdlib>
#include <type_traits>

#include "device.cuh"
#include "kernels.h"
#include "sinks.cuh"

namespace ciprng {

__device__ __forceinline__ uint32_t fold6(uint64_t t1, uint64_t t2, uint64_t t3) {
    return (uint32_t)t1 ^ (uint32_t)(t2 >> 32) ^ (uint32_t)(t3 >> 32) ^ (uint32_t)t2 ^ (uint32_t)(t1 >> 32) ^
           (uint32_t)t3;
}

// Which funnel shifts run as multiplies (device.cuh shl64/shr64 kF), as a
// 9-bit mask: bits 0-2 xor64 (13L, 7R, 17L), 3-5 xor128 (11L, 19R, 8R),
// 6-8 xorwow (2R, 4L, 1L).  Measured with L2 flushed (profiles/experiments/
// s19_funnel_summary.txt): all-SHF 4.59e11 numbers/s, 2 multiply funnels
// 4.51e11, 6 -> 3.38e11, all 9 -> 3.26e11 -- the heavy sub-pipe costs more
// than the ALU op it saves, so every funnel stays an SHF.
constexpr int kFunnelDefault = 0;

// CTA shape knobs (experiments through CIPRNG_NVCC_EXTRA): warps per CTA,
// min CTAs per SM for the register budget, and shared-memory padding per
// store CTA (limits residency, so the wave count of the grid can be chosen).
// Measured (profiles/experiments/s43_v0_cta_shape.jsonl): 4 or 8 warps per
// CTA and 5.5 vs 6.9 waves all within 1 % (4.56-4.57e11); padding to fewer
// resident warps -1 %, forcing 44 warps/SM (40 registers, spills) -29 %.
#ifndef CIPRNG_V0_WPB
#define CIPRNG_V0_WPB 8
#endif
#ifndef CIPRNG_V0_MINB
#define CIPRNG_V0_MINB 1
#endif
#ifndef CIPRNG_V0_PAD_SMEM
#define CIPRNG_V0_PAD_SMEM 0
#endif

// Launch-bounds minimum (kernels.h kLbForceMin1): 1 = relaxed register
// budget, 0 = ptxas' default (48 registers for the V0 store, 81 with 1).
template <class Sink, bool kComb>
constexpr int v0_min_blocks() {
    return CIPRNG_V0_MINB > 1 ? CIPRNG_V0_MINB
           : (kLbForceMin1 || (std::is_same<Sink, StatsSink>::value && !kComb) ||
              (std::is_same<Sink, StoreSink>::value && kComb))
               ? 1
               : 0;
}

template <class Sink, bool kComb, int kFun = kFunnelDefault>
__global__ void __launch_bounds__(32 * CIPRNG_V0_WPB, (v0_min_blocks<Sink, kComb>())) v0_kernel(GenArgs a) {
    constexpr int kFunnelXor64 = kFun & 7, kFunnelXor128 = (kFun >> 3) & 7, kFunnelXorwow = (kFun >> 6) & 7;
    Sink sink(a);
    pdl_launch_dependents();
    pdl_wait();  // previous grid on the stream complete + visible
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t off = lane % a.C, gbase = lane - off;  // V4 only
    const uint32_t src1 = gbase + a.comb.t[0][off], src2 = gbase + a.comb.t[1][off];
    const uint64_t n_tiles = (a.s_count + 31) / 32;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    const StateIO sio(a);

    for (uint64_t tile = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); tile < n_tiles;
         tile += warps) {
        const uint64_t row = tile * 32 + lane;
        const bool valid = row < a.s_count;
        const uint64_t s = a.s_begin + row;
        uint64_t ra = 0, rb[4] = {0, 0, 0, 0}, rc[5] = {0, 0, 0, 0, 0}, rd = 0;
        uint32_t x = 0, tp = 0;
        auto ld64 = [&](int k) -> uint64_t {
            return (uint64_t)sio.ld(2 * k, s) | ((uint64_t)sio.ld(2 * k + 1, s) << 32);
        };
        if (valid) {
            ra = ld64(0);
#pragma unroll
            for (int k = 0; k < 4; ++k) rb[k] = ld64(1 + k);
#pragma unroll
            for (int k = 0; k < 5; ++k) rc[k] = ld64(5 + k);
            rd = ld64(10);
            x = sio.ld(22, s);
            if (kComb) tp = sio.ld(23, s);
        }
        // x ^= f (V0), or Alg. 4's combination with f as the source (V4)
        auto update = [&](uint32_t f) {
            if constexpr (kComb) {
                const uint32_t t = f ^ __shfl_sync(kFull, tp, src1) ^ __shfl_sync(kFull, tp, src2);
                tp = t;
                x ^= t;
            } else {
                x ^= f;
            }
        };
        sink.begin_row(0, row);
        uint64_t i = 0;
        for (; i + 20 <= a.n; i += 20) {
            // unrolled on (lo, hi) halves: funnel shifts on the ALU pipe, plain
            // shifts as multiplies on the FMA pipe (device.cuh, u64p)
            u64p pa = {(uint32_t)ra, (uint32_t)(ra >> 32)}, pd = {(uint32_t)rd, (uint32_t)(rd >> 32)};
            u64p pb[4], pc[5];
#pragma unroll
            for (int k = 0; k < 4; ++k) pb[k] = {(uint32_t)rb[k], (uint32_t)(rb[k] >> 32)};
#pragma unroll
            for (int k = 0; k < 5; ++k) pc[k] = {(uint32_t)rc[k], (uint32_t)(rc[k] >> 32)};
            const u64p weyl = {362437u, 0u};
            uint32_t o[4];
#pragma unroll
            for (int k = 0; k < 20; ++k) {
                pa = xor64_step_p<kFunnelXor64>(pa);
                pb[k % 4] = xor128_f64p<kFunnelXor128>(pb[k % 4], pb[(k + 3) % 4]);
                pc[k % 5] = xorwow_f64p<kFunnelXorwow>(pc[k % 5], pc[(k + 4) % 5]);
                pd = add64p(pd, weyl);
                const u64p t3 = add64p(pd, pc[k % 5]);
                update(pa.lo ^ pb[k % 4].hi ^ t3.hi ^ pb[k % 4].lo ^ pa.hi ^ t3.lo);
                o[k % 4] = x;
                if (k % 4 == 3) sink.put4(0, i + k - 3, o[0], o[1], o[2], o[3], valid);
            }
            ra = (uint64_t)pa.hi << 32 | pa.lo;
            rd = (uint64_t)pd.hi << 32 | pd.lo;
#pragma unroll
            for (int k = 0; k < 4; ++k) rb[k] = (uint64_t)pb[k].hi << 32 | pb[k].lo;
#pragma unroll
            for (int k = 0; k < 5; ++k) rc[k] = (uint64_t)pc[k].hi << 32 | pc[k].lo;
        }
        // tail (fewer than 20 rounds): same recurrences with register moves
        auto step = [&]() -> uint32_t {
            ra = xor64_step(ra);
            uint64_t nb = xor128_f64(rb[0], rb[3]);
            rb[0] = rb[1]; rb[1] = rb[2]; rb[2] = rb[3]; rb[3] = nb;
            uint64_t nc = xorwow_f64(rc[0], rc[4]);
            rc[0] = rc[1]; rc[1] = rc[2]; rc[2] = rc[3]; rc[3] = rc[4]; rc[4] = nc;
            rd += 362437u;
            update(fold6(ra, nb, rd + nc));
            return x;
        };
        for (; i + 4 <= a.n; i += 4) {
            uint32_t o0 = step(), o1 = step(), o2 = step(), o3 = step();
            sink.put4(0, i, o0, o1, o2, o3, valid);
        }
        for (; i < a.n; ++i) sink.put1(0, i, step(), valid);
        sink.end_rows(valid ? 1u : 0u);
        if (valid) {
            auto st64 = [&](int k, uint64_t v) {
                sio.st(2 * k, s, (uint32_t)v);
                sio.st(2 * k + 1, s, (uint32_t)(v >> 32));
            };
            st64(0, ra);
#pragma unroll
            for (int k = 0; k < 4; ++k) st64(1 + k, rb[k]);
#pragma unroll
            for (int k = 0; k < 5; ++k) st64(5 + k, rc[k]);
            st64(10, rd);
            sio.st(22, s, x);
            if (kComb) sio.st(23, s, tp);
        }
    }
    sink.finish(a);
}

template <bool kComb>
static int launch_v0x(const GenArgs &a, int mode, cudaStream_t st) {
    if (a.s_count == 0) return 0;
    const uint64_t tiles = (a.s_count + 31) / 32;
    const int wpb = CIPRNG_V0_WPB;
    uint64_t blocks = (tiles + wpb - 1) / wpb;
    if (mode == 2) {
        auto kern = v0_kernel<StatsSink, kComb>;
        const size_t sm = wpb * StatsSink::kSmemBytesPerWarp + StatsSink::kSmemBytesExtra;
        launch_k(kern, dim3(persistent_grid(kern, 32 * wpb, sm, blocks)), dim3(32 * wpb), sm, st, a);
    } else if (mode == 3) {
        auto kern = v0_kernel<BatterySink, kComb>;
        const size_t sm = wpb * BatterySink::kSmemBytesPerWarp + BatterySink::kSmemBytesExtra;
        launch_k(kern, dim3(persistent_grid(kern, 32 * wpb, sm, blocks)), dim3(32 * wpb), sm, st, a);
    } else {
        auto kern = v0_kernel<StoreSink, kComb>;
        if (CIPRNG_V0_PAD_SMEM > 48 * 1024)
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, CIPRNG_V0_PAD_SMEM);
        launch_k(kern, dim3((int)blocks), dim3(32 * wpb), (size_t)CIPRNG_V0_PAD_SMEM, st, a);
    }
    return 1;
}

int launch_v0(const GenArgs &a, int mode, cudaStream_t st) {
    return launch_v0x<false>(a, mode, st);
}

int launch_v4(const GenArgs &a, int mode, cudaStream_t st) {
    return launch_v0x<true>(a, mode, st);
}

}  // namespace ciprng
