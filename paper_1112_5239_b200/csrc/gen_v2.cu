// gen_v2.cu -- V2: Alg. 5 BBS kernel on sm_100a.
//
// Per stream: 8 BBS instances (y_j, modulus index m_j) with M_j < 2^16
// (Q13), x and the shared cell tp.  Per call: the arrangement
// arrays are chosen from the call-entry states of bbs1 and bbs2:
//   o1 = array_comb[bbs1 & 7], o2 = array_comb[8 + (bbs2 & 7)]  (Q15, Q16)
// Per round:
//   8 x { y_j = y_j^2 mod M_j;  t = (t << 4) | (y_j & 15) }
//   shift = sq(bbs3) & 3;  t <<= shift;  t |= sq(bbs1) & array_shift[shift]
//   shift = sq(bbs7) & 3;  t <<= shift;  t |= sq(bbs2) & array_shift[shift]
//   t ^= tp[o1] ^ tp[o2];  tp = t;  x ^= t;  emit x
// with array_shift[s] = {0,1,3,7}[s] = (1 << s) - 1 (Q17, Q18).
// At the end of a call with n > 0 the (y, m) pairs rotate: instance j is
// stored in place j+1, instance 8 in place 1 (Q19, Q20).
//
// The modulus is division-free (Barrett with mu = floor(2^32 / M), one
// conditional subtraction; device.cuh).  The neighbour exchange is two
// data-dependent SHFL.IDX per number.  12 squarings (~5 integer ops each)
// per number: integer-issue bound.
#include <type_traits>

#include "device.cuh"
#include "kernels.h"
// the V2 consumer keeps the add.cc pi-pair test (sinks.cuh count_outside:
// the mad-carry form is 1.3 % slower on V2's heavy-pipe-bound kernel)
#define CIPRNG_PAIR_ADDCC 1
#include "sinks.cuh"

namespace ciprng {

struct Bbs8 {
    uint32_t y[8], nM[8], mu[8], K[8], iF[8];  // nM = 2^32 - M; K, iF: fbarrett_sq (device.cuh)
    uint32_t yh[8];                            // Montgomery kinds: y*2^32 mod M; nM, mu hold M, Mp
};

// y << k on the ALU pipe (funnel shift with a zero low word): the heavy FMA
// sub-pipe is V2's bound (Barrett's IMAD / IMAD.HI), so the nibble
// placement must not land there as IMAD.SHL.
template <int k>
__device__ __forceinline__ uint32_t shl_alu(uint32_t y) {
    uint32_t r;
    asm("shf.l.clamp.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(0u), "r"(y), "n"(k));
    return r;
}

// (t >> 4) | (y << 28): one funnel shift (SHF) that pushes y's low nibble in
// at the top of t.  Applied for j = 7, 6, ..., 0 it builds
// y0:y1:...:y7 (most significant first), Alg. 5's t = (t << 4) | (y_j & 15)
// chain for j = 0..7, in 8 ALU instructions instead of 7
// shifts + 7 merges; the 8 shifts flush t's initial bits.
__device__ __forceinline__ uint32_t push_nibble(uint32_t t, uint32_t y) {
    uint32_t r;
    asm("shf.r.clamp.b32 %0, %1, %2, 4;" : "=r"(r) : "r"(t), "r"(y));
    return r;
}

// bmsk: the low `n` bits set (n in 0..3 here), one BMSK instruction
__device__ __forceinline__ uint32_t low_mask(uint32_t n) {
    uint32_t m;
    asm("bmsk.clamp.b32 %0, 0, %1;" : "=r"(m) : "r"(n));
    return m;
}

// One squaring of instance j: instances in kFMask take the quotient from the
// FP32 pipe (fbarrett_sq), the others Barrett with IMAD.HI (barrett_sq);
// kFMask == kMontMask runs every instance in Montgomery form (mont_sq).
constexpr uint32_t kMontMask = 0x100;
template <uint32_t kFMask, int j>
__device__ __forceinline__ uint32_t sq(Bbs8 &b) {
    if constexpr (kFMask == kMontMask)
        b.y[j] = mont_sq(b.yh[j], b.nM[j], b.mu[j]);
    else if constexpr ((kFMask >> j) & 1u)
        b.y[j] = fbarrett_sq(b.y[j], b.nM[j], b.K[j], b.iF[j]);
    else
        b.y[j] = barrett_sq(b.y[j], b.nM[j], b.mu[j]);
    return b.y[j];
}

// One number's strategy word.  kPack: nibbles pushed in by one
// funnel shift each (push_nibble); otherwise the eight 4-bit fields are
// placed independently (y_j << (28 - 4j)) and merged by a 3-level LOP3 tree
// -- (hi & mask) | (lo & ~mask) -- same word, depth 3 instead of 8.
template <uint32_t kFMask, bool kPack>
__device__ __forceinline__ uint32_t v2_strategy(Bbs8 &b) {
    uint32_t t;
    if constexpr (kPack) {
        t = push_nibble(0u, sq<kFMask, 7>(b));
        t = push_nibble(t, sq<kFMask, 6>(b));
        t = push_nibble(t, sq<kFMask, 5>(b));
        t = push_nibble(t, sq<kFMask, 4>(b));
        t = push_nibble(t, sq<kFMask, 3>(b));
        t = push_nibble(t, sq<kFMask, 2>(b));
        t = push_nibble(t, sq<kFMask, 1>(b));
        t = push_nibble(t, sq<kFMask, 0>(b));
    } else {
        sq<kFMask, 0>(b), sq<kFMask, 1>(b), sq<kFMask, 2>(b), sq<kFMask, 3>(b);
        sq<kFMask, 4>(b), sq<kFMask, 5>(b), sq<kFMask, 6>(b), sq<kFMask, 7>(b);
        const uint32_t f0 = shl_alu<28>(b.y[0]), f1 = shl_alu<24>(b.y[1]), f2 = shl_alu<20>(b.y[2]);
        const uint32_t f3 = shl_alu<16>(b.y[3]), f4 = shl_alu<12>(b.y[4]), f5 = shl_alu<8>(b.y[5]);
        const uint32_t f6 = shl_alu<4>(b.y[6]), f7 = b.y[7];
        const uint32_t p01 = (f0 & 0xF0000000u) | (f1 & ~0xF0000000u);
        const uint32_t p23 = (f2 & 0xFFF00000u) | (f3 & ~0xFFF00000u);
        const uint32_t p45 = (f4 & 0xFFFFF000u) | (f5 & ~0xFFFFF000u);
        const uint32_t p67 = (f6 & 0xFFFFFFF0u) | (f7 & ~0xFFFFFFF0u);
        const uint32_t p03 = (p01 & 0xFF000000u) | (p23 & ~0xFF000000u);
        const uint32_t p47 = (p45 & 0xFFFFFF00u) | (p67 & ~0xFFFFFF00u);
        t = (p03 & 0xFFFF0000u) | (p47 & 0x0000FFFFu);
    }
    // two variable shifts with fillers: t <<= sh; t |= bbs & array_shift[sh]
    uint32_t sh = sq<kFMask, 2>(b) & 3u;
    t = (t << sh) | (sq<kFMask, 0>(b) & low_mask(sh));
    sh = sq<kFMask, 6>(b) & 3u;
    t = (t << sh) | (sq<kFMask, 1>(b) & low_mask(sh));
    return t;
}

// occupancy / CTA-shape knobs (experiments set them through CIPRNG_NVCC_EXTRA).
// Forcing 5 or 6 CTAs per SM (48 / 40 registers) spills and loses 5-8 %
// (profiles/experiments/s36_v2_occupancy.txt): V2 is heavy-FMA-pipe bound,
// not latency bound, at 32 resident warps per SM (64 registers).
#ifndef CIPRNG_V2_MINB
#define CIPRNG_V2_MINB 1
#endif
#ifndef CIPRNG_V2_WPB
#define CIPRNG_V2_WPB 4  // 4 warps per CTA: 2.82e11 vs 2.80e11 at 8 (profiles/experiments/s36)
#endif

// An explicit minimum of 1 CTA per SM is NOT the same as none (0): it lets
// ptxas spend registers freely -- 72 instead of 64 in the store kernel
// (2.80 vs 2.82e11 numbers/s), but 93 instead of 72 in the consumer, which
// is faster with them (2.99 vs 2.95e11; profiles/experiments/s43).  So the
// consumer instantiation asks for 1 and the others for none, unless a larger
// minimum is set for an experiment.
template <class Sink>
constexpr int v2_min_blocks() {
    return CIPRNG_V2_MINB > 1 ? CIPRNG_V2_MINB
                              : ((std::is_same<Sink, StatsSink>::value || Sink::kCtaHist) ? 1 : 0);
}
// Experiment CIPRNG_V2_HIST_CTA: the CTA-histogram consumer (sinks.cuh
// StatsSinkCta1), one CTA of kV2CtaWarps warps per SM sharing the 64 KiB
// conflict-free histogram (slower, see launch_v2).
#ifndef CIPRNG_V2C_CTA_WARPS
#define CIPRNG_V2C_CTA_WARPS 21
#endif
constexpr int kV2CtaWarps = CIPRNG_V2C_CTA_WARPS;
template <class Sink>
constexpr int v2_max_threads() {
    return Sink::kCtaHist ? 32 * kV2CtaWarps : 32 * CIPRNG_V2_WPB;
}

template <class Sink, uint32_t kFMask, bool kPack>
__global__ void __launch_bounds__(v2_max_threads<Sink>(), v2_min_blocks<Sink>()) v2_kernel(GenArgs a) {
    Sink sink(a);
    pdl_launch_dependents();
    pdl_wait();  // previous grid on the stream complete + visible
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t C = a.C;
    const uint32_t off = lane % C, gbase = lane - off;
    const uint64_t n_tiles = (a.s_count + 31) / 32;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    const StateIO sio(a);
    const uint4 *modtab = reinterpret_cast<const uint4 *>(a.mod);

    for (uint64_t tile = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); tile < n_tiles;
         tile += warps) {
        const uint64_t row = tile * 32 + lane;
        const bool valid = row < a.s_count;
        const uint64_t s = a.s_begin + row;
        Bbs8 b;
        // every lane loads (an invalid lane reads the tile's first row and
        // discards it): no branch between the 8 dependent state -> modulus loads
        const uint64_t sl = valid ? s : a.s_begin + tile * 32;
        uint32_t m[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            b.y[j] = sio.ld(j, sl);
            m[j] = sio.ld(8 + j, sl);
        }
        uint32_t x = sio.ld(16, sl), tp = sio.ld(17, sl);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if constexpr (kFMask == kMontMask) {
                const uint4 e = __ldg(modtab + 2 * m[j] + 1);  // {M, Mp, R2, 0} (api.cu)
                b.nM[j] = e.x;
                b.mu[j] = e.y;
                b.K[j] = e.z;
            } else {
                const uint4 e = __ldg(modtab + 2 * m[j]);  // {invMf, mu, 2^32 - M, K} (api.cu)
                b.iF[j] = e.x;
                b.mu[j] = e.y;
                b.nM[j] = e.z;
                b.K[j] = e.w;
            }
        }
        if (!valid) {
            // the CTA histogram needs an invalid lane to emit zeros: y = 0
            // squares to 0, so every nibble, shift and filler is 0 (its
            // combination group is all invalid: s_count % C == 0)
#pragma unroll
            for (int j = 0; j < 8; ++j) b.y[j] = Sink::kCtaHist ? 0u : 2u;
            x = tp = 0;
        }
        if constexpr (kFMask == kMontMask) {
#pragma unroll
            for (int j = 0; j < 8; ++j) b.yh[j] = mont_enter(b.y[j], b.nM[j], b.mu[j], b.K[j]);
        }
        const uint32_t src1 = gbase + a.comb.t[b.y[0] & 7u][off];
        const uint32_t src2 = gbase + a.comb.t[8u + (b.y[1] & 7u)][off];
        sink.begin_row(0, row);
        auto round = [&]() -> uint32_t {
            uint32_t t = v2_strategy<kFMask, kPack>(b);
            t ^= __shfl_sync(kFull, tp, src1) ^ __shfl_sync(kFull, tp, src2);
            tp = t;
            x ^= t;
            return x;
        };
        uint64_t i = 0;
        if constexpr (Sink::kStats) {
            // consumers: n < 2^24 (host-checked), 32-bit trip counter and index
            const uint32_t n4 = (uint32_t)a.n & ~3u;
            for (uint32_t i32 = 0; i32 != n4; i32 += 4) {
                uint32_t o0 = round(), o1 = round(), o2 = round(), o3 = round();
                sink.put4(0, i32, o0, o1, o2, o3, valid);
            }
            i = n4;
        } else {
            for (; i + 4 <= a.n; i += 4) {
                uint32_t o0 = round(), o1 = round(), o2 = round(), o3 = round();
                sink.put4(0, i, o0, o1, o2, o3, valid);
            }
        }
        for (; i < a.n; ++i) sink.put1(0, i, round(), valid);
        sink.end_rows(valid ? 1u : 0u);
        if (valid && a.n > 0) {
            // rotation (Q19): instance j moves to slot j+1 with its modulus
            // index, re-read from the untouched call-entry plane instead of
            // being held in 8 registers through the loop
#pragma unroll
            for (int j = 0; j < 8; ++j) m[j] = sio.ld(8 + j, s);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                sio.st((j + 1) & 7, s, b.y[j]);
                sio.st(8 + ((j + 1) & 7), s, m[j]);
            }
            sio.st(16, s, x);
            sio.st(17, s, tp);
        }
    }
    sink.finish(a);
}

// Exhaustive device-side check of both squarings (the FP32 rounding modes
// of fbarrett_sq are hardware behaviour the host emulation only models):
// one thread per (modulus, y < 2^16); y >= M threads idle.
__global__ void modsq_check_kernel(const uint32_t *mod, uint32_t n_mod, unsigned long long *bad) {
    const uint32_t e = blockIdx.y, y = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n_mod) return;
    const uint4 w = reinterpret_cast<const uint4 *>(mod)[2 * e];  // {invMf, mu, 2^32 - M, K}
    const uint32_t M = mod[kModWords * e + 4];
    if (y >= M) return;
    const uint32_t ref = (y * y) % M;
    const uint4 v = reinterpret_cast<const uint4 *>(mod)[2 * e + 1];  // {M, Mp, R2, 0}
    uint32_t yh = mont_enter(y, v.x, v.y, v.z);
    const uint32_t ym = mont_sq(yh, v.x, v.y);
    const uint32_t nb = (barrett_sq(y, w.z, w.y) != ref) + (fbarrett_sq(y, w.z, w.w, w.x) != ref) + (ym != ref);
    if (nb) atomicAdd(bad, (unsigned long long)nb);
}

int launch_modsq_check(const uint32_t *mod, uint32_t n_mod, unsigned long long *bad, cudaStream_t st) {
    modsq_check_kernel<<<dim3(65536 / 256, n_mod), 256, 0, st>>>(mod, n_mod, bad);
    return 1;
}

// Default squaring split and nibble packing, from B200 measurements
// (profiles/experiments/s33_v2_kinds.json, C3, L2 flushed): funnel-shift
// packing 2.79e11 numbers/s vs 2.59e11 for the LOP3 tree (-10 % issued
// instructions); moving 1-12 of the 12 squarings per number to the FP32
// quotient gives 2.79e11 down to 2.59e11 -- never faster: the freed heavy-pipe
// cycles are paid back in issue slots (7 instructions per squaring, not 4),
// so every squaring stays Barrett. `kind` (CIPRNG_V2_KIND,
// read at prng_create) selects another store-mode instantiation for experiments.
constexpr uint32_t kV2FMask = 0x00;
constexpr bool kV2Pack = true;

int launch_v2(const GenArgs &a, int mode, cudaStream_t st, int kind) {
    if (a.s_count == 0) return 0;
    const uint64_t tiles = (a.s_count + 31) / 32;
    const int wpb = CIPRNG_V2_WPB;
    uint64_t blocks = (tiles + wpb - 1) / wpb;
    if (mode == 2) {
        // The CTA histogram (StatsSinkCta1) measured SLOWER here than the
        // per-warp one (C5 shape, n = 1024: 2.54 / 2.84 / 2.94e11 at 21 / 24 /
        // 16 warps per CTA against 2.99e11; profiles/experiments/s63-s64) --
        // the heavy-pipe bound V2 consumer gains nothing from the freed IMAD
        // and loses ILP at the lower register budget.  Kept as an experiment.
#if defined(CIPRNG_V2_HIST_CTA)
        if (cta_hist_ok()) {
            static_assert(StatsSinkCta1::kResv == (uint32_t)kCtaHistResvBytes, "reserved shared memory");
            launch_cta_hist(v2_kernel<StatsSinkCta1, kV2FMask, kV2Pack>, kV2CtaWarps, StatsSinkCta1::kSmemBytesExtra,
                            tiles, a.n, st, a);
            return 1;
        }
#endif
        auto kern = v2_kernel<StatsSink, kV2FMask, kV2Pack>;
        const size_t sm = wpb * StatsSink::kSmemBytesPerWarp + StatsSink::kSmemBytesExtra;
        launch_k(kern, dim3(persistent_grid(kern, 32 * wpb, sm, blocks)), dim3(32 * wpb), sm, st, a);
    } else if (mode == 3) {
        auto kern = v2_kernel<BatterySink, kV2FMask, kV2Pack>;
        const size_t sm = wpb * BatterySink::kSmemBytesPerWarp + BatterySink::kSmemBytesExtra;
        launch_k(kern, dim3(persistent_grid(kern, 32 * wpb, sm, blocks)), dim3(32 * wpb), sm, st, a);
    } else {
        void (*kern)(GenArgs) = v2_kernel<StoreSink, kV2FMask, kV2Pack>;
        switch (kind) {
            case 0: kern = v2_kernel<StoreSink, 0x00, false>; break;
            case 1: kern = v2_kernel<StoreSink, 0x00, true>; break;
            case 2: kern = v2_kernel<StoreSink, 0x08, true>; break;   // 1 FP32-quotient squaring per number
            case 3: kern = v2_kernel<StoreSink, 0x01, true>; break;   // 2
            case 4: kern = v2_kernel<StoreSink, 0x09, true>; break;   // 3
            case 5: kern = v2_kernel<StoreSink, 0x03, true>; break;   // 4
            case 6: kern = v2_kernel<StoreSink, 0x0B, true>; break;   // 5
            case 7: kern = v2_kernel<StoreSink, 0x18, true>; break;   // 2 (two single-squared)
            case 8: kern = v2_kernel<StoreSink, 0x01, false>; break;  // 2, LOP3 tree
            case 9: kern = v2_kernel<StoreSink, 0xFF, true>; break;   // 12
            case 10: kern = v2_kernel<StoreSink, kMontMask, true>; break;  // all 12 in Montgomery form
            default: break;
        }
        launch_k(kern, dim3((int)blocks), dim3(32 * wpb), 0, st, a);
    }
    return 1;
}

}  // namespace ciprng
