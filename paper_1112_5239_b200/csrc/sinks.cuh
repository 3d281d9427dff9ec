// sinks.cuh -- what a kernel does with each emitted x (P:903 / P:976 /
// P:1285 "store the new PRNG in NewNb", or the fused consumer of
// P:1031-1033).  Every generator kernel is templated on one of these, so the
// state evolution is literally the same code in store and consume mode.
#pragma once

#include "device.cuh"

namespace ciprng {

// Direct store: out[row * n + i] (stream-major, reading Q9).  put4 is called
// with i % 4 == 0; when rows are 16-byte aligned (vec) it is one 128-bit
// STG per 4 rounds per stream, otherwise 4 scalar stores.
struct StoreSink {
    uint32_t *out;
    uint64_t n;
    bool vec, cs;       // cs: L2 evict-first (streaming) stores
    uint32_t *base[2];  // row start of each of the lane's (up to two) streams
    // Per-lane stores are 16-byte pieces of rows n*4 bytes apart: L2 must hold
    // each line until its other pieces arrive, so an evict-first hint here
    // forces partial-sector read-modify-writes (V1 direct: 293 MB of DRAM
    // reads per launch, profiles/experiments/s27) -- plain stores only.
    __device__ __forceinline__ explicit StoreSink(const GenArgs &a)
        : out(a.out), n(a.n), vec(a.vec != 0), cs(false) {}
    // slot: which of the lane's streams (the V1 fast kernel owns two)
    __device__ __forceinline__ void begin_row(int slot, uint64_t row) { base[slot] = out + row * n; }
    __device__ __forceinline__ void put4(int slot, uint64_t i, uint32_t o0, uint32_t o1, uint32_t o2,
                                         uint32_t o3, bool valid) {
        if (!valid) return;
        uint32_t *p = base[slot] + i;
        if (vec) {
            if (cs) st_v4_cs(p, o0, o1, o2, o3);
            else st_v4(p, o0, o1, o2, o3);
        } else {
            put1(slot, i, o0, true);
            put1(slot, i + 1, o1, true);
            put1(slot, i + 2, o2, true);
            put1(slot, i + 3, o3, true);
        }
    }
    __device__ __forceinline__ void put1(int slot, uint64_t i, uint32_t o, bool valid) {
        if (!valid) return;
        if (cs) __stcs(base[slot] + i, o);
        else base[slot][i] = o;
    }
    __device__ __forceinline__ void end_rows(uint32_t) {}
    __device__ __forceinline__ void finish(const GenArgs &) {}
    static constexpr int kSmemBytesPerWarp = 0;
    static constexpr int kSmemBytesExtra = 0;
    static constexpr bool kStats = false;
    static constexpr bool kCtaHist = false;
};

// Consumer statistics (reading Q24): per-warp 256-bin shared-memory
// histogram of x >> 24, per-lane count of Monte-Carlo pi pairs
// (x_{2k}, x_{2k+1}) OUTSIDE the quarter disc.  Flushed once per CTA into the
// caller's u64 stats[258] with global atomics (integer sums: order-free).
//
// Issue economy (the consumer is integer-issue bound, ncu r1c: ALU pipe 84 %):
//  * a pair is outside iff u^2 + v^2 carries out of 64 bits, so the test is
//    two IMAD.WIDE (FMA pipe) and a three-instruction carry chain whose last
//    add-with-carry IS the counter update (no compare, no select);
//  * the bin's byte offset (x >> 24) * 4 is one IMAD.HI plus one LOP3;
//  * pair counts are not counted per pair: end_rows() adds n/2 per valid row,
//    and inside = pairs - outside at the end.
// Flush a warp's 256-bin u32 shared histogram into u64 global counters and
// zero it (all 32 lanes call it together).  The sinks call it whenever the
// increments since the last flush could reach 2^31, so the u32 bins never
// wrap whatever the data.
__device__ __forceinline__ void warp_hist_flush(uint32_t hist, uint64_t *gdst) {
    __syncwarp();
    const uint32_t lane = threadIdx.x & 31u;
#pragma unroll
    for (uint32_t k = 0; k < 8; ++k) {
        const uint32_t addr = hist + 4u * (8u * lane + k);
        uint32_t v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
        if (v) {
            atomicAdd(reinterpret_cast<unsigned long long *>(gdst + 8u * lane + k), (unsigned long long)v);
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(0u) : "memory");
        }
    }
    __syncwarp();
}
constexpr uint64_t kHistFlushAt = 1ull << 31;
constexpr uint64_t kMaxRowsPerWarpTile = 64;  // the fast kernels' tile; others use 32

#if !defined(CIPRNG_PAIR_ADDCC)
// r2: v^2 + u^2 as ONE 64-bit multiply-add whose carry-out is the test --
// the mad.lo.cc / madc.hi.cc chain compiles to IMAD.WIDE.U32 RZ, Pc, v, v, U
// (carry into a predicate), and ptxas folds the counter updates of two pairs
// into one IADD3.X cnt, RZ, RZ, cnt, Pc0, Pc1: per pair 2 IMAD.WIDE + 0.5
// ALU instead of 2 IMAD.WIDE + 2.5 ALU (the add.cc form below).  Measured
// (C5 shape, L2 flushed, profiles/experiments/s50_pair.jsonl): V1 consumer
// 1.69 -> 1.81e12 numbers/s, V3 1.15 -> 1.20e12, V0 +1.5 %; V2 -1.3 % (its
// heavy pipe is the binding one), so gen_v2.cu keeps the add.cc form
// (CIPRNG_PAIR_ADDCC defined before this header).
__device__ __forceinline__ void count_outside(uint32_t &cnt, uint32_t u, uint32_t v) {
    asm("{\n\t"
        ".reg .u64 U;\n\t"
        ".reg .u32 ul, uh, d;\n\t"
        "mul.wide.u32 U, %1, %1;\n\t"
        "mov.b64 {ul, uh}, U;\n\t"
        "mad.lo.cc.u32 d, %2, %2, ul;\n\t"
        "madc.hi.cc.u32 d, %2, %2, uh;\n\t"
        "addc.u32 %0, %0, 0;\n\t"
        "}"
        : "+r"(cnt)
        : "r"(u), "r"(v));
}
#else
__device__ __forceinline__ void count_outside(uint32_t &cnt, uint32_t u, uint32_t v) {
    asm("{\n\t"
        ".reg .u64 U, V;\n\t"
        ".reg .u32 ul, uh, vl, vh, d;\n\t"
        "mul.wide.u32 U, %1, %1;\n\t"
        "mul.wide.u32 V, %2, %2;\n\t"
        "mov.b64 {ul, uh}, U;\n\t"
        "mov.b64 {vl, vh}, V;\n\t"
        "add.cc.u32 d, ul, vl;\n\t"
        "addc.cc.u32 d, uh, vh;\n\t"
        "addc.u32 %0, %0, 0;\n\t"
        "}"
        : "+r"(cnt)
        : "r"(u), "r"(v));
}
#endif
// The same with the counter's add-with-carry as zero*zero + cnt + CF
// (madc: IMAD.X on the FMA pipe instead of IADD3.X on the ALU pipe; `zero`
// is GenArgs::zero, a 0 the compiler cannot fold).  Experiment only
// (CIPRNG_EXP_MADC): 4 fewer ALU instructions per 16 numbers, but measured
// 3.7 % slower for V1 (1.61 vs 1.67e12), 1 % for V3
// (profiles/experiments/s39_consume_madc.jsonl).
__device__ __forceinline__ void count_outside_madc(uint32_t &cnt, uint32_t u, uint32_t v, uint32_t zero) {
    asm("{\n\t"
        ".reg .u64 U, V;\n\t"
        ".reg .u32 ul, uh, vl, vh, d;\n\t"
        "mul.wide.u32 U, %1, %1;\n\t"
        "mul.wide.u32 V, %2, %2;\n\t"
        "mov.b64 {ul, uh}, U;\n\t"
        "mov.b64 {vl, vh}, V;\n\t"
        "add.cc.u32 d, ul, vl;\n\t"
        "addc.cc.u32 d, uh, vh;\n\t"
        "madc.lo.u32 %0, %3, %3, %0;\n\t"
        "}"
        : "+r"(cnt)
        : "r"(u), "r"(v), "r"(zero));
}

struct StatsSink {
    uint32_t hist;       // shared address of this warp's 256 u32 bins
    uint32_t junk;       // shared address of the CTA's discard bins (invalid lanes)
    uint32_t out32;      // outside pairs since the last end_rows (< 2^31, host-checked n)
    uint64_t outside;    // this lane's outside pairs
    uint64_t pairs;      // this lane's valid pairs
    uint32_t pend[2];    // stashed even-round value for put1 tails, per stream slot
    uint64_t n;
    uint64_t pending;    // bin increments of this warp since its last flush (upper bound)
    uint64_t *gstats;
    uint32_t zero;       // GenArgs::zero (count_outside_madc)
    __device__ __forceinline__ explicit StatsSink(const GenArgs &a)
        : out32(0), outside(0), pairs(0), pend{0, 0}, n(a.n), pending(0), gstats(a.stats), zero(a.zero) {
        extern __shared__ __align__(1024) uint8_t smem_dyn[];
        uint32_t *all = reinterpret_cast<uint32_t *>(smem_dyn);
        for (uint32_t k = threadIdx.x; k < 256u * (blockDim.x >> 5); k += blockDim.x) all[k] = 0;
        __syncthreads();
        hist = smem_u32(all) + 1024u * (threadIdx.x >> 5);
        junk = smem_u32(all) + 1024u * (blockDim.x >> 5);  // kSmemBytesExtra, never read
    }
    // Invalid lanes (rows past s_count in a partial tile) run the same
    // instructions -- no branch around the consumer inside the round loop --
    // with their bins redirected to the discard area and their outside count
    // dropped by end_rows.  Bin address = base + (x >> 24) * 4: SHF + LEA.
    __device__ __forceinline__ void bin(uint32_t base, uint32_t o) {
        uint32_t addr;
#if defined(CIPRNG_EXP_BIN_HI)  // experiment: x >> 24 as IMAD.HI (FMA pipe) instead of SHF (ALU):
        // V1 -4 %, V3 -0.8 %, V0 +0.3 % (profiles/experiments/s40_consume_bin_hi.jsonl), off
        asm("{\n\t.reg .u32 b;\n\tmul.hi.u32 b, %1, 256;\n\tmad.lo.u32 %0, b, 4, %2;\n\t}" : "=r"(addr) : "r"(o), "r"(base));
#elif defined(CIPRNG_EXP_BIN_LEA)  // experiment: the scaled add as LEA (ALU) instead of IMAD (heavy FMA):
        // V1 1.840 -> 1.667e12, V3 -6 % (profiles/experiments/s54_consumer_pipes.jsonl), off
        addr = base + ((o >> 24) << 2);
#else
        asm("{\n\t.reg .u32 b;\n\tshr.u32 b, %1, 24;\n\tmad.lo.u32 %0, b, 4, %2;\n\t}" : "=r"(addr) : "r"(o), "r"(base));
#endif
#if defined(CIPRNG_EXP_NOHIST)  // experiment: consumer without the histogram
        (void)addr;
#elif defined(CIPRNG_EXP_HIST_LANE)  // experiment: conflict-free bins (bin = lane)
        asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(base + 4u * (threadIdx.x & 31u)) : "memory");
#else
        asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr) : "memory");
#endif
    }
    __device__ __forceinline__ void pair(uint32_t u, uint32_t v) {
#if defined(CIPRNG_EXP_MADC)
        count_outside_madc(out32, u, v, zero);
#else
        count_outside(out32, u, v);
#endif
    }
    __device__ __forceinline__ void begin_row(int, uint64_t) {}
    __device__ __forceinline__ void put4(int, uint64_t, uint32_t o0, uint32_t o1, uint32_t o2, uint32_t o3,
                                         bool valid) {
        const uint32_t base = valid ? hist : junk;
        bin(base, o0);
        bin(base, o1);
        bin(base, o2);
        bin(base, o3);
        pair(o0, o1);
        pair(o2, o3);
    }
    __device__ __forceinline__ void put1(int slot, uint64_t i, uint32_t o, bool valid) {
        bin(valid ? hist : junk, o);
        if (i & 1) pair(pend[slot], o);
        else pend[slot] = o;
    }
    // after the rounds of a tile: this lane owned `rows` valid streams (0 for
    // an invalid lane, whose outside count is discarded)
    __device__ __forceinline__ void end_rows(uint32_t rows) {
        outside += rows ? out32 : 0u;
        out32 = 0;
        pairs += (uint64_t)rows * (n >> 1);
        pending += kMaxRowsPerWarpTile * n;
        if (pending + kMaxRowsPerWarpTile * n >= kHistFlushAt) {  // warp-uniform
            warp_hist_flush(hist, gstats + 2);
            pending = 0;
        }
    }
    __device__ void finish(const GenArgs &a) {
        uint64_t v = pairs - outside, p = pairs;
#pragma unroll
        for (int d = 16; d; d >>= 1) {
            v += __shfl_xor_sync(kFull, v, d);
            p += __shfl_xor_sync(kFull, p, d);
        }
        extern __shared__ __align__(1024) uint8_t smem_dyn[];
        uint32_t *all = reinterpret_cast<uint32_t *>(smem_dyn);
        const uint32_t nw = blockDim.x >> 5;
        __syncthreads();
        // fold warp histograms, then one atomic per bin per CTA
        for (uint32_t b = threadIdx.x; b < 256u; b += blockDim.x) {
            uint64_t acc = 0;  // per-warp bins may each approach 2^31 before a flush
            for (uint32_t w = 0; w < nw; ++w) acc += all[256u * w + b];
            if (acc) atomicAdd(reinterpret_cast<unsigned long long *>(a.stats + 2 + b), (unsigned long long)acc);
        }
        if ((threadIdx.x & 31) == 0) {
            if (v) atomicAdd(reinterpret_cast<unsigned long long *>(a.stats + 0), (unsigned long long)v);
            if (p) atomicAdd(reinterpret_cast<unsigned long long *>(a.stats + 1), (unsigned long long)p);
        }
    }
    static constexpr int kSmemBytesPerWarp = 1024;
    static constexpr int kSmemBytesExtra = 1024;  // the discard bins
    static constexpr bool kStats = true;
    static constexpr bool kCtaHist = false;
};

// StatsSink with a PRIVATE histogram column per lane (experiment
// CIPRNG_V1_HIST_PRIV, V1 fast consumer only).  The shared histogram's random
// bins cost ~3.15 bank-conflicted wavefronts per ATOMS (ncu r2a: the
// L1/shared data pipe 72 % busy).  Here bin b of lane l is the 16-bit half
// (l & 1) of word b*16 + (l >> 1): lanes 2k, 2k+1 share bank k + 16 (b & 1),
// so an atomic is at most 2-way conflicted.  16 KiB per warp (fewer
// resident warps); the u16 halves are folded into u64 before they could
// carry into the neighbour half.  Measured (C5 shape, L2 flushed, parity
// green, profiles/experiments/s52_hist_priv.jsonl): 1.70e12 numbers/s at 1,
// 2 or 4 warps per CTA against 1.82e12 for the shared histogram -- the
// occupancy lost to 16 KiB per warp (<= 14 warps/SM vs 24) costs more than
// the bank conflicts saved.  Kept as the measured alternative, off.
struct StatsSinkLane {
    uint32_t col;        // shared address of this lane's column: warp base + (lane >> 1) * 4
    uint32_t inc;        // 1 (even lane) or 65536 (odd lane)
    uint32_t warp_base;  // shared address of the warp's 4096 words
    uint32_t cta_bins;   // shared address of the CTA's u64 bins[256]
    uint32_t out32;
    uint64_t outside, pairs;
    uint32_t pend[2];
    uint64_t n;
    uint64_t pending;  // increments of one lane's bin since the last fold (upper bound)
    static constexpr int kWordsPerWarp = 4096;
    __device__ __forceinline__ explicit StatsSinkLane(const GenArgs &a)
        : out32(0), outside(0), pairs(0), pend{0, 0}, n(a.n), pending(0) {
        extern __shared__ __align__(1024) uint8_t smem_dyn[];
        const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
        const uint32_t all = smem_u32(smem_dyn);
        cta_bins = all;  // 2 KiB of u64 bins first
        warp_base = all + 2048u + warp * (kWordsPerWarp * 4u);
        col = warp_base + (lane >> 1) * 4u;
        inc = (lane & 1u) ? 65536u : 1u;
        for (uint32_t k = lane; k < (uint32_t)kWordsPerWarp / 4u; k += 32u)
            asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(warp_base + 16u * k), "r"(0u) : "memory");
        uint64_t *cb = reinterpret_cast<uint64_t *>(smem_dyn);
        for (uint32_t b = threadIdx.x; b < 256u; b += blockDim.x) cb[b] = 0;
        __syncthreads();
    }
    __device__ __forceinline__ void bin(uint32_t add, uint32_t o) {
        asm volatile("{\n\t.reg .u32 b, a;\n\tshr.u32 b, %0, 24;\n\tmad.lo.u32 a, b, 64, %1;\n\t"
                     "red.shared.add.u32 [a], %2;\n\t}" ::"r"(o), "r"(col), "r"(add) : "memory");
    }
    __device__ __forceinline__ void pair(uint32_t u, uint32_t v) { count_outside(out32, u, v); }
    __device__ __forceinline__ void begin_row(int, uint64_t) {}
    __device__ __forceinline__ void put4(int, uint64_t, uint32_t o0, uint32_t o1, uint32_t o2, uint32_t o3,
                                         bool valid) {
        const uint32_t add = valid ? inc : 0u;
        bin(add, o0);
        bin(add, o1);
        bin(add, o2);
        bin(add, o3);
        pair(o0, o1);
        pair(o2, o3);
    }
    __device__ __forceinline__ void put1(int slot, uint64_t i, uint32_t o, bool valid) {
        bin(valid ? inc : 0u, o);
        if (i & 1) pair(pend[slot], o);
        else pend[slot] = o;
    }
    // fold the warp's 16 lane-pair columns into the CTA's u64 bins and zero
    // them (all 32 lanes together): lane l sums bins l, l + 32, ...
    __device__ __forceinline__ void fold() {
        __syncwarp();
        const uint32_t lane = threadIdx.x & 31u;
#pragma unroll 1
        for (uint32_t b = lane; b < 256u; b += 32u) {
            uint32_t lo = 0, hi = 0;
#pragma unroll
            for (uint32_t k = 0; k < 16u; k += 4u) {
                uint32_t v0, v1, v2, v3;
                const uint32_t addr = warp_base + (b * 16u + k) * 4u;
                asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3)
                             : "r"(addr));
                asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(addr), "r"(0u) : "memory");
                lo += (v0 & 0xFFFFu) + (v1 & 0xFFFFu) + (v2 & 0xFFFFu) + (v3 & 0xFFFFu);
                hi += (v0 >> 16) + (v1 >> 16) + (v2 >> 16) + (v3 >> 16);
            }
            const uint64_t tot = (uint64_t)lo + hi;
            if (tot) asm volatile("red.shared.add.u64 [%0], %1;" ::"r"(cta_bins + 8u * b), "l"(tot) : "memory");
        }
        __syncwarp();
    }
    __device__ __forceinline__ void end_rows(uint32_t rows) {
        outside += rows ? out32 : 0u;
        out32 = 0;
        pairs += (uint64_t)rows * (n >> 1);
        pending += 2 * n;                  // a lane adds at most 2 per round to one bin
        if (pending + 2 * n >= 65536u) {  // warp-uniform
            fold();
            pending = 0;
        }
    }
    __device__ void finish(const GenArgs &a) {
        uint64_t v = pairs - outside, p = pairs;
#pragma unroll
        for (int d = 16; d; d >>= 1) {
            v += __shfl_xor_sync(kFull, v, d);
            p += __shfl_xor_sync(kFull, p, d);
        }
        fold();
        __syncthreads();
        extern __shared__ __align__(1024) uint8_t smem_dyn[];
        const uint64_t *cb = reinterpret_cast<const uint64_t *>(smem_dyn);
        for (uint32_t b = threadIdx.x; b < 256u; b += blockDim.x)
            if (cb[b]) atomicAdd(reinterpret_cast<unsigned long long *>(a.stats + 2 + b), (unsigned long long)cb[b]);
        if ((threadIdx.x & 31) == 0) {
            if (v) atomicAdd(reinterpret_cast<unsigned long long *>(a.stats + 0), (unsigned long long)v);
            if (p) atomicAdd(reinterpret_cast<unsigned long long *>(a.stats + 1), (unsigned long long)p);
        }
    }
    static constexpr int kSmemBytesPerWarp = kWordsPerWarp * 4;
    static constexpr int kSmemBytesExtra = 2048;
    static constexpr bool kStats = true;
    static constexpr bool kCtaHist = false;
};

// StatsSink with ONE histogram per CTA laid out so that a warp's atomics never
// share a bank: bin b of column c is the u32 at byte offset 256 b + 4 c of a
// 64 KiB block, c = lane (the lane's first stream) or 32 + lane (its second).
// Bank = c mod 32 = lane, so every red.shared is one conflict-free wavefront
// (StatsSink: ~3.15), and the offset is ONE byte permute -- PRMT puts x's top
// byte into byte 1 of the lane's column word -- against SHF + IMAD, with the
// CTA base folded into the atomic's uniform-register operand by ptxas.  All
// warps of the CTA share the block (same-address atomics from different
// instructions are still atomic).  No in-kernel flush: the host sizes the
// grid so that no word can reach 2^31 increments (v1_cta_hist_grid).
// kLaneStreams: streams per lane of the kernel using it (2: the V1 / V3 fast
// kernels' lanes own rows j and j + 16; 1: one stream per lane, V2)
template <int kLaneStreams>
struct StatsSinkCtaT {
    uint32_t cols;   // byte 0: 4 * lane, byte 2: 4 * (32 + lane), byte 3: the
                     // window address' CTA-in-cluster byte; byte 1 zero
    uint32_t out32;  // outside pairs since the last end_rows
    uint64_t outside, pairs;
    uint64_t junk;   // bin-0 increments of this lane's invalid rows (see end_rows)
    uint32_t pend[2];
    uint64_t n;
    static constexpr uint32_t kBytes = 65536;
    // Dynamic shared memory starts kResv bytes into the CTA's shared window
    // (the 1 KiB reserved by the driver, cudaDevAttrReservedSharedMemoryPerBlock;
    // the host checks it before choosing this sink, the ctor traps otherwise),
    // so the block's address is (cta byte << 24) | kResv and the atomic takes
    // kResv as its immediate offset: PRMT + ATOMS [R + 0x400], nothing else.
    static constexpr uint32_t kResv = 1024;
    static __device__ __forceinline__ uint32_t base() {
        extern __shared__ __align__(1024) uint8_t smem_dyn[];
        return smem_u32(smem_dyn);
    }
    __device__ __forceinline__ explicit StatsSinkCtaT(const GenArgs &a)
        : out32(0), outside(0), pairs(0), junk(0), pend{0, 0}, n(a.n) {
        zero = a.zero;
        const uint32_t lane = threadIdx.x & 31u, b = base();
        if ((b & 0x00FFFFFFu) != kResv) __trap();
        cols = (4u * lane) | ((128u + 4u * lane) << 16) | (b & 0xFF000000u);
        for (uint32_t k = threadIdx.x; k < kBytes / 16u; k += blockDim.x)
            asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(b + 16u * k), "r"(0u) : "memory");
        __syncthreads();
    }
    // Invalid lanes (rows past s_count: a half-warp of the fast kernels, whole
    // combination groups of V2) run the same instructions with an all-zero
    // state, so every number they emit is 0: they add exactly n per stream
    // slot to bin 0 per tile, which end_rows books and finish takes back -- no
    // predicate or branch in the round loop.
#ifndef CIPRNG_CTA_BIN_HI  // experiment: this many of the two slots form the offset on the heavy pipe
#define CIPRNG_CTA_BIN_HI 0   // (IMAD.HI x >> 24, IMAD bin * 256 + column) instead of one PRMT
#endif
    template <int kSlot>
    __device__ __forceinline__ void bin(uint32_t o) {
        uint32_t off;  // {column byte, x >> 24, 0, CTA byte}
        if constexpr (kSlot < CIPRNG_CTA_BIN_HI) {
            const uint32_t col = kSlot == 0 ? (cols & 0xFF0000FFu) : ((cols >> 16) & 0xFFu) | (cols & 0xFF000000u);
            asm("{\n\t.reg .u32 b;\n\tmul.hi.u32 b, %1, 256;\n\tmad.lo.u32 %0, b, 256, %2;\n\t}"
                : "=r"(off) : "r"(o), "r"(col));
        } else if constexpr (kSlot == 0) asm("prmt.b32 %0, %1, %2, 0x7534;" : "=r"(off) : "r"(o), "r"(cols));
        else asm("prmt.b32 %0, %1, %2, 0x7536;" : "=r"(off) : "r"(o), "r"(cols));
        asm volatile("red.shared.add.u32 [%0+1024], 1;" ::"r"(off) : "memory");
    }
    uint32_t zero = 0;  // GenArgs::zero (experiment CIPRNG_EXP_CTA_MADC)
    __device__ __forceinline__ void pair(uint32_t u, uint32_t v) {
#if defined(CIPRNG_EXP_CTA_MADC)  // the counter's add-with-carry on the heavy pipe (IMAD.X)
        count_outside_madc(out32, u, v, zero);
#else
        count_outside(out32, u, v);
#endif
    }
    __device__ __forceinline__ void begin_row(int, uint64_t) {}
    __device__ __forceinline__ void put4(int slot, uint64_t, uint32_t o0, uint32_t o1, uint32_t o2, uint32_t o3,
                                         bool) {
        if (slot == 0) {
            bin<0>(o0); bin<0>(o1); bin<0>(o2); bin<0>(o3);
        } else {
            bin<1>(o0); bin<1>(o1); bin<1>(o2); bin<1>(o3);
        }
        pair(o0, o1);
        pair(o2, o3);
    }
    __device__ __forceinline__ void put1(int slot, uint64_t i, uint32_t o, bool) {
        if (slot == 0) bin<0>(o);
        else bin<1>(o);
        if (i & 1) pair(pend[slot], o);
        else pend[slot] = o;
    }
    // rows: kLaneStreams for a valid lane, 0 for an invalid one
    __device__ __forceinline__ void end_rows(uint32_t rows) {
        outside += rows ? out32 : 0u;
        junk += rows ? 0u : (uint64_t)kLaneStreams * n;
        out32 = 0;
        pairs += (uint64_t)rows * (n >> 1);
    }
    __device__ void finish(const GenArgs &a) {
        uint64_t v = pairs - outside, p = pairs, jk = junk;
#pragma unroll
        for (int d = 16; d; d >>= 1) {
            v += __shfl_xor_sync(kFull, v, d);
            p += __shfl_xor_sync(kFull, p, d);
            jk += __shfl_xor_sync(kFull, jk, d);
        }
        __syncthreads();
        // bin b = sum of its 64 columns; thread b starts at column b (mod 64)
        // so a warp's 32 loads of one step fall in 32 different banks
        for (uint32_t b = threadIdx.x; b < 256u; b += blockDim.x) {
            uint64_t acc = 0;
#pragma unroll 8
            for (uint32_t c = 0; c < 64u; ++c) {
                uint32_t w;
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w) : "r"(base() + 256u * b + 4u * ((c + b) & 63u)));
                acc += w;
            }
            if (acc) atomicAdd(reinterpret_cast<unsigned long long *>(a.stats + 2 + b), (unsigned long long)acc);
        }
        if ((threadIdx.x & 31) == 0) {
            if (v) atomicAdd(reinterpret_cast<unsigned long long *>(a.stats + 0), (unsigned long long)v);
            if (p) atomicAdd(reinterpret_cast<unsigned long long *>(a.stats + 1), (unsigned long long)p);
            // the invalid rows' zeros (u64 wrap-around subtraction: the CTA's
            // own bin-0 total above already holds them)
            if (jk) atomicAdd(reinterpret_cast<unsigned long long *>(a.stats + 2), (unsigned long long)(0ull - jk));
        }
    }
    static constexpr int kSmemBytesPerWarp = 0;
    static constexpr int kSmemBytesExtra = kBytes;
    static constexpr bool kStats = true;
    static constexpr bool kCtaHist = true;
    // CTA shape of the kernels that use it: kWarps warps, kMinBlocks CTAs per
    // SM (2 x 64 KiB of histogram; 2 x 14 warps at <= 72 registers).  28 warps
    // per SM also divide the C5 shard evenly: 2^14 tiles over 148 x 28 warps
    // = 3.95 tiles per warp (32 warps: 3.46 -> 4 rounds, 13 % idle).
#ifndef CIPRNG_V1C_CTA_WARPS
#define CIPRNG_V1C_CTA_WARPS 14
#endif
#ifndef CIPRNG_V1C_CTA_MINB
#define CIPRNG_V1C_CTA_MINB 2
#endif
    static constexpr int kWarps = CIPRNG_V1C_CTA_WARPS;
    static constexpr int kMinBlocks = CIPRNG_V1C_CTA_MINB;
};
using StatsSinkCta = StatsSinkCtaT<2>;
using StatsSinkCta1 = StatsSinkCtaT<1>;

// Statistical battery counts (reading
// Q31: a stream's bit sequence within one call is its words in round order,
// each most significant bit first).  Same state evolution as StatsSink; per
// word the lane adds into u32 tile accumulators (folded into u64 by
// end_rows; the host caps n < 2^20 so they cannot wrap):
//   ones, adjacent differing pairs, adjacent 11 pairs, pairs 8 apart that
//   differ (the cross-word terms use the previous word of the same stream),
//   sum over 4-word blocks of (ones - 64)^2; the first / last bit of each
//   stream; and a per-warp shared histogram of all four bytes of every word.
// stats layout (264 u64): [0] ones [1] diff [2] c11 [3] lag8 [4] block_sq
// [5] blocks [6] first ones [7] last ones [8 + b] byte b.
// kCta = false: per-warp 256-bin histograms (3.15 bank-conflicted wavefronts
// per atomic; the L1/shared data pipe binds, ncu r2e 0.81).  kCta = true: the
// conflict-free CTA layout of StatsSinkCta (byte k of x lands in byte 1 of the
// lane's column word by one PRMT, selector 0x75k4 / 0x75k6), no in-kernel
// flush (the host sizes the grid for 4 increments per word, launch_cta_hist).
template <bool kCta>
struct BatterySinkT {
    static constexpr int kWords = 264;
    uint32_t hist;           // per-warp: shared address of this warp's 256 u32 bins; CTA: the column word
    uint32_t ones, diff, c11, lag8, bsq;
    uint64_t acc[8];
    uint32_t prev[2];
    uint64_t n;
    uint64_t pending;
    uint64_t *gstats;
    __device__ __forceinline__ explicit BatterySinkT(const GenArgs &a)
        : ones(0), diff(0), c11(0), lag8(0), bsq(0), acc{0, 0, 0, 0, 0, 0, 0, 0}, prev{0, 0}, n(a.n), pending(0),
          gstats(a.stats) {
        extern __shared__ __align__(1024) uint8_t smem_dyn[];
        if constexpr (kCta) {
            const uint32_t lane = threadIdx.x & 31u, b = StatsSinkCta::base();
            if ((b & 0x00FFFFFFu) != StatsSinkCta::kResv) __trap();
            hist = (4u * lane) | ((128u + 4u * lane) << 16) | (b & 0xFF000000u);
            for (uint32_t k = threadIdx.x; k < StatsSinkCta::kBytes / 16u; k += blockDim.x)
                asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(b + 16u * k), "r"(0u) : "memory");
        } else {
            uint32_t *all = reinterpret_cast<uint32_t *>(smem_dyn);
            for (uint32_t k = threadIdx.x; k < 256u * (blockDim.x >> 5); k += blockDim.x) all[k] = 0;
            hist = smem_u32(all) + 1024u * (threadIdx.x >> 5);
        }
        __syncthreads();
    }
    // byte kByte of x into the histogram (slot: the lane's stream, CTA layout only)
    template <int kByte>
    __device__ __forceinline__ void bin(int slot, uint32_t x) {
        if constexpr (kCta) {
            constexpr uint32_t selA = 0x7504u | (kByte << 4), selB = 0x7506u | (kByte << 4);
            uint32_t off;
            if (slot == 0) asm("prmt.b32 %0, %1, %2, %3;" : "=r"(off) : "r"(x), "r"(hist), "n"(selA));
            else asm("prmt.b32 %0, %1, %2, %3;" : "=r"(off) : "r"(x), "r"(hist), "n"(selB));
            asm volatile("red.shared.add.u32 [%0+1024], 1;" ::"r"(off) : "memory");
        } else {
            const uint32_t b = kByte == 3 ? (x >> 24) : ((x >> (8 * kByte)) & 0xFFu);
            asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(hist + 4u * b) : "memory");
        }
    }
    // one word x of a stream whose previous word in this call is p (has_prev)
    __device__ __forceinline__ void word(int slot, uint32_t x, uint32_t p, bool has_prev) {
        ones += __popc(x);
        diff += __popc((x ^ (x >> 1)) & 0x7FFFFFFFu);
        c11 += __popc(x & (x >> 1));
        lag8 += __popc((x ^ (x >> 8)) & 0x00FFFFFFu);
        if (has_prev) {
            diff += (p ^ (x >> 31)) & 1u;
            c11 += p & (x >> 31) & 1u;
            lag8 += __popc((p ^ (x >> 24)) & 0xFFu);
        }
        bin<0>(slot, x);
        bin<1>(slot, x);
        bin<2>(slot, x);
        bin<3>(slot, x);
    }
    __device__ __forceinline__ void begin_row(int, uint64_t) {}
    __device__ __forceinline__ void put4(int slot, uint64_t i, uint32_t o0, uint32_t o1, uint32_t o2, uint32_t o3,
                                         bool valid) {
        if (!valid) return;
        if (i == 0) acc[6] += o0 >> 31;
        word(slot, o0, prev[slot], i != 0);
        word(slot, o1, o0, true);
        word(slot, o2, o1, true);
        word(slot, o3, o2, true);
        const int c = (int)(__popc(o0) + __popc(o1) + __popc(o2) + __popc(o3)) - 64;
        bsq += (uint32_t)(c * c);
        prev[slot] = o3;
    }
    __device__ __forceinline__ void put1(int slot, uint64_t i, uint32_t o, bool valid) {
        if (!valid) return;
        if (i == 0) acc[6] += o >> 31;
        word(slot, o, prev[slot], i != 0);
        prev[slot] = o;
    }
    __device__ __forceinline__ void end_rows(uint32_t rows) {
        acc[0] += ones; acc[1] += diff; acc[2] += c11; acc[3] += lag8; acc[4] += bsq;
        ones = diff = c11 = lag8 = bsq = 0;
        acc[5] += (uint64_t)rows * (n >> 2);
        if (rows >= 1) acc[7] += prev[0] & 1u;
        if (rows >= 2) acc[7] += prev[1] & 1u;
        if constexpr (!kCta) {
            pending += 4 * kMaxRowsPerWarpTile * n;
            if (pending + 4 * kMaxRowsPerWarpTile * n >= kHistFlushAt) {  // warp-uniform
                warp_hist_flush(hist, gstats + 8);
                pending = 0;
            }
        }
    }
    __device__ void finish(const GenArgs &a) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            uint64_t v = acc[k];
#pragma unroll
            for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(kFull, v, d);
            acc[k] = v;
        }
        extern __shared__ __align__(1024) uint8_t smem_dyn[];
        uint32_t *all = reinterpret_cast<uint32_t *>(smem_dyn);
        const uint32_t nw = blockDim.x >> 5;
        __syncthreads();
        for (uint32_t b = threadIdx.x; b < 256u; b += blockDim.x) {
            uint64_t s = 0;
            if constexpr (kCta) {
#pragma unroll 8
                for (uint32_t c = 0; c < 64u; ++c) s += all[64u * b + ((c + b) & 63u)];
            } else {
                for (uint32_t w = 0; w < nw; ++w) s += all[256u * w + b];
            }
            if (s) atomicAdd(reinterpret_cast<unsigned long long *>(a.stats + 8 + b), (unsigned long long)s);
        }
        if ((threadIdx.x & 31) == 0) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (acc[k]) atomicAdd(reinterpret_cast<unsigned long long *>(a.stats + k), (unsigned long long)acc[k]);
        }
    }
    static constexpr int kSmemBytesPerWarp = kCta ? 0 : 1024;
    static constexpr int kSmemBytesExtra = kCta ? (int)StatsSinkCta::kBytes : 0;
    static constexpr bool kStats = true;
    static constexpr bool kCtaHist = kCta;
    // CTA shape with the CTA histogram: ONE CTA of 28 warps per SM (72
    // registers) -- 6.61 vs 6.40e11 numbers/s for 2 x 14 (profiles/experiments/s80)
#ifndef CIPRNG_BATTERY_CTA_WARPS
#define CIPRNG_BATTERY_CTA_WARPS 28
#endif
    static constexpr int kWarps = CIPRNG_BATTERY_CTA_WARPS;
    static constexpr int kMinBlocks = 1;
};
using BatterySink = BatterySinkT<false>;
using BatterySinkCta = BatterySinkT<true>;

// CTA shape of a CTA-histogram sink (0 for the others), for launch bounds
template <class Sink>
constexpr int cta_hist_warps() {
    if constexpr (Sink::kCtaHist) return Sink::kWarps;
    else return 0;
}
template <class Sink>
constexpr int cta_hist_min_blocks() {
    if constexpr (Sink::kCtaHist) return Sink::kMinBlocks;
    else return 0;
}

}  // namespace ciprng
