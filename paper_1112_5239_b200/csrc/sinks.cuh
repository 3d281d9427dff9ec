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
    bool vec;
    uint32_t *base[2];  // row start of each of the lane's (up to two) streams
    __device__ __forceinline__ explicit StoreSink(const GenArgs &a) : out(a.out), n(a.n), vec(a.vec != 0) {}
    // slot: which of the lane's streams (the V1 fast kernel owns two)
    __device__ __forceinline__ void begin_row(int slot, uint64_t row) { base[slot] = out + row * n; }
    __device__ __forceinline__ void put4(int slot, uint64_t i, uint32_t o0, uint32_t o1, uint32_t o2,
                                         uint32_t o3, bool valid) {
        if (!valid) return;
        uint32_t *p = base[slot] + i;
        if (vec) {
            st_v4(p, o0, o1, o2, o3);
        } else {
            p[0] = o0;
            p[1] = o1;
            p[2] = o2;
            p[3] = o3;
        }
    }
    __device__ __forceinline__ void put1(int slot, uint64_t i, uint32_t o, bool valid) {
        if (valid) base[slot][i] = o;
    }
    __device__ __forceinline__ void finish(const GenArgs &) {}
    static constexpr int kSmemBytesPerWarp = 0;
    static constexpr bool kStats = false;
};

// Consumer statistics (reading Q24): per-warp 256-bin shared-memory
// histogram of x >> 24, per-lane count of Monte-Carlo pi pairs
// (x_{2k}, x_{2k+1}) inside the quarter disc.  Flushed once per CTA into the
// caller's u64 stats[258] with global atomics (integer sums: order-free).
struct StatsSink {
    uint32_t *hist;      // this warp's 256 bins
    uint64_t inside;     // this lane's count
    uint32_t inside32;   // fast accumulator, folded into `inside`
    uint32_t pend[2];    // stashed even-round value for put1 tails, per stream slot
    uint64_t pairs;      // valid pairs seen by this lane
    uint64_t n;
    __device__ __forceinline__ explicit StatsSink(const GenArgs &a)
        : inside(0), inside32(0), pend{0, 0}, pairs(0), n(a.n) {
        extern __shared__ __align__(1024) uint8_t smem_dyn[];
        uint32_t *all = reinterpret_cast<uint32_t *>(smem_dyn);
        for (uint32_t k = threadIdx.x; k < 256u * (blockDim.x >> 5); k += blockDim.x) all[k] = 0;
        __syncthreads();
        hist = all + 256u * (threadIdx.x >> 5);
    }
    __device__ __forceinline__ void begin_row(int, uint64_t) {}
    __device__ __forceinline__ void put4(int, uint64_t, uint32_t o0, uint32_t o1, uint32_t o2, uint32_t o3,
                                         bool valid) {
        if (!valid) return;
        atomicAdd(&hist[o0 >> 24], 1u);
        atomicAdd(&hist[o1 >> 24], 1u);
        atomicAdd(&hist[o2 >> 24], 1u);
        atomicAdd(&hist[o3 >> 24], 1u);
        inside32 += pi_inside(o0, o1) + pi_inside(o2, o3);
        pairs += 2;
        if (inside32 >= 0x80000000u) { inside += inside32; inside32 = 0; }
    }
    __device__ __forceinline__ void put1(int slot, uint64_t i, uint32_t o, bool valid) {
        if (!valid) return;
        atomicAdd(&hist[o >> 24], 1u);
        if (i & 1) {
            inside32 += pi_inside(pend[slot], o);
            pairs += 1;
        } else {
            pend[slot] = o;
        }
    }
    __device__ void finish(const GenArgs &a) {
        uint64_t v = inside + inside32, p = pairs;
#pragma unroll
        for (int d = 16; d; d >>= 1) {
            v += __shfl_xor_sync(kFull, v, d);
            p += __shfl_xor_sync(kFull, p, d);
        }
        extern __shared__ __align__(1024) uint8_t smem_dyn[];
        uint32_t *all = reinterpret_cast<uint32_t *>(smem_dyn);
        const uint32_t nw = blockDim.x >> 5;
        __syncthreads();
        // fold warp histograms into warp 0's copy, then one atomic per bin
        for (uint32_t b = threadIdx.x; b < 256u; b += blockDim.x) {
            uint32_t acc = 0;
            for (uint32_t w = 0; w < nw; ++w) acc += all[256u * w + b];
            if (acc) atomicAdd(reinterpret_cast<unsigned long long *>(a.stats + 2 + b), (unsigned long long)acc);
        }
        if ((threadIdx.x & 31) == 0) {
            if (v) atomicAdd(reinterpret_cast<unsigned long long *>(a.stats + 0), (unsigned long long)v);
            if (p) atomicAdd(reinterpret_cast<unsigned long long *>(a.stats + 1), (unsigned long long)p);
        }
    }
    static constexpr int kSmemBytesPerWarp = 1024;
    static constexpr bool kStats = true;
};

}  // namespace ciprng
