// init_digest.cu -- a1 state initialisation (replaces the paper's host-side
// ISAAC seeding + host->device copy) and the
// verification digest (reading Q28).
//
// Seeder (Q11): W(seed, s, k) = SplitMix64 output 16 s + k + 1 from `seed`,
// computed on device, O(1) per stream, no H2D traffic, identical for any
// sharding of the stream space.
#include "device.cuh"
#include "kernels.h"

namespace ciprng {

__device__ __forceinline__ uint32_t gcd_u32(uint32_t a, uint32_t b) {
    while (b) {
        uint32_t t = a % b;
        a = b;
        b = t;
    }
    return a;
}

__global__ void __launch_bounds__(256) init_kernel(InitArgs a) {
    pdl_launch_dependents();
    pdl_wait();  // previous grid on the stream complete + visible
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint32_t *P = a.state;
    const uint64_t L = a.n_local;
    for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < L; r += stride) {
        const uint64_t s = a.first_stream + r;
        if (a.variant == 0) {
            uint64_t w[12];
            if (a.paper_defaults) {  // Listing 1: x = 123123123, Marsaglia seeds (Q12)
                const uint64_t def[12] = {88172645463325252ull, 123456789u, 362436069u, 521288629u,
                                          88675123u,            123456789u, 362436069u, 521288629u,
                                          88675123u,            5783321u,   6615241u,   123123123u};
                for (int k = 0; k < 12; ++k) w[k] = def[k];
            } else {
                for (int k = 0; k < 12; ++k) w[k] = seed_word(a.seed, s, k);
                if (w[0] == 0) w[0] = 88172645463325252ull;  // xorshift fixed point
                if ((w[1] | w[2] | w[3] | w[4]) == 0) {
                    w[1] = 123456789u; w[2] = 362436069u; w[3] = 521288629u; w[4] = 88675123u;
                }
                if ((w[5] | w[6] | w[7] | w[8] | w[9]) == 0) {
                    w[5] = 123456789u; w[6] = 362436069u; w[7] = 521288629u; w[8] = 88675123u; w[9] = 5783321u;
                }
            }
            for (int k = 0; k < 11; ++k) {
                P[(2 * k) * L + r] = (uint32_t)w[k];
                P[(2 * k + 1) * L + r] = (uint32_t)(w[k] >> 32);
            }
            P[22 * L + r] = (uint32_t)w[11];
        } else if (a.variant == 1) {
            uint32_t g[4];
            for (int k = 0; k < 4; ++k) g[k] = (uint32_t)seed_word(a.seed, s, k);
            if ((g[0] | g[1] | g[2] | g[3]) == 0) {
                g[0] = 123456789u; g[1] = 362436069u; g[2] = 521288629u; g[3] = 88675123u;
            }
            for (int k = 0; k < 4; ++k) P[k * L + r] = g[k];
            P[4 * L + r] = (uint32_t)seed_word(a.seed, s, 4);
            P[5 * L + r] = (uint32_t)seed_word(a.seed, s, 5);
        } else if (a.variant == 3) {
            // V3 (NEXT-1): xor64 a = W(s,0) (0 -> Marsaglia seed), x, tp
            uint64_t w0 = seed_word(a.seed, s, 0);
            if (w0 == 0) w0 = 88172645463325252ull;
            P[0 * L + r] = (uint32_t)w0;
            P[1 * L + r] = (uint32_t)(w0 >> 32);
            P[2 * L + r] = (uint32_t)seed_word(a.seed, s, 1);
            P[3 * L + r] = (uint32_t)seed_word(a.seed, s, 2);
        } else if (a.variant == 4) {
            // V4 (NEXT-1): V0's generator words, x = W(s,11), tp = W(s,12)
            uint64_t w[11];
            for (int k = 0; k < 11; ++k) w[k] = seed_word(a.seed, s, k);
            if (w[0] == 0) w[0] = 88172645463325252ull;
            if ((w[1] | w[2] | w[3] | w[4]) == 0) {
                w[1] = 123456789u; w[2] = 362436069u; w[3] = 521288629u; w[4] = 88675123u;
            }
            if ((w[5] | w[6] | w[7] | w[8] | w[9]) == 0) {
                w[5] = 123456789u; w[6] = 362436069u; w[7] = 521288629u; w[8] = 88675123u; w[9] = 5783321u;
            }
            for (int k = 0; k < 11; ++k) {
                P[(2 * k) * L + r] = (uint32_t)w[k];
                P[(2 * k + 1) * L + r] = (uint32_t)(w[k] >> 32);
            }
            P[22 * L + r] = (uint32_t)seed_word(a.seed, s, 11);
            P[23 * L + r] = (uint32_t)seed_word(a.seed, s, 12);
        } else {
            // Q21: y = r^2 mod M, gcd(r, M) = 1, y not in {0, 1}
            for (int j = 0; j < 8; ++j) {
                const uint64_t w = seed_word(a.seed, s, j);
                const uint32_t mi = (uint32_t)(w >> 32) % a.n_mod;
                const uint32_t M = a.mod[kModWords * mi + 4];
                uint32_t rr = 2u + (uint32_t)w % (M - 3u);
                while (gcd_u32(rr, M) != 1u || (rr * rr) % M <= 1u) rr = (rr == M - 2u) ? 2u : rr + 1u;
                P[j * L + r] = (rr * rr) % M;
                P[(8 + j) * L + r] = mi;
            }
            P[16 * L + r] = (uint32_t)seed_word(a.seed, s, 8);
            P[17 * L + r] = (uint32_t)seed_word(a.seed, s, 9);
        }
    }
}

int launch_init(const InitArgs &a, cudaStream_t st) {
    uint64_t blocks = (a.n_local + 255) / 256;
    if (blocks > 148u * 32u) blocks = 148u * 32u;
    launch_k(init_kernel, dim3((int)blocks), dim3(256), 0, st, a);
    return 1;
}

// ------------------------------------------------------------------ digest
// Q28 (r2): d = sum_idx h(idx, x_idx) mod 2^64 with idx = global s*n + i and
// h(idx, x) = m(idx * G + x), m(z) = { z ^= z >> 32; z *= K; z ^= z >> 32 }.
// h is a bijection of x for a fixed idx (add, xorshift, odd multiply are all
// invertible), so any single wrong word changes the digest.  Per word: one
// 64-bit multiply (3 IMAD) and about 8 ALU ops -- about 9 TB/s of ALU
// throughput on 148 SMs, above HBM, so the kernel streams at memory speed
// (the r1 definition, two SplitMix64 finalisers per word, ran at 1.36 TB/s).
// idx * G advances by G per word, so it is an add, not a multiply.
constexpr uint64_t kDigestG = 0x9E3779B97F4A7C15ull, kDigestK = 0xD6E8FEB86659FD93ull;

__device__ __forceinline__ uint64_t digest_mix(uint64_t z) {
    z ^= z >> 32;
    z *= kDigestK;
    return z ^ (z >> 32);
}

__device__ __forceinline__ uint4 ld_stream_v4(const uint32_t *p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

// Thread t of the grid takes 16-byte chunks t, t + stride, ... (two in
// flight per iteration); `head` scalar words before the first aligned chunk
// and the ragged tail go to the first threads.
__global__ void __launch_bounds__(256) digest_kernel(const uint32_t *__restrict__ out, uint64_t first_stream,
                                                     uint64_t total, uint64_t n, uint64_t *digest) {
    pdl_launch_dependents();
    pdl_wait();  // previous grid on the stream complete + visible
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t base = first_stream * n;  // global index of out[0]
    const uint32_t mis = (uint32_t)((reinterpret_cast<uintptr_t>(out) >> 2) & 3u);
    const uint64_t head = total < (uint64_t)((4u - mis) & 3u) ? total : (uint64_t)((4u - mis) & 3u);
    const uint64_t chunks = (total - head) >> 2;
    const uint32_t *body = out + head;
    uint64_t acc = 0;
    uint64_t c = tid;
    for (; c + stride < chunks; c += 2 * stride) {
        const uint4 v0 = ld_stream_v4(body + 4 * c);
        const uint4 v1 = ld_stream_v4(body + 4 * (c + stride));
        uint64_t g0 = (base + head + 4 * c) * kDigestG, g1 = (base + head + 4 * (c + stride)) * kDigestG;
        acc += digest_mix(g0 + v0.x); g0 += kDigestG;
        acc += digest_mix(g0 + v0.y); g0 += kDigestG;
        acc += digest_mix(g0 + v0.z); g0 += kDigestG;
        acc += digest_mix(g0 + v0.w);
        acc += digest_mix(g1 + v1.x); g1 += kDigestG;
        acc += digest_mix(g1 + v1.y); g1 += kDigestG;
        acc += digest_mix(g1 + v1.z); g1 += kDigestG;
        acc += digest_mix(g1 + v1.w);
    }
    if (c < chunks) {
        const uint4 v0 = ld_stream_v4(body + 4 * c);
        uint64_t g0 = (base + head + 4 * c) * kDigestG;
        acc += digest_mix(g0 + v0.x); g0 += kDigestG;
        acc += digest_mix(g0 + v0.y); g0 += kDigestG;
        acc += digest_mix(g0 + v0.z); g0 += kDigestG;
        acc += digest_mix(g0 + v0.w);
    }
    // head words [0, head) and tail words [head + 4 chunks, total): at most 6
    const uint64_t tail0 = head + 4 * chunks;
    if (tid < head) acc += digest_mix((base + tid) * kDigestG + out[tid]);
    if (tid < total - tail0) acc += digest_mix((base + tail0 + tid) * kDigestG + out[tail0 + tid]);
#pragma unroll
    for (int d = 16; d; d >>= 1) acc += __shfl_xor_sync(kFull, acc, d);
    if ((threadIdx.x & 31u) == 0 && acc) atomicAdd(reinterpret_cast<unsigned long long *>(digest), (unsigned long long)acc);
}

int launch_digest(const uint32_t *out, uint64_t first_stream, uint64_t n_local, uint64_t n, uint64_t *digest,
                  cudaStream_t st, int grid) {
    const uint64_t total = n_local * n;
    if (total == 0) return 0;
    uint64_t blocks = (total / 8 + 255) / 256;  // two 16-byte chunks per thread per iteration
    if (blocks < 1) blocks = 1;
    if (blocks > (uint64_t)grid) blocks = grid;
    launch_k(digest_kernel, dim3((int)blocks), dim3(256), 0, st, out, first_stream, total, n, digest);
    return 1;
}

}  // namespace ciprng
