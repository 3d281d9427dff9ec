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
// Q28 (r2): the words of each stream's row are taken in pairs (x_2j, x_2j+1)
// -- a lone last word of an odd row is paired with 0 -- and
//   d = sum over pairs of mix64((x_2j+1 << 32 | x_2j) + P * G)  (mod 2^64),
// P = global stream * ceil(n / 2) + j the pair's global position, mix64 the
// SplitMix64 finaliser and G its increment: h is output number P of
// SplitMix64 seeded with the pair, so the mixer is pinned by the published
// SplitMix64 sequence.  For a fixed position h is a bijection of the pair
// (add and mix64 are invertible), so any wrong word changes the digest; rows
// are whole units, so shard digests add.  One finaliser per TWO words: ~9
// ALU ops per word, above HBM speed on 148 SMs (one finaliser per word ran
// at 3.6 TB/s, ALU bound; the r1 definition, two finalisers per word and
// scalar loads, at 1.36 TB/s).  P * G advances by G per pair: an add.
constexpr uint64_t kDigestG = 0x9E3779B97F4A7C15ull;

__device__ __forceinline__ uint64_t digest_pair(uint32_t lo, uint32_t hi, uint64_t pg) {
    return splitmix_fin(((uint64_t)hi << 32 | lo) + pg);
}

__device__ __forceinline__ uint4 ld_stream_v4(const uint32_t *p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ void digest_reduce(uint64_t acc, uint64_t *digest) {
#pragma unroll
    for (int d = 16; d; d >>= 1) acc += __shfl_xor_sync(kFull, acc, d);
    if ((threadIdx.x & 31u) == 0 && acc) atomicAdd(reinterpret_cast<unsigned long long *>(digest), (unsigned long long)acc);
}

// Fast path: n even and out 8-byte aligned, so the block is a flat array of
// pairs, pair k at global position first_stream * n/2 + k.  Thread t takes
// 16-byte chunks (two pairs) t, t + stride, ... (two chunks in flight); a
// head pair before the first 16-byte boundary and a tail pair go to thread 0.
__global__ void __launch_bounds__(256) digest_kernel(const uint32_t *__restrict__ out, uint64_t first_stream,
                                                     uint64_t total, uint64_t n, uint64_t *digest) {
    pdl_launch_dependents();
    pdl_wait();  // previous grid on the stream complete + visible
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t pairs = total >> 1;
    const uint64_t p0 = first_stream * (n >> 1);  // global position of pair 0
    const uint64_t head = (reinterpret_cast<uintptr_t>(out) & 8u) && pairs ? 1 : 0;
    const uint64_t chunks = (pairs - head) >> 1;
    const uint32_t *body = out + 2 * head;
    uint64_t acc = 0;
    uint64_t c = tid;
    for (; c + stride < chunks; c += 2 * stride) {
        const uint4 v0 = ld_stream_v4(body + 4 * c);
        const uint4 v1 = ld_stream_v4(body + 4 * (c + stride));
        const uint64_t g0 = (p0 + head + 2 * c) * kDigestG, g1 = (p0 + head + 2 * (c + stride)) * kDigestG;
        acc += digest_pair(v0.x, v0.y, g0);
        acc += digest_pair(v0.z, v0.w, g0 + kDigestG);
        acc += digest_pair(v1.x, v1.y, g1);
        acc += digest_pair(v1.z, v1.w, g1 + kDigestG);
    }
    if (c < chunks) {
        const uint4 v0 = ld_stream_v4(body + 4 * c);
        const uint64_t g0 = (p0 + head + 2 * c) * kDigestG;
        acc += digest_pair(v0.x, v0.y, g0);
        acc += digest_pair(v0.z, v0.w, g0 + kDigestG);
    }
    if (tid == 0) {
        if (head) acc += digest_pair(out[0], out[1], p0 * kDigestG);
        const uint64_t tl = head + 2 * chunks;  // at most one pair left
        if (tl < pairs) acc += digest_pair(out[2 * tl], out[2 * tl + 1], (p0 + tl) * kDigestG);
    }
    digest_reduce(acc, digest);
}

// General path (n odd, or out not 8-byte aligned): pair k = (row, j) by
// division, scalar loads; the lone last word of an odd row pairs with 0.
__global__ void __launch_bounds__(256) digest_general_kernel(const uint32_t *__restrict__ out, uint64_t first_stream,
                                                             uint64_t n_local, uint64_t n, uint64_t *digest) {
    pdl_launch_dependents();
    pdl_wait();
    const uint64_t hn = (n + 1) >> 1, pairs = n_local * hn;
    uint64_t acc = 0;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < pairs; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = k / hn, j = k - r * hn;
        const uint32_t *row = out + r * n;
        const uint32_t lo = row[2 * j], hi = 2 * j + 1 < n ? row[2 * j + 1] : 0u;
        acc += digest_pair(lo, hi, ((first_stream + r) * hn + j) * kDigestG);
    }
    digest_reduce(acc, digest);
}

int launch_digest(const uint32_t *out, uint64_t first_stream, uint64_t n_local, uint64_t n, uint64_t *digest,
                  cudaStream_t st, int grid) {
    const uint64_t total = n_local * n;
    if (total == 0) return 0;
    uint64_t blocks = (total / 8 + 255) / 256;  // two 16-byte chunks per thread per iteration
    if (blocks < 1) blocks = 1;
    if (blocks > (uint64_t)grid) blocks = grid;
    if (n % 2 == 0 && reinterpret_cast<uintptr_t>(out) % 8 == 0)
        launch_k(digest_kernel, dim3((int)blocks), dim3(256), 0, st, out, first_stream, total, n, digest);
    else
        launch_k(digest_general_kernel, dim3((int)blocks), dim3(256), 0, st, out, first_stream, n_local, n, digest);
    return 1;
}

}  // namespace ciprng
