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
__global__ void __launch_bounds__(256) digest_kernel(const uint32_t *__restrict__ out, uint64_t first_stream,
                                                     uint64_t total, uint64_t n, uint64_t *digest) {
    pdl_launch_dependents();
    pdl_wait();  // previous grid on the stream complete + visible
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t base = first_stream * n;  // global index of out[0]
    uint64_t acc = 0;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += stride)
        acc += splitmix_fin(splitmix_fin(base + k) ^ (uint64_t)out[k]);
#pragma unroll
    for (int d = 16; d; d >>= 1) acc += __shfl_xor_sync(kFull, acc, d);
    if ((threadIdx.x & 31u) == 0 && acc) atomicAdd(reinterpret_cast<unsigned long long *>(digest), (unsigned long long)acc);
}

int launch_digest(const uint32_t *out, uint64_t first_stream, uint64_t n_local, uint64_t n, uint64_t *digest,
                  cudaStream_t st, int grid) {
    const uint64_t total = n_local * n;
    if (total == 0) return 0;
    uint64_t blocks = (total + 255) / 256;
    if (blocks > (uint64_t)grid) blocks = grid;
    launch_k(digest_kernel, dim3((int)blocks), dim3(256), 0, st, out, first_stream, total, n, digest);
    return 1;
}

}  // namespace ciprng
