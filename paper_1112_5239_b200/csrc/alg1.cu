// alg1.cu -- SURVEY s8(f) NEXT-4: Algorithm 1 "PRNG with chaotic functions"
// for many independent streams, and the iteration-graph
// checks behind Theorems 1 and 2.
//
// Reading Q34: cells i in [1, n] are bits i-1 of the n-bit configuration x;
// F_f(i, x) replaces bit i-1 of x by bit i-1 of f(x) (Def. 1);
// XORshift(m) = 1 + (xorshift32() mod m) with Alg. 2's generator,
// one state z per stream drawn in program order; k = b + XORshift(b) and the
// loop "for i = 0..k" runs k + 1 single-cell updates per output.  f == NULL
// is the vectorial negation (it "satisfies the hypotheses of both
// theorems"); otherwise a table of 2^n words (n <= 16) read through L1/L2.
//
// Gamma(f) check: reachability from and to vertex 0 by level-synchronous
// breadth-first search inside one CTA (2^n <= 65536 vertices, levels
// separated by __syncthreads), plus the in/out-degree balance that makes
// Theorem 2's Markov matrix doubly stochastic.
#include "device.cuh"
#include "kernels.h"

namespace ciprng {

__device__ __forceinline__ uint32_t xs32(uint32_t &z) {  // Alg. 2
    z ^= z << 13;
    z ^= z >> 17;
    z ^= z << 5;
    return z;
}

__device__ __forceinline__ uint32_t f_single(const uint32_t *f, uint32_t nmask, uint32_t i, uint32_t x) {
    const uint32_t fx = f ? __ldg(f + x) : ~x & nmask;
    const uint32_t bit = 1u << (i - 1u);
    return (x & ~bit) | (fx & bit);
}

// One thread per stream.  Outputs go out in 8-word chunks (two 16-byte
// stores = one full 32-byte sector) when the rows allow it: r1 stored one
// word per thread per output, rows n_out words apart, and ncu counted 110 MB
// of partial-sector read-modify-write DRAM reads per launch
// (profiles/r1zc_ncu_summary.md).  XORshift(n) for a power-of-two n (the
// common cell counts) is a mask instead of a division by a runtime n.
__global__ void __launch_bounds__(256) alg1_kernel(const uint32_t *f, uint32_t n, uint32_t b, uint32_t *zs,
                                                   uint32_t *xs, uint64_t n_streams, uint64_t n_out,
                                                   uint32_t *out) {
    pdl_launch_dependents();
    pdl_wait();
    const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_streams) return;
    const uint32_t nmask = n == 32 ? 0xFFFFFFFFu : (1u << n) - 1u;
    const bool n_pow2 = (n & (n - 1u)) == 0;
    uint32_t z = zs[s], x = xs[s];
    uint32_t *row = out + s * n_out;
    const bool vec8 = (n_out % 8 == 0) && (reinterpret_cast<uintptr_t>(out) % 32 == 0);
    auto next = [&]() {
        const uint32_t k = b + 1u + xs32(z) % b;
        for (uint32_t i = 0; i <= k; ++i) {
            const uint32_t r = xs32(z);
            const uint32_t cell = 1u + (n_pow2 ? (r & (n - 1u)) : r % n);
            x = f_single(f, nmask, cell, x);
        }
        return x;
    };
    uint64_t j = 0;
    if (vec8) {
        for (; j < n_out; j += 8) {
            uint32_t o[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) o[q] = next();
            st_v4(row + j, o[0], o[1], o[2], o[3]);
            st_v4(row + j + 4, o[4], o[5], o[6], o[7]);
        }
    }
    for (; j < n_out; ++j) row[j] = next();
    zs[s] = z;
    xs[s] = x;
}

// report[0] = #reachable from 0, [1] = #reaching 0, [2] = #unbalanced.
// scratch: 2^n bytes of visit marks (two passes).
__global__ void __launch_bounds__(1024) gamma_kernel(const uint32_t *f, uint32_t n, uint8_t *mark,
                                                     unsigned long long *report) {
    pdl_launch_dependents();
    pdl_wait();
    const uint32_t V = 1u << n, nmask = V - 1u;
    __shared__ int changed;
    __shared__ unsigned long long cnt;
    for (int dir = 0; dir < 2; ++dir) {
        // mark: 0 unvisited, 1 frontier of this level, 2 visited
        for (uint32_t v = threadIdx.x; v < V; v += blockDim.x) mark[v] = v == 0 ? 1 : 0;
        __syncthreads();
        for (;;) {
            if (threadIdx.x == 0) changed = 0;
            __syncthreads();
            // expand the frontier: new vertices get 3 (next frontier)
            for (uint32_t u = threadIdx.x; u < V; u += blockDim.x) {
                if (mark[u] != 1) continue;
                for (uint32_t i = 1; i <= n; ++i) {
                    if (dir == 0) {
                        const uint32_t w = f_single(f, nmask, i, u);
                        if (mark[w] == 0) {
                            mark[w] = 3;
                            changed = 1;
                        }
                    } else {
                        const uint32_t cand[2] = {u, u ^ (1u << (i - 1u))};
                        for (int c = 0; c < 2; ++c)
                            if (mark[cand[c]] == 0 && f_single(f, nmask, i, cand[c]) == u) {
                                mark[cand[c]] = 3;
                                changed = 1;
                            }
                    }
                }
            }
            __syncthreads();
            for (uint32_t v = threadIdx.x; v < V; v += blockDim.x) {
                if (mark[v] == 1) mark[v] = 2;
                else if (mark[v] == 3) mark[v] = 1;
            }
            __syncthreads();
            if (!changed) break;
            __syncthreads();
        }
        if (threadIdx.x == 0) cnt = 0;
        __syncthreads();
        unsigned long long local = 0;
        for (uint32_t v = threadIdx.x; v < V; v += blockDim.x) local += mark[v] != 0;
        atomicAdd(&cnt, local);
        __syncthreads();
        if (threadIdx.x == 0) report[dir] = cnt;
        __syncthreads();
    }
    // degree balance: out-degree counts cells i with F(i, v) != v; in-degree
    // counts predecessors p = v ^ bit(i-1) with F(i, p) == v
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    unsigned long long bad = 0;
    for (uint32_t v = threadIdx.x; v < V; v += blockDim.x) {
        uint32_t outd = 0, ind = 0;
        for (uint32_t i = 1; i <= n; ++i) {
            outd += f_single(f, nmask, i, v) != v;
            const uint32_t p = v ^ (1u << (i - 1u));
            ind += f_single(f, nmask, i, p) == v;
        }
        bad += outd != ind;
    }
    atomicAdd(&cnt, bad);
    __syncthreads();
    if (threadIdx.x == 0) report[2] = cnt;
}

int launch_alg1(const uint32_t *f, uint32_t n, uint32_t b, uint32_t *z, uint32_t *x, uint64_t n_streams,
                uint64_t n_out, uint32_t *out, cudaStream_t st) {
    if (n_streams == 0) return 0;
    launch_k(alg1_kernel, dim3((unsigned)((n_streams + 255) / 256)), dim3(256), 0, st, f, n, b, z, x, n_streams,
             n_out, out);
    return 1;
}

int launch_gamma(const uint32_t *f, uint32_t n, uint8_t *mark, unsigned long long *report, cudaStream_t st) {
    launch_k(gamma_kernel, dim3(1), dim3(1024), 0, st, f, n, mark, report);
    return 1;
}

}  // namespace ciprng
