// v0_jump.cu -- one V0 stream split across the whole GPU (BASELINE configs[0],
// "1 stream, fixed seed, 10^6 outputs").
//
// Listing 1 is one sequential chain per stream: on a GPU a single
// stream runs on one thread at ~20 M numbers/s (r1's C1 row).  But every
// generator of Listing 1 is linear over GF(2) -- xor64, xor128 and xorwow's
// shift register are xorshift recurrences; xorwow's Weyl counter d advances
// by a constant -- and the chaotic-iteration state is a prefix XOR,
// x_k = x_0 ^ f_1 ^ ... ^ f_k (Eq. Oplus).  So the stream splits
// into P = B*T segments of L rounds:
//
//  * jump-ahead: with m_g(z) the minimal polynomial of generator g's state
//    transition A_g (host, once per process: Krylov elimination, verified on
//    every basis vector), the state J steps ahead is
//        S_J = sum_i c_i S_i,   c(z) = z^J mod m_g(z),
//    S_i the state i steps ahead -- a "window" of the generator's own output
//    sequence.  Segment j = b T + t (thread t of block b) jumps straight from
//    the chunk start with z^(j L) (host-computed polynomials, one per segment,
//    cached per (L, B) in the handle; the two-level form -- block start with
//    z^(b T L), then z^(t L) from it -- is the CIPRNG_JUMP_ONE_LEVEL=0 build);
//  * each thread generates its L words as a LOCAL prefix XOR (staged in
//    shared memory), a block-wide XOR scan and a look-back over the earlier
//    blocks' aggregates (cooperative launch: all blocks co-resident) give
//    every segment its x offset, and the block writes its T*L contiguous
//    output words coalesced;
//  * the thread owning the chunk's last round writes the state back.
//
// Bit-exact with the sequential chain (and the oracle) by construction: the
// jump is exact linear algebra over GF(2) and XOR is associative.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include "device.cuh"
#include "kernels.h"

namespace ciprng {

namespace {

// -------------------------------------------------------------- host GF(2)
// Polynomials over GF(2): bit i of word i/64 = coefficient of z^i.
using Poly = std::vector<uint64_t>;

int pdeg(const Poly &p) {
    for (int w = (int)p.size() - 1; w >= 0; --w)
        if (p[w]) return 64 * w + 63 - __builtin_clzll(p[w]);
    return -1;
}
inline bool pbit(const Poly &p, int i) { return (p[i >> 6] >> (i & 63)) & 1u; }
inline void pflip(Poly &p, int i) { p[i >> 6] ^= 1ull << (i & 63); }

// r ^= m << s (m has `words` words, r is long enough)
void xor_shifted(Poly &r, const Poly &m, int s) {
    const int ws = s >> 6, bs = s & 63;
    for (size_t w = 0; w < m.size(); ++w) {
        if (!m[w]) continue;
        r[w + ws] ^= m[w] << bs;
        if (bs && w + ws + 1 < r.size()) r[w + ws + 1] ^= m[w] >> (64 - bs);
    }
}

// a * b mod m, deg a, deg b < deg m = dm
Poly mulmod(const Poly &a, const Poly &b, const Poly &m, int dm) {
    const size_t W = (size_t)(2 * dm + 64) / 64 + 1;
    Poly r(W, 0), bb(b);
    bb.resize(W, 0);
    for (int i = 0; i <= pdeg(a); ++i)
        if (pbit(a, i)) xor_shifted(r, b, i);
    for (int i = pdeg(r); i >= dm; --i)
        if (pbit(r, i)) xor_shifted(r, m, i - dm);
    r.resize((size_t)dm / 64 + 1);
    return r;
}

// z^e mod m
Poly zpow(uint64_t e, const Poly &m, int dm) {
    Poly r((size_t)dm / 64 + 1, 0), base = r;
    r[0] = 1;  // 1
    if (dm == 0) return r;
    base[0] = 2;  // z (dm >= 2 here)
    while (e) {
        if (e & 1) r = mulmod(r, base, m, dm);
        e >>= 1;
        if (e) base = mulmod(base, base, m, dm);
    }
    return r;
}

// Generator g's state transition on a bit vector of W words.
void step_state(int g, uint64_t *s) {
    if (g == 0) {
        s[0] = xor64_step(s[0]);
    } else if (g == 1) {
        const uint64_t nb = xor128_f64(s[0], s[3]);
        s[0] = s[1]; s[1] = s[2]; s[2] = s[3]; s[3] = nb;
    } else {
        const uint64_t nc = xorwow_f64(s[0], s[4]);
        s[0] = s[1]; s[1] = s[2]; s[2] = s[3]; s[3] = s[4]; s[4] = nc;
    }
}
constexpr int kGenWords[3] = {1, 4, 5};

// Minimal polynomial of the Krylov sequence v, A v, A^2 v, ... by Gaussian
// elimination: the first A^k v in the span of the earlier ones gives
// A^k v = sum c_i A^i v, i.e. the polynomial z^k + sum c_i z^i.
Poly krylov_minpoly(int g, const uint64_t *v0) {
    const int W = kGenWords[g], D = 64 * W;
    struct Row {
        uint64_t v[5];
        Poly c;
    };
    std::vector<int> piv_row(D, -1);
    std::vector<Row> rows;
    uint64_t cur[5] = {0, 0, 0, 0, 0};
    std::memcpy(cur, v0, W * 8);
    for (int k = 0; k <= D; ++k) {
        Row r;
        std::memcpy(r.v, cur, sizeof(r.v));
        r.c.assign((size_t)D / 64 + 1, 0);
        pflip(r.c, k);
        for (int bit = D - 1; bit >= 0; --bit) {
            if (!((r.v[bit >> 6] >> (bit & 63)) & 1u) || piv_row[bit] < 0) continue;
            const Row &p = rows[piv_row[bit]];
            for (int w = 0; w < W; ++w) r.v[w] ^= p.v[w];
            for (size_t w = 0; w < r.c.size(); ++w) r.c[w] ^= p.c[w];
        }
        int top = -1;
        for (int bit = D - 1; bit >= 0 && top < 0; --bit)
            if ((r.v[bit >> 6] >> (bit & 63)) & 1u) top = bit;
        if (top < 0) return r.c;  // dependency found
        piv_row[top] = (int)rows.size();
        rows.push_back(r);
        step_state(g, cur);
    }
    return Poly();  // unreachable: D + 1 vectors in a D-dimensional space
}

// m(A) e_j == 0 for every basis vector e_j
bool annihilates(int g, const Poly &m) {
    const int W = kGenWords[g], D = 64 * W, dm = pdeg(m);
    for (int j = 0; j < D; ++j) {
        uint64_t cur[5] = {0, 0, 0, 0, 0}, acc[5] = {0, 0, 0, 0, 0};
        cur[j >> 6] = 1ull << (j & 63);
        for (int i = 0; i <= dm; ++i) {
            if (pbit(m, i))
                for (int w = 0; w < W; ++w) acc[w] ^= cur[w];
            step_state(g, cur);
        }
        for (int w = 0; w < W; ++w)
            if (acc[w]) return false;
    }
    return true;
}

struct MinPolys {
    Poly m[3];
    int deg[3] = {0, 0, 0};
    bool ok = false;
};

const MinPolys &min_polys() {
    static MinPolys mp;
    static std::once_flag once;
    std::call_once(once, [] {
        bool ok = true;
        for (int g = 0; g < 3; ++g) {
            // a fixed, dense start vector (SplitMix64 words): a cyclic vector
            // of A_g with overwhelming probability; verified below
            uint64_t v[5];
            for (int w = 0; w < 5; ++w) v[w] = splitmix_fin(0x5EEDull + 0x9E3779B97F4A7C15ull * (uint64_t)(8 * g + w + 1));
            mp.m[g] = krylov_minpoly(g, v);
            mp.deg[g] = pdeg(mp.m[g]);
            ok = ok && mp.deg[g] > 0 && mp.deg[g] <= kJumpMaxDeg[g] && annihilates(g, mp.m[g]);
        }
        mp.ok = ok;
    });
    return mp;
}

}  // namespace

bool v0_jump_available() { return min_polys().ok; }

// Host self-test of the jump-ahead algebra (no GPU): for each generator, from
// a few seeded states, the state J steps ahead computed as sum_i c_i S_i with
// c = z^J mod m_g must equal J plain steps, for J up to 3*10^5.
int v0_jump_selftest(uint64_t *mismatches, uint32_t *degrees) {
    const MinPolys &mp = min_polys();
    uint64_t bad = mp.ok ? 0 : 1;
    for (int g = 0; g < 3; ++g) {
        degrees[g] = (uint32_t)mp.deg[g];
        if (!mp.ok) continue;
        const int W = kGenWords[g], dm = mp.deg[g];
        for (uint64_t seed = 1; seed <= 3; ++seed) {
            uint64_t s[5];
            for (int w = 0; w < 5; ++w) s[w] = splitmix_fin(seed * 0x9E3779B97F4A7C15ull + 77u * (uint64_t)(w + 1) + g);
            std::vector<uint64_t> win((size_t)dm * W);
            uint64_t cur[5];
            std::memcpy(cur, s, sizeof(cur));
            for (int i = 0; i < dm; ++i) {
                std::memcpy(&win[(size_t)i * W], cur, (size_t)W * 8);
                step_state(g, cur);
            }
            uint64_t ref[5];
            std::memcpy(ref, s, sizeof(ref));
            uint64_t done = 0;
            for (uint64_t J : {0ull, 1ull, 2ull, 63ull, 64ull, 253ull, 320ull, 1000ull, 6784ull, 299999ull}) {
                for (; done < J; ++done) step_state(g, ref);
                const Poly c = zpow(J, mp.m[g], dm);
                uint64_t acc[5] = {0, 0, 0, 0, 0};
                for (int i = 0; i < dm; ++i)
                    if (pbit(c, i))
                        for (int w = 0; w < W; ++w) acc[w] ^= win[(size_t)i * W + w];
                for (int w = 0; w < W; ++w) bad += acc[w] != ref[w];
            }
        }
    }
    *mismatches = bad;
    return 0;
}

// ------------------------------------------------------------------ kernel
// Shared-memory windows: generator g's output sequence, window i = state
// after i steps = words [i, i + kGenWords[g]).  Each array ends in zero
// words: the sweep's sliding window reads up to 64 * ceil(deg / 64) + W - 1
// (the polynomial bits past deg are zero, so those words never count).
constexpr uint32_t kZ1 = kJumpMaxDeg[0], kZ2 = kJumpMaxDeg[1] + 3, kZ3 = kJumpMaxDeg[2] + 4;
struct JumpSmem {
    uint64_t w1[kZ1 + 1];
    uint64_t w2[kZ2 + 4];
    uint64_t w3[kZ3 + 5];
    uint64_t part[kJumpThreads / 32][10];
    uint64_t bstart[10];
    uint64_t bpoly[3][kJumpPolyWords];  // this block's level-1 polynomials
    uint32_t st0[24];                   // the chunk-start state planes
    uint32_t warp_tot[kJumpThreads / 32];
    uint32_t block_base;
};

struct JumpArgs {
    uint32_t *state;        // V0 SoA planes: word k of stream s at state[k * state_stride + s]
    uint64_t state_stride;  // = n_local
    uint32_t *out;          // this chunk's first word of stream 0; stream s at out + s * out_stride
    uint64_t out_stride;    // = n (rounds per stream of the whole call)
    uint64_t n_chunk;       // rounds in this chunk
    const uint64_t *poly;   // jump polynomials, generator g at poly + g * (T + B) * kJumpPolyWords:
                            // thread slots [q][t], then block slots [b][q]
    uint32_t deg[3];
    uint32_t L, B;
    uint32_t *flags;  // [B] epoch flags
    uint32_t *aggs;   // [B] block aggregates (XOR of the block's f)
    uint32_t epoch;
    unsigned long long *dbg;  // CIPRNG_JUMP_TIMING builds: [B][16] phase timestamps
};

// Phase timestamps (diagnostic builds, -DCIPRNG_JUMP_TIMING): thread 0 of
// every CTA records %globaltimer at each phase boundary; the host prints the
// latest CTA's time per phase (the timestamp stores themselves can queue
// behind pending loads, so a phase right after a barrier may absorb their
// latency).  Measured (r2, 10^6 numbers, 24.8 us per call): Krylov windows
// 1.7, block jump 3.0, Krylov again 1.7, table build 4.7, nibble lookups 3.2,
// generation 2.6, scans + look-back 2.5, write 0.5 us.  Tried and slower: a
// bit-by-bit sweep (11.8 us, ALU bound), the sweep split over 4 threads per
// segment (30.7 us per call), a branch-free masked table build (26.6 us).
#if defined(CIPRNG_JUMP_TIMING)
#define JT(k)                                                              \
    do {                                                                   \
        if (t == 0 && blockIdx.y == 0 && a.dbg) {                          \
            unsigned long long ts;                                         \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));         \
            a.dbg[b * 16 + (k)] = ts;                                      \
        }                                                                  \
    } while (0)
#else
#define JT(k) \
    do {      \
    } while (0)
#endif

// One thread per generator: the first deg_g windows of the state in s10
// (word layout: a | b0..b3 | c0..c4), then the zero tail.  The register
// rings are unrolled by their period so the loop body is the recurrence
// and one shared store per step.
__device__ __forceinline__ void krylov_windows(JumpSmem &sm, const uint64_t (&s10)[10], const JumpArgs &a) {
    const uint32_t t = threadIdx.x;
    if (t == 0) {
        uint64_t v = s10[0];
        for (uint32_t i = 0; i < a.deg[0]; i += 4) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                sm.w1[i + u] = v;
                v = xor64_step(v);
            }
        }
        sm.w1[kZ1] = 0;
    } else if (t == 32) {
        uint64_t b0 = s10[1], b1 = s10[2], b2 = s10[3], b3 = s10[4];
        sm.w2[0] = b0; sm.w2[1] = b1; sm.w2[2] = b2; sm.w2[3] = b3;
        for (uint32_t k = 4; k < a.deg[1] + 3; k += 4) {
            b0 = xor128_f64(b0, b3); sm.w2[k] = b0;
            b1 = xor128_f64(b1, b0); sm.w2[k + 1] = b1;
            b2 = xor128_f64(b2, b1); sm.w2[k + 2] = b2;
            b3 = xor128_f64(b3, b2); sm.w2[k + 3] = b3;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) sm.w2[kZ2 + k] = 0;
    } else if (t == 64) {
        uint64_t c0 = s10[5], c1 = s10[6], c2 = s10[7], c3 = s10[8], c4 = s10[9];
        sm.w3[0] = c0; sm.w3[1] = c1; sm.w3[2] = c2; sm.w3[3] = c3; sm.w3[4] = c4;
        for (uint32_t k = 5; k < a.deg[2] + 4; k += 5) {
            c0 = xorwow_f64(c0, c4); sm.w3[k] = c0;
            c1 = xorwow_f64(c1, c0); sm.w3[k + 1] = c1;
            c2 = xorwow_f64(c2, c1); sm.w3[k + 2] = c2;
            c3 = xorwow_f64(c3, c2); sm.w3[k + 3] = c3;
            c4 = xorwow_f64(c4, c3); sm.w3[k + 4] = c4;
        }
#pragma unroll
        for (int k = 0; k < 5; ++k) sm.w3[kZ3 + k] = 0;
    }
}

// Level-2 jump by the "method of four Russians": the windows are taken in
// chunks of four (indices 4c .. 4c+3) and for every chunk the 16 XOR
// combinations of its four windows are tabulated in shared memory,
// tab[c][k][p] = XOR over the set bits j of p of word k of window 4c + j.
// A thread then applies its polynomial one NIBBLE at a time: one table load
// and one XOR per state word per four bits, against 4 masked XORs per word
// in a bit-by-bit sweep (which was ALU bound: 11.8 of 27 us per C1 call).
// The 16 entries of tab[c][k] are 128 contiguous bytes -- one per bank pair
// -- so lanes reading different nibbles never conflict and equal nibbles
// broadcast.
constexpr uint32_t kTab1 = kJumpMaxDeg[0] / 4, kTab2 = kJumpMaxDeg[1] / 4, kTab3 = kJumpMaxDeg[2] / 4;
constexpr size_t kTabWords = (size_t)16 * (kTab1 * 1 + kTab2 * 4 + kTab3 * 5);

// Build generator g's tables: thread t computes entries (2t, 2t + 1),
// (2t + 2T, 2t + 2T + 1), ... of the flat [chunk][word][16] array -- each an
// XOR of at most four window words (broadcast loads: neighbouring threads
// share the chunk) -- so a warp's stores cover 256 contiguous bytes.
template <int W>
__device__ __forceinline__ void pair_vals(const uint64_t *w, uint32_t e2, uint64_t &even, uint64_t &odd) {
    const uint32_t ck = e2 >> 3, p0 = (e2 & 7u) * 2;  // (chunk, word) and the even pattern
    const uint32_t c = ck / W, k = ck - c * W;
    const uint64_t *wc = w + 4 * c + k;
    even = 0;
    if (p0 & 2) even ^= wc[1];
    if (p0 & 4) even ^= wc[2];
    if (p0 & 8) even ^= wc[3];
    odd = even ^ wc[0];  // p0 + 1 adds window 4c
}
__device__ __forceinline__ void st_pair(uint64_t *tab, uint32_t e2, uint64_t even, uint64_t odd) {
    asm volatile("st.shared.v2.u64 [%0], {%1, %2};" ::"r"(smem_u32(tab + 2 * (size_t)e2)), "l"(even), "l"(odd)
                 : "memory");
}
template <int W>
__device__ __forceinline__ void build_tables(const uint64_t *w, uint32_t chunks, uint64_t *tab) {
    const uint32_t pairs = chunks * W * 8;  // two entries per pair
#if !defined(CIPRNG_JUMP_TAB_SINGLE)
    // four independent pairs per iteration, all loads before the stores (one
    // warp per SMSP: a lone pair waits out the shared-memory latency of its
    // loads): 25.3 -> 24.6 us per C1 call (profiles/experiments/s67); the
    // one-pair loop below is the CIPRNG_JUMP_TAB_SINGLE comparison build
    const uint32_t T = blockDim.x;
    uint32_t e2 = threadIdx.x;
    for (; e2 + 3 * T < pairs; e2 += 4 * T) {
        uint64_t e[4], o[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) pair_vals<W>(w, e2 + r * T, e[r], o[r]);
#pragma unroll
        for (int r = 0; r < 4; ++r) st_pair(tab, e2 + r * T, e[r], o[r]);
    }
    for (; e2 < pairs; e2 += T) {
        uint64_t e0, o0;
        pair_vals<W>(w, e2, e0, o0);
        st_pair(tab, e2, e0, o0);
    }
    return;
#endif
    for (uint32_t e2 = threadIdx.x; e2 < pairs; e2 += blockDim.x) {
        const uint32_t ck = e2 >> 3, p0 = (e2 & 7u) * 2;  // (chunk, word) and the even pattern
        const uint32_t c = ck / W, k = ck - c * W;
        const uint64_t *wc = w + 4 * c + k;
        uint64_t even = 0;
        if (p0 & 2) even ^= wc[1];
        if (p0 & 4) even ^= wc[2];
        if (p0 & 8) even ^= wc[3];
        const uint64_t odd = even ^ wc[0];  // p0 + 1 adds window 4c
        asm volatile("st.shared.v2.u64 [%0], {%1, %2};" ::"r"(smem_u32(tab + 2 * (size_t)e2)), "l"(even), "l"(odd)
                     : "memory");
    }
}

template <int W, int Q>
__device__ __forceinline__ void jump_tab(const uint64_t *tab, const uint64_t (&poly)[Q], uint32_t deg, uint64_t *acc) {
#pragma unroll 1
    for (uint32_t q = 0; q < (uint32_t)Q && q * 64 < deg; ++q) {
        uint64_t bits = 0;
#pragma unroll
        for (int r = 0; r < Q; ++r)
            if (r == (int)q) bits = poly[r];
        const uint64_t *tq = tab + (size_t)q * 16 * W * 16;  // 16 chunks per poly word
#if defined(CIPRNG_JUMP_LOOKUP_UNROLL)  // experiment: 4 / 1 measured 22.0 / 23.5 vs 20.5 us (s75)
        constexpr int kU = CIPRNG_JUMP_LOOKUP_UNROLL;
#pragma unroll kU
#else
#pragma unroll
#endif
        for (uint32_t j = 0; j < 16; ++j) {
            const uint32_t nib = (uint32_t)(bits >> (4 * j)) & 15u;
#pragma unroll
            for (int k = 0; k < W; ++k) acc[k] ^= tq[(j * W + k) * 16 + nib];
        }
    }
}

__global__ void __launch_bounds__(kJumpThreads) v0_jump_kernel(JumpArgs a) {
    extern __shared__ __align__(16) uint8_t jsm_raw[];
    JumpSmem &sm = *reinterpret_cast<JumpSmem *>(jsm_raw);
    uint32_t *stage = reinterpret_cast<uint32_t *>(jsm_raw + ((sizeof(JumpSmem) + 15) & ~size_t(15)));
    // grid: x = CTA of the stream's segment range, y = stream (one stream per
    // grid row; each row has its own look-back flags)
    const uint32_t T = kJumpThreads, t = threadIdx.x, b = blockIdx.x, L = a.L;
    const uint64_t sid = blockIdx.y;
    uint32_t *const flags = a.flags + sid * a.B, *const aggs = a.aggs + sid * a.B;
    uint32_t *const out = a.out + sid * a.out_stride;
    const uint32_t lane = t & 31u, warp = t >> 5;
    uint64_t pj1[1], pj2[4], pj3[5];
#if kJumpOneLevel
    // this thread's segment polynomial z^((b T + t) L), loaded early and
    // coalesced ([g][q][segment]): the jump goes straight from the chunk start
    {
        const size_t J = (size_t)a.B * T, j = (size_t)b * T + t, PW = J * kJumpPolyWords;
        pj1[0] = __ldg(a.poly + j);
#pragma unroll
        for (int q = 0; q < 4; ++q) pj2[q] = __ldg(a.poly + PW + (size_t)q * J + j);
#pragma unroll
        for (int q = 0; q < 5; ++q) pj3[q] = __ldg(a.poly + 2 * PW + (size_t)q * J + j);
    }
#else
    const size_t PW = (size_t)(T + a.B) * kJumpPolyWords;  // poly words per generator
    // this thread's level-2 jump polynomials (z^(t L)), loaded early
    pj1[0] = __ldg(a.poly + t);
#pragma unroll
    for (int q = 0; q < 4; ++q) pj2[q] = __ldg(a.poly + PW + (size_t)q * T + t);
#pragma unroll
    for (int q = 0; q < 5; ++q) pj3[q] = __ldg(a.poly + 2 * PW + (size_t)q * T + t);

    // this block's level-1 polynomials (z^(b T L)) into shared memory now, so
    // the level-1 pass after the first Krylov phase reads no global memory
    if (t < 3 * kJumpPolyWords) {
        const uint32_t g = t / kJumpPolyWords, q = t % kJumpPolyWords;
        sm.bpoly[g][q] = __ldg(a.poly + g * PW + (size_t)T * kJumpPolyWords + (size_t)b * kJumpPolyWords + q);
    }
#endif

    // chunk start state (words: a, b0..b3, c0..c4), d, x
    // One coalesced load per CTA (lanes 0..22 of warp 0), shared through
    // shared memory: every thread loading the 23 words itself sent 13 k
    // requests for one cache line from all CTAs to one L2 slice -- ~4 us of
    // queueing at the start of every call (found with -DCIPRNG_JUMP_TIMING).
    if (t < 23) sm.st0[t] = a.state[t * a.state_stride + sid];
    __syncthreads();
    uint64_t s0[10];
#pragma unroll
    for (int k = 0; k < 10; ++k) s0[k] = (uint64_t)sm.st0[2 * k] | ((uint64_t)sm.st0[2 * k + 1] << 32);
    const uint64_t d0 = (uint64_t)sm.st0[20] | ((uint64_t)sm.st0[21] << 32);
    const uint32_t x0 = sm.st0[22];

    // level 1: this block's start = z^(b T L) applied to the chunk start.
    // Every thread takes a slice of the list; XOR-reduce over the block.
    JT(0);
    krylov_windows(sm, s0, a);
    __syncthreads();
    JT(1);
#if !kJumpOneLevel
    {
        uint64_t part[10];
#pragma unroll
        for (int k = 0; k < 10; ++k) part[k] = 0;
        // <= 3 iterations per generator: NOT unrolled.  This code runs once
        // per warp, so its size is its cost -- ptxas' 8-way unrolled copy
        // (21 KB of SASS) took 5.1 us of instruction-cache misses per call
        const uint64_t *q1 = sm.bpoly[0], *q2 = sm.bpoly[1], *q3 = sm.bpoly[2];
#pragma unroll 1
        for (uint32_t i = t; i < kZ1; i += T)  // bits past deg are 0
            if ((q1[i >> 6] >> (i & 63)) & 1u) part[0] ^= sm.w1[i];
        JT(12);
#pragma unroll 1
        for (uint32_t i = t; i < kZ2 - 3; i += T)
            if ((q2[i >> 6] >> (i & 63)) & 1u)
#pragma unroll
                for (int k = 0; k < 4; ++k) part[1 + k] ^= sm.w2[i + k];
        JT(13);
#pragma unroll 1
        for (uint32_t i = t; i < kZ3 - 4; i += T)
            if ((q3[i >> 6] >> (i & 63)) & 1u)
#pragma unroll
                for (int k = 0; k < 5; ++k) part[5 + k] ^= sm.w3[i + k];
        JT(9);
#pragma unroll
        for (int k = 0; k < 10; ++k) {
#pragma unroll
            for (int dlt = 16; dlt; dlt >>= 1) part[k] ^= __shfl_xor_sync(kFull, part[k], dlt);
        }
        JT(10);
        if (lane == 0)
#pragma unroll
            for (int k = 0; k < 10; ++k) sm.part[warp][k] = part[k];
    }
    __syncthreads();
    JT(11);
    if (t < 10) {
        uint64_t v = 0;
        for (uint32_t w = 0; w < T / 32; ++w) v ^= sm.part[w][t];
        sm.bstart[t] = v;
    }
    __syncthreads();
    uint64_t sb[10];
#pragma unroll
    for (int k = 0; k < 10; ++k) sb[k] = sm.bstart[k];
    __syncthreads();
    // level 2: this thread's start = z^(t L) applied to the block start
    JT(2);
    krylov_windows(sm, sb, a);
    __syncthreads();
#endif
    JT(3);
    uint64_t *tab1 = reinterpret_cast<uint64_t *>(stage + (size_t)T * L);  // after the staging area
    uint64_t *tab2 = tab1 + (size_t)16 * kTab1, *tab3 = tab2 + (size_t)16 * kTab2 * 4;
    build_tables<1>(sm.w1, (a.deg[0] + 3) / 4, tab1);
    build_tables<4>(sm.w2, (a.deg[1] + 3) / 4, tab2);
    build_tables<5>(sm.w3, (a.deg[2] + 3) / 4, tab3);
    __syncthreads();
    uint64_t s[10];
#pragma unroll
    for (int k = 0; k < 10; ++k) s[k] = 0;
    jump_tab<1>(tab1, pj1, a.deg[0], s);
    jump_tab<4>(tab2, pj2, a.deg[1], s + 1);
    jump_tab<5>(tab3, pj3, a.deg[2], s + 5);

    JT(4);
    // generate this segment as a local prefix XOR
    const uint64_t seg = (uint64_t)b * T + t, r0 = seg * L;
    const uint32_t len = r0 >= a.n_chunk ? 0u : (uint32_t)(a.n_chunk - r0 < L ? a.n_chunk - r0 : L);
    uint64_t ra = s[0], rb0 = s[1], rb1 = s[2], rb2 = s[3], rb3 = s[4];
    uint64_t rc0 = s[5], rc1 = s[6], rc2 = s[7], rc3 = s[8], rc4 = s[9];
    uint64_t rd = d0 + r0 * 362437ull;
    uint32_t xl = 0;
    for (uint32_t k = 0; k < len; ++k) {
        ra = xor64_step(ra);
        const uint64_t nb = xor128_f64(rb0, rb3);
        rb0 = rb1; rb1 = rb2; rb2 = rb3; rb3 = nb;
        const uint64_t nc = xorwow_f64(rc0, rc4);
        rc0 = rc1; rc1 = rc2; rc2 = rc3; rc3 = rc4; rc4 = nc;
        rd += 362437u;
        const uint64_t t3 = rd + nc;
        xl ^= (uint32_t)ra ^ (uint32_t)(nb >> 32) ^ (uint32_t)(t3 >> 32) ^ (uint32_t)nb ^ (uint32_t)(ra >> 32) ^
              (uint32_t)t3;
        stage[t * L + k] = xl;
    }

    JT(5);
    // block-wide exclusive XOR scan of the segment totals
    uint32_t incl = xl;
#pragma unroll
    for (int dlt = 1; dlt < 32; dlt <<= 1) {
        const uint32_t v = __shfl_up_sync(kFull, incl, dlt);
        if (lane >= (uint32_t)dlt) incl ^= v;
    }
    if (lane == 31) sm.warp_tot[warp] = incl;
    __syncthreads();
    uint32_t wpre = 0, agg = 0;
#pragma unroll
    for (uint32_t w = 0; w < T / 32; ++w) {
        if (w < warp) wpre ^= sm.warp_tot[w];
        agg ^= sm.warp_tot[w];
    }
    const uint32_t excl = wpre ^ incl ^ xl;
    JT(6);
    // publish this block's aggregate, then look back over the earlier blocks
    // (all co-resident: cooperative launch)
    if (t == 0) {
        aggs[b] = agg;
        __threadfence();
        atomicExch(flags + b, a.epoch);
    }
    uint32_t prev = 0;
    for (uint32_t j = t; j < b; j += T) {
        while (atomicAdd(flags + j, 0u) != a.epoch) {
        }
        __threadfence();
        prev ^= *reinterpret_cast<volatile uint32_t *>(aggs + j);
    }
#pragma unroll
    for (int dlt = 16; dlt; dlt >>= 1) prev ^= __shfl_xor_sync(kFull, prev, dlt);
    __syncthreads();  // every warp has read warp_tot above
    if (lane == 0) sm.warp_tot[warp] = prev;  // reuse: per-warp partial of the look-back
    __syncthreads();
    if (t == 0) {
        uint32_t base = x0;
        for (uint32_t w = 0; w < T / 32; ++w) base ^= sm.warp_tot[w];
        sm.block_base = base;
    }
    __syncthreads();
    const uint32_t base = sm.block_base ^ excl;
    for (uint32_t k = 0; k < len; ++k) stage[t * L + k] ^= base;
    __syncthreads();
    JT(7);
    // coalesced write of the block's contiguous T*L words
    const uint64_t blk0 = (uint64_t)b * T * L;
    const uint64_t blen =
        blk0 >= a.n_chunk ? 0 : (a.n_chunk - blk0 < (uint64_t)T * L ? a.n_chunk - blk0 : (uint64_t)T * L);
    for (uint64_t k = t; k < blen; k += T) out[blk0 + k] = stage[k];

    JT(8);
    // state after the chunk: owned by the segment holding its last round
    if (len > 0 && r0 + len == a.n_chunk) {
        const uint64_t v[11] = {ra, rb0, rb1, rb2, rb3, rc0, rc1, rc2, rc3, rc4, rd};
#pragma unroll
        for (int k = 0; k < 11; ++k) {
            a.state[(2 * k) * a.state_stride + sid] = (uint32_t)v[k];
            a.state[(2 * k + 1) * a.state_stride + sid] = (uint32_t)(v[k] >> 32);
        }
        a.state[22 * a.state_stride + sid] = base ^ xl;
    }
}

// ------------------------------------------------------------------- host
void v0_jump_free(V0JumpPlan &p) {
    cudaFree(p.poly);
    cudaFree(p.flags);
    p = V0JumpPlan();
}

static size_t jump_smem(uint32_t L) {
    // staging area (T * L words, padded to 16 bytes), then the nibble tables
    return ((sizeof(JumpSmem) + 15) & ~size_t(15)) + (((size_t)kJumpThreads * L * 4 + 15) & ~size_t(15)) +
           kTabWords * 8;
}

// (Re)build the plan for (L, B): polynomials z^(t L), t < T (thread slots,
// interleaved [q][t]) and z^(b T L), b < B (block slots, [b][q]), as
// kJumpPolyWords-word bit masks per generator.
static int v0_jump_build(V0JumpPlan &p, const MinPolys &mp, uint32_t L, uint32_t B, uint32_t streams) {
    const uint32_t T = kJumpThreads;
    v0_jump_free(p);
#if kJumpOneLevel
    // one polynomial per segment j = b T + t: c_j = z^(j L) mod m_g, as
    // c_{j+1} = (z^L) c_j mod m_g -- multiplication by a fixed polynomial is
    // GF(2)-linear, so it is the XOR of precomputed columns z^i z^L mod m_g
    // over the set bits i of c_j (~10 us per thousand segments on the host)
    const size_t J = (size_t)B * T, PW = J * kJumpPolyWords;
    std::vector<uint64_t> host(3 * PW, 0);
    for (int g = 0; g < 3; ++g) {
        const int dm = mp.deg[g];
        const size_t nw = (size_t)dm / 64 + 1;
        std::vector<Poly> col((size_t)dm);
        col[0] = zpow(L, mp.m[g], dm);
        col[0].resize(nw, 0);
        for (int i = 1; i < dm; ++i) {  // col[i] = z col[i-1] mod m
            Poly c = col[i - 1];
            uint64_t carry = 0;
            for (size_t w = 0; w < nw; ++w) {
                const uint64_t nc = c[w] >> 63;
                c[w] = (c[w] << 1) | carry;
                carry = nc;
            }
            if (pbit(c, dm))
                for (size_t w = 0; w < nw && w < mp.m[g].size(); ++w) c[w] ^= mp.m[g][w];
            col[i] = c;
        }
        Poly c(nw, 0);
        c[0] = 1;
        for (size_t j = 0; j < J; ++j) {
            for (size_t q = 0; q < nw && q < (size_t)kJumpPolyWords; ++q) host[g * PW + q * J + j] = c[q];
            Poly nx(nw, 0);
            for (int i = 0; i < dm; ++i)
                if (pbit(c, i))
                    for (size_t w = 0; w < nw; ++w) nx[w] ^= col[i][w];
            c.swap(nx);
        }
    }
#else
    const size_t PW = (size_t)(T + B) * kJumpPolyWords;
    std::vector<uint64_t> host(3 * PW, 0);
    for (int g = 0; g < 3; ++g) {
        const int dm = mp.deg[g];
        const Poly zL = zpow(L, mp.m[g], dm), zTL = zpow((uint64_t)T * L, mp.m[g], dm);
        for (int level = 0; level < 2; ++level) {
            const Poly &step = level == 0 ? zL : zTL;
            const uint32_t n_slots = level == 0 ? T : B;
            Poly c((size_t)dm / 64 + 1, 0);
            c[0] = 1;
            for (uint32_t k = 0; k < n_slots; ++k) {
                for (size_t q = 0; q < c.size() && q < (size_t)kJumpPolyWords; ++q) {
                    const size_t pos = level == 0 ? q * T + k : (size_t)T * kJumpPolyWords + (size_t)k * kJumpPolyWords + q;
                    host[g * PW + pos] = c[q];
                }
                c = mulmod(c, step, mp.m[g], dm);
            }
        }
    }
#endif
    if (cudaMalloc(&p.poly, host.size() * 8) != cudaSuccess) return -2;
    if (cudaMalloc(&p.flags, (size_t)2 * streams * B * 4) != cudaSuccess) return -2;
    cudaMemcpy(p.poly, host.data(), host.size() * 8, cudaMemcpyHostToDevice);
    cudaMemset(p.flags, 0, (size_t)2 * streams * B * 4);
    p.L = L;
    p.B = B;
    p.streams = streams;
    p.epoch = 0;
    return 0;
}

int v0_jump_launch(V0JumpPlan &p, uint32_t *state, uint64_t n_local, uint32_t *out, uint64_t n, cudaStream_t st) {
    const MinPolys &mp = min_polys();
    if (!mp.ok || n == 0 || n_local == 0 || n_local > kJumpMaxStreams) return -1;
    const uint32_t T = kJumpThreads;
    // The device queries below cost more host time than the kernel runs, so
    // they are made once per plan; a call with the plan's n reuses it as is.
    if (!(p.poly && p.n == n && p.streams == n_local)) {
        int dev = 0, sms = 148, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        // CTAs per stream: the SMs shared among the streams (one grid row each)
        const uint64_t per_stream = std::max<uint64_t>(1, (uint64_t)sms / n_local);
        // L: about one segment per thread of one CTA per SM, 16..kJumpMaxL rounds
        uint64_t L = (n + (uint64_t)T * per_stream - 1) / ((uint64_t)T * per_stream);
        L = L < 16 ? 16 : (L > kJumpMaxL ? kJumpMaxL : L);
        const size_t smem = jump_smem((uint32_t)L);
        if (cudaFuncSetAttribute(v0_jump_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
            return -1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, v0_jump_kernel, T, smem);
        if (per_sm < 1) return -1;
        uint64_t B = (n + T * L - 1) / (T * L);
        const uint64_t maxB = (uint64_t)sms * (uint64_t)per_sm / n_local;  // co-resident, all streams
        if (maxB < 1) return -1;
        if (B > maxB) B = maxB;
        if (!(p.poly && p.L == L && p.B == B && p.streams == n_local)) {
            const int rc = v0_jump_build(p, mp, (uint32_t)L, (uint32_t)B, (uint32_t)n_local);
            if (rc < 0) return rc;
        }
        p.n = n;
        p.smem = smem;
    }
    const uint64_t L = p.L, B = p.B;
    const size_t smem = p.smem;
    const uint64_t chunk = (uint64_t)T * B * L;
    int launches = 0;
    for (uint64_t r = 0; r < n; r += chunk) {
        JumpArgs ja;
        ja.state = state;
        ja.state_stride = n_local;
        ja.out = out + r;
        ja.out_stride = n;
        ja.n_chunk = n - r < chunk ? n - r : chunk;
        ja.poly = p.poly;
        for (int g = 0; g < 3; ++g) ja.deg[g] = (uint32_t)mp.deg[g];
        ja.L = p.L;
        ja.B = p.B;
        ja.flags = p.flags;
        ja.aggs = p.flags + n_local * p.B;
        ja.dbg = nullptr;
#if defined(CIPRNG_JUMP_TIMING)
        static unsigned long long *dbg = nullptr;
        if (!dbg) cudaMalloc(&dbg, (size_t)16 * 4096 * 8);
        cudaMemset(dbg, 0, (size_t)16 * 4096 * 8);
        ja.dbg = dbg;
#endif
        ja.epoch = ++p.epoch;
        if (ja.epoch == 0) ja.epoch = ++p.epoch;  // flags start at 0: never reuse 0
        // cooperative: the look-back spins on earlier blocks' flags
        const uint32_t blocks = (uint32_t)((ja.n_chunk + (uint64_t)T * L - 1) / ((uint64_t)T * L));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(blocks, (uint32_t)n_local);
        cfg.blockDim = dim3(T);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        const cudaError_t e = cudaLaunchKernelEx(&cfg, v0_jump_kernel, ja);
        if (e != cudaSuccess) {
            // nothing enqueued yet: the caller may fall back to the one-thread
            // kernel; after a chunk ran, the state has moved -- report it
            if (launches == 0) {
                cudaGetLastError();  // clear the launch error before the fallback
                return -3;
            }
            return -4;
        }
        ++launches;
#if defined(CIPRNG_JUMP_TIMING)
        {
            std::vector<unsigned long long> h((size_t)16 * blocks);
            cudaMemcpy(h.data(), ja.dbg, h.size() * 8, cudaMemcpyDeviceToHost);
            unsigned long long t0 = ~0ull;
            for (uint32_t bb = 0; bb < blocks; ++bb) t0 = std::min(t0, h[bb * 16]);
            double mx[9] = {0};
            for (uint32_t bb = 0; bb < blocks; ++bb)
                for (int k = 0; k < 9; ++k) mx[k] = std::max(mx[k], (double)(h[bb * 16 + k] - t0) * 1e-3);
            fprintf(stderr, "jump phases (us, latest CTA, from the first start): start %.2f krylov1 %.2f lvl1 %.2f "
                    "krylov2 %.2f sweep %.2f gen %.2f scan %.2f lookback %.2f write %.2f\n",
                    mx[0], mx[1], mx[2], mx[3], mx[4], mx[5], mx[6], mx[7], mx[8]);
            // per-CTA phase durations: median and max over CTAs
            for (int k : {1, 12, 13, 9, 10, 11, 2, 3, 4, 5, 6, 7, 8}) {
                std::vector<double> dd;
                const int kp = k == 12 ? 1 : k == 13 ? 12 : k == 9 ? 13 : k == 10 ? 9 : k == 11 ? 10 : k == 2 ? 11 : k - 1;
                for (uint32_t bb = 0; bb < blocks; ++bb)
                    if (h[bb * 16 + k] && h[bb * 16 + kp])  // the one-level jump skips the block-start stamps
                        dd.push_back((double)(h[bb * 16 + k] - h[bb * 16 + kp]) * 1e-3);
                if (dd.empty()) continue;
                std::sort(dd.begin(), dd.end());
                fprintf(stderr, "  phase %d: median %.2f max %.2f us\n", k, dd[dd.size() / 2], dd.back());
            }
        }
#endif
    }
    return launches;
}

}  // namespace ciprng
