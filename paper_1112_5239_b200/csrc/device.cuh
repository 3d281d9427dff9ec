// device.cuh -- sm_100a device primitives of the chaotic-iteration PRNG.
//
// Independent of oracle/ (no shared code or tables).  Citations: P:a-b =
// PAPER.md lines; Qn = DESIGN.md s3 readings.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace ciprng {

constexpr uint32_t kFull = 0xFFFFFFFFu;

// ---------------------------------------------------------------- seeder
// Q11: W(seed, s, k) = SplitMix64 output number 16 s + k + 1 from `seed`.
__host__ __device__ __forceinline__ uint64_t splitmix_fin(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}
__host__ __device__ __forceinline__ uint64_t seed_word(uint64_t seed, uint64_t s, uint32_t k) {
    return splitmix_fin(seed + 0x9E3779B97F4A7C15ull * (s * 16u + k + 1u));
}

// ------------------------------------------------------- xor-like sources
// Marsaglia xor128 on 32-bit words (Alg. 4 source), written as
// the 4-term recurrence w_{k+4} = f(w_k, w_{k+3}) so an unroll-by-4 loop
// keeps the state in a register ring with no moves.
// Constant right shift as a high multiply (IMAD.HI on the heavy FMA
// sub-pipe) instead of SHF on the ALU pipe.  Inline PTX so the compiler
// cannot canonicalise it back into SHF.  Pipe costs measured with ncu (r1d):
// an ALU op or IMAD/IMAD.SHL holds its pipe 2 cycles per warp, IMAD.HI 4.
template <int k>
__device__ __forceinline__ uint32_t shr_fma(uint32_t v) {
    uint32_t r;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(v), "n"(1u << (32 - k)));
    return r;
}
// xor128 step with the pipes balanced: x << 11 is IMAD.SHL, w >> 19 is
// IMAD.HI, t >> 8 stays SHF; with the combination's LOP3s the V1 kernels
// spend ~11 ALU and ~6 heavy-FMA cycles per warp-number (all shifts on SHF:
// 13 / 2; both right shifts as IMAD.HI: 9 / 10).
__device__ __forceinline__ uint32_t xor128_f(uint32_t xk, uint32_t wk3) {
    uint32_t t = xk ^ (xk << 11);
#if defined(CIPRNG_EXP_X128_ALL_HI)  // experiment: both right shifts as IMAD.HI (heavy FMA)
    return (wk3 ^ shr_fma<19>(wk3)) ^ (t ^ shr_fma<8>(t));
#else
    return (wk3 ^ shr_fma<19>(wk3)) ^ (t ^ (t >> 8));
#endif
}
// The same with both right shifts on SHF (ALU): the V1 fused consumer, whose
// pi-pair test is IMAD.WIDE-heavy, balances its pipes better this way --
// 1.816 -> 1.847e12 numbers/s; both shifts as IMAD.HI 1.740e12
// (profiles/experiments/s53_x128_shifts.jsonl).
__device__ __forceinline__ uint32_t xor128_f_alu(uint32_t xk, uint32_t wk3) {
#if defined(CIPRNG_EXP_X128_SHL_ALU)  // experiment: the left shift on SHF too: 1.840 -> 1.698e12 (s54), off
    uint32_t sh;
    asm("shf.l.clamp.b32 %0, %1, %2, 11;" : "=r"(sh) : "r"(0u), "r"(xk));
    uint32_t t = xk ^ sh;
#else
    uint32_t t = xk ^ (xk << 11);
#endif
    return (wk3 ^ (wk3 >> 19)) ^ (t ^ (t >> 8));
}
// Same on 64-bit words (Listing 1's xor128, reading Q2).
__host__ __device__ __forceinline__ uint64_t xor128_f64(uint64_t xk, uint64_t wk3) {
    uint64_t t = xk ^ (xk << 11);
    return (wk3 ^ (wk3 >> 19)) ^ (t ^ (t >> 8));
}
// xorwow shift register on 64-bit words: v_{k+5} = (v ^ v<<4) ^ (t ^ t<<1),
// t = x ^ x>>2 with x = v_k, v = v_{k+4} (Q2, Q3).
__host__ __device__ __forceinline__ uint64_t xorwow_f64(uint64_t xk, uint64_t vk4) {
    uint64_t t = xk ^ (xk >> 2);
    return (vk4 ^ (vk4 << 4)) ^ (t ^ (t << 1));
}
// Marsaglia xor64 (13, 7, 17) (Listing 1's xorshift, reading Q1-A).
__host__ __device__ __forceinline__ uint64_t xor64_step(uint64_t a) {
    a ^= a << 13;
    a ^= a >> 7;
    a ^= a << 17;
    return a;
}

// --------------------------------------------------------------- BBS mod
// Division-free x^2 mod M for M < 2^16 (P:1209-1214 wants 32-bit modular
// arithmetic only).  Barrett: mu = floor(2^32 / M); for T = y*y < 2^32,
// q = hi32(T * mu) is floor(T/M) or floor(T/M) - 1, so r = T - q*M < 2M and
// one conditional subtraction (unsigned min, one VIADDMNMX) finishes.  The
// modulus is kept negated (nM = 2^32 - M) so r = T + q*nM is a single IMAD:
// 4 instructions per squaring.  Exhaustively checked by prng_selftest_modsq()
// for every modulus and every y < M.
__host__ __device__ __forceinline__ uint32_t barrett_sq(uint32_t y, uint32_t nM, uint32_t mu) {
    uint32_t T = y * y;
#ifdef __CUDA_ARCH__
    uint32_t q = __umulhi(T, mu);
#else
    uint32_t q = (uint32_t)(((uint64_t)T * mu) >> 32);
#endif
    uint32_t r = T + q * nM;  // T - q*M
    uint32_t r2 = r + nM;     // r - M (wraps iff r < M)
    return r2 < r ? r2 : r;
}

// Montgomery form (north_star's "Montgomery-style" squaring; SURVEY s8(d)
// asks for the Barrett-vs-Montgomery comparison).  R = 2^32, Mp = -M^{-1}
// mod 2^32.  For a single word T with T < M^2 (or T < M):
//   m = T*Mp (mod 2^32);  T + m*M = 0 (mod 2^32), so lo(m*M) = 2^32 - T when
//   T != 0 and REDC(T) = (T + m*M) / 2^32 = hi(m*M) + [T != 0];
//   REDC(T) < (M^2 + 2^32*M) / 2^32 < M + 1, and REDC(T) = M would need
//   M | T, which for T = yh^2 or T = y*R2 (yh, y < M = pq) means T = 0, and
//   T = 0 gives 0: the result is canonical with no final subtraction.
// Squaring in the Montgomery domain, yh = y*R mod M: yh' = REDC(yh^2); the
// canonical y' (whose low bits Alg. 5 consumes) costs a second REDC(yh').
// Heavy-pipe cost per squaring: 3 IMAD + 2 IMAD.HI = 14 cycles per warp vs
// Barrett's 8 -- built as a measured alternative (CIPRNG_V2_KIND=10),
// exhaustively checked like the others.
__host__ __device__ __forceinline__ uint32_t mont_redc(uint32_t T, uint32_t M, uint32_t Mp) {
    const uint32_t m = T * Mp;
#ifdef __CUDA_ARCH__
    // [T != 0] as min(T, 1), the addend of one IMAD.HI (written in PTX: from
    // C++ the compiler evaluates both hi(m*M) and hi(m*M) + 1 and selects)
    uint32_t r;
    asm("{\n\t.reg .u32 c;\n\tmin.u32 c, %1, 1;\n\tmad.hi.u32 %0, %2, %3, c;\n\t}"
        : "=r"(r)
        : "r"(T), "r"(m), "r"(M));
    return r;
#else
    return (uint32_t)(((uint64_t)m * M) >> 32) + (T < 1u ? T : 1u);
#endif
}
// enter: y*R mod M = REDC(y * (R^2 mod M)) (y*R2 < M^2)
__host__ __device__ __forceinline__ uint32_t mont_enter(uint32_t y, uint32_t M, uint32_t Mp, uint32_t R2) {
    return mont_redc(y * R2, M, Mp);
}
// one BBS squaring in Montgomery form: yh <- REDC(yh^2); returns canonical y
__host__ __device__ __forceinline__ uint32_t mont_sq(uint32_t &yh, uint32_t M, uint32_t Mp) {
    yh = mont_redc(yh * yh, M, Mp);
    return mont_redc(yh, M, Mp);
}

// The same squaring with the quotient taken from the FP32 pipe, which runs
// beside the heavy FMA sub-pipe (IMAD + FFMA interleaved: 118 lane-ops/clk/SM,
// profiles/r1e_pipe_microbench.json), so the half-rate IMAD.HI leaves the
// bound pipe: 2 IMAD (4 heavy cycles) instead of IMAD + IMAD.HI + IMAD (8).
//   yf = y exactly (y < 2^23: magic-exponent conversion, LOP3 + FADD)
//   Tf = RZ(y*y)              relative error < 2^-23, Tf <= y^2
//   invMf = RZ(1/M)           relative error < 2^-23, invMf <= 1/M
//   qb = RZ(Tf*invMf + 2^23)  one FFMA: the exact product, one rounding; the
//        sum lies in [2^23, 2^24) where RZ = floor, so bits(qb) = 0x4B000000
//        + floor(Tf*invMf), and y^2/M - Tf*invMf < 2^-22 * y^2/M < 2^-6
//        gives floor(Tf*invMf) in {q - 1, q}, q = floor(y^2 / M).
//   r = y*y + K + bits(qb)*(2^32 - M) = y^2 - q_est*M (mod 2^32), with
//        K = 0x4B000000 * M mod 2^32 cancelling the exponent bits; r < 2M,
//        so the same unsigned-min subtraction finishes.
// Exhaustively checked against % by prng_selftest_modsq() (host emulation
// below, bit-exact by construction) and by the GPU test of every modulus
// and every y < M through the kernel itself.
__host__ __device__ __forceinline__ uint32_t fbarrett_sq(uint32_t y, uint32_t nM, uint32_t K, uint32_t invMf) {
#ifdef __CUDA_ARCH__
    const float yf = __uint_as_float(y | 0x4B000000u) - 8388608.0f;
    const float Tf = __fmul_rz(yf, yf);
    const uint32_t qb = __float_as_uint(__fmaf_rz(Tf, __uint_as_float(invMf), 8388608.0f));
#else
    uint64_t T = (uint64_t)y * y;  // RZ to 24 significant bits
    int bl = 0;
    while (bl < 64 && (T >> bl)) ++bl;
    if (bl > 24) T = (T >> (bl - 24)) << (bl - 24);
    const uint64_t m = (invMf & 0x7FFFFFu) | 0x800000u;           // invMf = m * 2^-e
    const int e = 127 + 23 - (int)((invMf >> 23) & 0xFFu);           // e in (23, 64) here
    const uint32_t qb = 0x4B000000u + (uint32_t)((T * m) >> e);     // T*m < 2^56
#endif
    const uint32_t r = y * y + K + qb * nM;
    const uint32_t r2 = r + nM;
    return r2 < r ? r2 : r;
}

// ---------------------------------------------------------------- stores
__device__ __forceinline__ void st_v4(uint32_t *p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}
// streaming (evict-first) variant: the output is written once, never re-read
__device__ __forceinline__ void st_v4_cs(uint32_t *p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.global.cs.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c,
                                             uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}

// ------------------------------------------------------------------- TMA
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap *map, uint32_t smem_addr, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
            reinterpret_cast<uint64_t>(map)),
        "r"(smem_addr), "r"(c0), "r"(c1)
        : "memory");
}
// Same with an L2 cache-eviction policy (createpolicy): the output is written
// once and never re-read by this kernel, so it is stored evict-first and does
// not push the L2-persisting state planes out.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t l2_evict_normal_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// State-plane accesses with an L2 policy (evict-last keeps the planes, read
// and rewritten every call, resident while the output streams through L2).
__device__ __forceinline__ uint32_t ld_state(const uint32_t *p, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_state(uint32_t *p, uint32_t v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void tma_store_2d_hint(const CUtensorMap *map, uint32_t smem_addr, int c0, int c1,
                                                  uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], %4;" ::"l"(
            reinterpret_cast<uint64_t>(map)),
        "r"(smem_addr), "r"(c0), "r"(c1), "l"(pol)
        : "memory");
}
// L2 prefetch of `bytes` (multiple of 16, 16-byte aligned) global bytes
__device__ __forceinline__ void bulk_prefetch_l2(const void *p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Byte offset of 16-byte chunk c of row r in a tile of kCols u32 columns
// (row pitch P = 4 kCols bytes) written with CU_TENSOR_MAP_SWIZZLE_{P}B:
// the chunk index is XORed with address bits [7, 7 + log2(P/16)), i.e. with
// (r * P / 128) mod (P / 16).  For every P this makes the 8 lanes of one
// STS.128 phase (8 consecutive rows, same chunk) hit 8 distinct 16-byte
// bank groups.
template <int kCols>
__device__ __forceinline__ uint32_t swz(uint32_t r, uint32_t c) {
    constexpr uint32_t P = kCols * 4;
    return r * P + ((c ^ ((r * P >> 7) & (P / 16 - 1))) << 4);
}

// Write a warp's swizzled shared-memory box (64 rows x kCols words, rows
// 0..63 of the tile at row0, rounds i0..i0+cols) to out[row * n + round]
// with coalesced stores -- the staged store path (no TMA descriptor needed):
// rows 16-byte aligned (vec): lane l moves 16-byte chunk l%8 of rows 4k+l/8
// (STG.128, 4 rows per instruction); otherwise lane l moves word l of one
// row (128 contiguous bytes per instruction at any 4-byte alignment).  Both
// read the swizzled box bank-conflict-free.
template <int kCols>
__device__ __forceinline__ void staged_writeback(uint32_t buf, uint32_t *out, uint64_t row0, uint64_t rows_valid,
                                                 uint64_t n, uint64_t i0, uint64_t cols, bool vec, bool cs,
                                                 uint32_t lane) {
    static_assert(kCols == 32, "staged write-back is for 32-round boxes");
    if (vec) {
        const uint32_t c = lane & 7u, rsub = lane >> 3;
#pragma unroll 4
        for (uint32_t r = rsub; r < 64u; r += 4) {
            if (row0 + r >= rows_valid || 4u * c >= cols) continue;
            uint32_t v0, v1, v2, v3;
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3)
                         : "r"(buf + swz<kCols>(r, c)));
            uint32_t *dst = out + (row0 + r) * n + i0 + 4u * c;
            if (cs) st_v4_cs(dst, v0, v1, v2, v3);
            else st_v4(dst, v0, v1, v2, v3);
        }
    } else {
        const uint32_t c = lane >> 2, w = lane & 3u;
#pragma unroll 4
        for (uint32_t r = 0; r < 64u; ++r) {
            if (row0 + r >= rows_valid || lane >= cols) continue;
            uint32_t v;
            asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(buf + swz<kCols>(r, c) + 4u * w));
            uint32_t *dst = out + (row0 + r) * n + i0 + lane;
            if (cs) __stcs(dst, v);
            else *dst = v;
        }
    }
}

// ------------------------------------------- programmatic dependent launch
// Every kernel is launched with programmatic stream serialization (PDL): it
// lets the next kernel on the stream be scheduled while this one drains, and
// griddepcontrol.wait blocks until the previous grid has completed and its
// memory is visible -- so nothing global is touched before pdl_wait().
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// --------------------------------------------------- consumer statistics
// Q24: pair (u, v) is "inside" iff u^2 + v^2 < 2^64 <=> v^2 <= ~(u^2).
__device__ __forceinline__ uint32_t pi_inside(uint32_t u, uint32_t v) {
    uint64_t uu = (uint64_t)u * u, vv = (uint64_t)v * v;
    return vv <= ~uu ? 1u : 0u;
}

// ------------------------------------------------------ kernel arguments
struct CombTables {
    uint8_t t[16][32];  // V1 uses rows 0 (array_comb1) and 1 (array_comb2)
};

struct GenArgs {
    uint32_t *state;     // SoA planes, plane stride = n_local words
    uint64_t n_local;    // plane stride
    uint64_t s_begin;    // first local stream of this launch
    uint64_t s_count;    // streams in this launch (multiple of C for V1/V2)
    uint64_t n;          // rounds per stream
    uint32_t *out;       // row 0 = stream s_begin; row stride n (store kernels)
    uint64_t *stats;     // consume kernels: 258 u64
    const uint32_t *mod; // V2: [78][kModWords] = {invMf, mu, 2^32 - M, K, M, Mp, R2, 0} (api.cu)
    uint32_t C;          // combination_size
    uint32_t vec;        // 1: rows are 16-byte aligned, n % 4 == 0
    uint32_t evict_first; // 1: output stores carry an L2 evict-first hint
    uint32_t state_last;  // 1: state-plane loads/stores carry an L2 evict-last hint
    uint32_t pf_ahead;    // V1 TMA store: prefetch into L2 the state of tile + pf_ahead (0 = off)
    uint32_t zero;        // always 0 (memset): a multiplier the compiler cannot fold (sinks.cuh)
    CombTables comb;
};

// SoA state-plane access (plane k of local stream s at word k*L + s).  Every
// access carries an L2 cache-policy operand chosen once per kernel --
// evict-last when a.state_last, else evict-normal -- so there is no
// per-access branch (a branch per load serialised V2's dependent modulus
// loads: -10 %, gpurun_out/s14).
struct StateIO {
    uint32_t *P;
    uint64_t L;
    uint64_t pol;
    __device__ __forceinline__ explicit StateIO(const GenArgs &a)
        : P(a.state), L(a.n_local), pol(a.state_last ? l2_evict_last_policy() : l2_evict_normal_policy()) {}
    __device__ __forceinline__ uint32_t ld(uint32_t k, uint64_t s) const { return ld_state(P + k * L + s, pol); }
    __device__ __forceinline__ void st(uint32_t k, uint64_t s, uint32_t v) const { st_state(P + k * L + s, v, pol); }
};

}  // namespace ciprng

namespace ciprng {
// ------------------------------------------ 64-bit xor-like on 32-bit halves
// Listing 1's generators on (lo, hi) register pairs.  A 64-bit constant
// shift has a plain half (one 32-bit shift, written as a multiply: IMAD.SHL
// or IMAD.HI on the FMA pipe) and a funnel half that combines both words.
// The funnel half is either one SHF (ALU pipe) or -- template flag kF --
// two multiplies (IMAD.SHL + IMAD.HI) whose disjoint bit ranges are merged by
// the XOR that consumes the shift anyway (a 3-input LOP3), moving one ALU op
// to 6 heavy-FMA cycles.  Measured (ncu r1d/r1h): IMAD.HI holds the heavy
// sub-pipe twice as long as IMAD.SHL or an ALU op; all-SHF funnels leave V0
// ALU-bound (86 %) with the FMA pipe at 15 %, all-multiply funnels made V0
// heavy-bound and 15 % slower, so each generator converts only some shifts.
struct u64p {
    uint32_t lo, hi;
};
template <int k>
__device__ __forceinline__ uint32_t mul_pow2(uint32_t v) {  // v << k as IMAD.SHL
    uint32_t r;
    asm("mul.lo.u32 %0, %1, %2;" : "=r"(r) : "r"(v), "n"(1u << k));
    return r;
}
template <int k, bool kF = false>
__device__ __forceinline__ u64p shl64(u64p a) {  // a << k, 0 < k < 32
    if constexpr (kF) return {mul_pow2<k>(a.lo), mul_pow2<k>(a.hi) ^ shr_fma<32 - k>(a.lo)};
    else return {mul_pow2<k>(a.lo), __funnelshift_l(a.lo, a.hi, k)};
}
template <int k, bool kF = false>
__device__ __forceinline__ u64p shr64(u64p a) {  // a >> k, 0 < k < 32
    if constexpr (kF) return {shr_fma<k>(a.lo) ^ mul_pow2<32 - k>(a.hi), shr_fma<k>(a.hi)};
    else return {__funnelshift_r(a.lo, a.hi, k), shr_fma<k>(a.hi)};
}
__device__ __forceinline__ u64p xor64p(u64p a, u64p b) { return {a.lo ^ b.lo, a.hi ^ b.hi}; }
__device__ __forceinline__ u64p xor64p(u64p a, u64p b, u64p c) { return {a.lo ^ b.lo ^ c.lo, a.hi ^ b.hi ^ c.hi}; }
// kF bits select which of a generator's three shifts use the multiply funnel
template <int kF = 0>
__device__ __forceinline__ u64p xor64_step_p(u64p a) {
    a = xor64p(a, shl64<13, (kF & 1) != 0>(a));
    a = xor64p(a, shr64<7, (kF & 2) != 0>(a));
    a = xor64p(a, shl64<17, (kF & 4) != 0>(a));
    return a;
}
template <int kF = 0>
__device__ __forceinline__ u64p xor128_f64p(u64p xk, u64p wk3) {
    u64p t = xor64p(xk, shl64<11, (kF & 1) != 0>(xk));
    u64p r = xor64p(wk3, shr64<19, (kF & 2) != 0>(wk3), t);
    return xor64p(r, shr64<8, (kF & 4) != 0>(t));
}
template <int kF = 0>
__device__ __forceinline__ u64p xorwow_f64p(u64p xk, u64p vk4) {
    u64p t = xor64p(xk, shr64<2, (kF & 1) != 0>(xk));
    u64p r = xor64p(vk4, shl64<4, (kF & 2) != 0>(vk4), t);
    return xor64p(r, shl64<1, (kF & 4) != 0>(t));
}
__device__ __forceinline__ u64p add64p(u64p a, u64p b) {
    uint64_t s = ((uint64_t)a.hi << 32 | a.lo) + ((uint64_t)b.hi << 32 | b.lo);
    return {(uint32_t)s, (uint32_t)(s >> 32)};
}
}  // namespace ciprng
