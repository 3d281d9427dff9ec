/*
 * ciprng.h -- C ABI of the B200-native chaotic-iteration PRNG hot path
 * (arXiv 1112.5239, Bahi, Couturier, Guyeux, Heam).
 *
 * One handle = the persistent per-thread state of the paper's GPU kernels
 * ("InternalVarXorLikeArray" / "InternalVarBBSArray", P:895-905, P:959-978,
 * P:1254-1287) for a contiguous range of streams (one stream = one paper
 * thread), resident in HBM of the device that was current at creation.
 *
 * Citations: P:a-b = PAPER.md lines a-b; Qn = reading n of the ambiguity
 * ledger, DESIGN.md s3.
 *
 * Conventions for every entry point
 *  - Returns PRNG_OK (0) or a negative prng_status; never throws, never
 *    aborts.  PRNG_ECUDA carries a CUDA error (prng_last_cuda_error() gives
 *    its text); asynchronous kernel faults surface at the next synchronising
 *    call.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  Device-pointer calls only ENQUEUE work on `stream` and return
 *    immediately; handle state updates are stream-ordered.
 *  - A handle is single-owner: concurrent calls on one handle (from several
 *    host threads or on several streams without ordering) are undefined
 *    (SPEC S:85-86).  Distinct handles are independent.
 *  - Pointers named *_dev are device pointers (e.g. a torch tensor's
 *    data_ptr()); *_host are host pointers; the caller owns both.
 */
#ifndef CIPRNG_H
#define CIPRNG_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define CIPRNG_API __attribute__((visibility("default")))
#else
#define CIPRNG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct prng_s prng_t; /* opaque; owns the device state */

/* Variants:
 *  V0  Listing 1 per thread = Alg. 3 "naive" kernel:
 *      three 64-bit xor-like generators (xor64, xor128, xorwow; readings
 *      Q1-A, Q2, Q3); x ^= lo(t1)^hi(t2)^hi(t3)^lo(t2)^hi(t1)^lo(t3).
 *  V1  Alg. 4 "improved" kernel: one 32-bit xor128 per thread
 *      (Q5); t = xor128() ^ shmem[o1] ^ shmem[o2]; shmem[tid] = t; x ^= t.
 *  V2  Alg. 5 BBS kernel: 8 Blum-Blum-Shub instances, 4 low
 *      bits per squaring, two variable shifts, 16 arrangement arrays chosen
 *      per call, state rotation at exit.
 *  V3 Alg. 4 with the xor64 source of the paper's
 *      "optimized versions": t = low 32 bits of xor64()
 *      (reading Q29) ^ shmem[o1] ^ shmem[o2].
 *  V4  (NEXT-1) Alg. 4 with Listing 1's three generators and six-word fold
 *       as the strategy source (reading Q30).
 * V3 and V4 take Alg. 4's two combination arrays exactly like V1. */
enum prng_variant {
    PRNG_V0_XORLIKE3 = 0,
    PRNG_V1_XOR128_COMB = 1,
    PRNG_V2_BBS_COMB = 2,
    PRNG_V3_XOR64_COMB = 3,
    PRNG_V4_XORLIKE3_COMB = 4
};

enum prng_status {
    PRNG_OK = 0,
    PRNG_EINVAL = -1,  /* bad argument / configuration                */
    PRNG_ENOMEM = -2,  /* device or host allocation failed            */
    PRNG_ECUDA = -3,   /* CUDA runtime / driver error                 */
    PRNG_EALIGN = -4,  /* out_dev not 16-byte aligned when required   */
    PRNG_ESIZE = -5,   /* size overflow (n * n_local * 4 > SIZE_MAX)   */
    PRNG_ESTATE = -6,  /* state buffer size mismatch (get/set_state), or
                          set_state content invalid (see prng_set_state) */
    PRNG_EIO = -7      /* prng_emit: a write to the sink failed (errno is
                          left as write(2) set it)                    */
};

/* Serialisation formats of prng_emit. */
enum prng_emit_format {
    PRNG_EMIT_RAW_LE32 = 0, /* 4 bytes per word, little-endian u32         */
    PRNG_EMIT_HEX = 1,      /* "%08x\n": 8 lowercase hex digits + newline   */
    PRNG_EMIT_BITS = 2      /* 32 ASCII '0'/'1', most significant bit first
                               (reading Q31), + newline                     */
};

/* Store path of prng_generate (tuning knob; every path is bit-identical). */
enum prng_store_path {
    PRNG_STORE_AUTO = 0,   /* TMA tiles when possible, else shared-memory
                              staging + coalesced stores (V1 default tables) */
    PRNG_STORE_DIRECT = 1, /* per-thread 128-bit STG of 4-round buffers   */
    PRNG_STORE_TMA = 2,    /* warp tiles staged in shared memory, written
                              by cp.async.bulk.tensor (V1 default tables,
                              n % 4 == 0); falls back to DIRECT otherwise */
    PRNG_STORE_JUMP = 3    /* reported by prng_get_info only: a V0 handle
                              with at most 16 streams and n >= 4096 splits
                              each stream over the GPU by GF(2) jump-ahead
                              of its generators + an XOR scan of x (same
                              words; BASELINE configs[0] / C1) */
};

typedef struct prng_config {
    /* combination_size C (reading Q6): 0 = default 32.
     * Must be 1, 2, 4, 8, 16 or 32 (a group never straddles a warp).
     * V3 and V4 use V1's two arrays and defaults. */
    uint32_t comb_size;
    /* HOST pointer, copied at creation.  V1: 2*C entries, array_comb1 then
     * array_comb2.  V2: 16*C entries, array_comb[0..15][0..C-1]
     * row-major.  Each entry < C.  NULL = the default tables, which
     * exist for C = 32 only (Q6): V1 comb1[l] = l+1, comb2[l] = l+17 (mod
     * 32); V2 array_comb[a][l] = l+1+a, array_comb[8+a][l] = l+17+a (mod 32),
     * a = 0..7.  Ignored by V0. */
    const uint8_t *comb;
    /* V0 with a single stream only: Listing 1's initial state (x =
     * 123123123, with Marsaglia's published seeds; Q12). */
    int32_t paper_defaults;
    /* enum prng_store_path */
    int32_t store_path;
} prng_config;

/* ---------------------------------------------------------------------- */
/* Lifetime                                                               */
/* ---------------------------------------------------------------------- */

/* prng_create(seed, n_streams, variant, &h) == prng_create_shard(seed, 0,
 * n_streams, variant, NULL, &h).  Synchronous (returns with the state
 * initialised on the current device). */
CIPRNG_API int prng_create(uint64_t seed, uint64_t n_streams, int variant, prng_t **out);

/* Create the handle for global streams [first_stream, first_stream+n_local)
 * of the stream space seeded by `seed`.  The state of global stream s is a
 * pure function of (seed, s, variant) (seeder, reading Q11: SplitMix64
 * counter words W(seed, s, k)), so the output of stream s never depends on
 * how streams are sharded over handles or GPUs.
 * Errors: PRNG_EINVAL if variant unknown, n_local == 0, out == NULL,
 * comb_size not a power of two <= 32, a table entry >= C, comb == NULL with
 * C != 32, V1-V4 with first_stream % C or n_local % C != 0 (groups must be
 * complete), paper_defaults with anything but V0 and
 * (first_stream, n_local) == (0, 1) (Q26). PRNG_ENOMEM, PRNG_ECUDA. */
CIPRNG_API int prng_create_shard(uint64_t seed, uint64_t first_stream, uint64_t n_local, int variant,
                      const prng_config *cfg, prng_t **out);

/* Frees the device state and any staging buffers.  NULL is a no-op.
 * Synchronises with outstanding work of the handle's internal streams. */
CIPRNG_API int prng_destroy(prng_t *h);

/* ---------------------------------------------------------------------- */
/* Hot path                                                               */
/* ---------------------------------------------------------------------- */

/* One kernel call of n_per_stream rounds on every stream of the handle
 * (Alg. 3 / 4 / 5 "for i=1 to n"): each round draws
 * the strategy word t, combines it with the group's previous-round shared
 * cells (V1, V2), applies x ^= t (Eq. "Oplus") and emits x.
 * Output layout (reading Q9): stream-major, out_dev[s_local*n + i] is round
 * i of local stream s_local; n_local*n u32 words, caller-owned.  State is
 * written back at the end; V2 rotates its 8 BBS instances
 * (Q19, Q20).  n_per_stream == 0: no-op, no launch,
 * no V2 rotation.  V0/V1 are chunk-split invariant: generate(a+b) ==
 * generate(a) ++ generate(b) row-wise; V2 is not (its arrangement arrays are
 * chosen per call).
 * Errors: PRNG_EINVAL (h NULL, or out_dev NULL with n > 0), PRNG_ESIZE, PRNG_EALIGN (the TMA
 * store path requires 16-byte alignment; other paths fall back to scalar
 * stores when out_dev or n is not 16-byte friendly), PRNG_ECUDA. */
CIPRNG_API int prng_generate(prng_t *h, uint64_t n_per_stream, uint32_t *out_dev, void *stream);

/* Same words as prng_generate, written to a HOST buffer (n_local*n u32,
 * stream-major).  Generation runs on `stream` in stream-range chunks into
 * two device staging buffers owned by the handle while the previous chunk
 * is copied device->host on an internal copy stream.  Pinned host memory is
 * strongly recommended (pageable memory works but copies synchronously).
 * SYNCHRONOUS: returns after the last word has landed in out_host. */
CIPRNG_API int prng_generate_host(prng_t *h, uint64_t n_per_stream, uint32_t *out_host, void *stream);

/* Emitter for external test batteries (SURVEY s8(b) raw-LE32 sink; SPEC
 * S:378 "raw little-endian 32-bit words to file or standard output",
 * S:642-650 emit(generator, count, format); the paper fed its outputs to
 * DieHARD / TestU01 BigCrush).  Runs ONE call of n rounds --
 * the same words and state evolution as prng_generate -- and writes the
 * words in prng_generate's order (stream-major: local stream s, then round
 * i) to the open file descriptor `fd` (1 = standard output) in `format`
 * (enum prng_emit_format).  Pipeline: stream-range chunks of ~64 MiB of
 * serialised bytes are generated (and, for the text formats, formatted by a
 * kernel) on `stream`, copied to pinned host buffers owned by the handle on
 * an internal copy stream, and written by the calling thread while the next
 * chunk is generated.  SYNCHRONOUS.  *bytes_written (may be NULL) = bytes
 * successfully written.  n == 0 writes nothing.  Errors: PRNG_EINVAL (NULL
 * handle, fd < 0, unknown format), PRNG_ESIZE, PRNG_ENOMEM, PRNG_ECUDA,
 * PRNG_EIO (a write failed: the remaining chunks are still generated, so the
 * state has advanced by the whole call, but not written). */
CIPRNG_API int prng_emit(prng_t *h, uint64_t n_per_stream, int fd, int format, uint64_t *bytes_written,
                         void *stream);

/* Fused consumer mode (the paper removes the store; statistics
 * are reading Q24): run the same n rounds as prng_generate -- identical
 * state evolution -- but use every x in-kernel instead of storing it, and
 * ADD into stats_dev[258] (u64, caller-zeroed):
 *   [0] pairs (u, v) = (x_{2k}, x_{2k+1}) of one stream within the call with
 *       u^2 + v^2 < 2^64 (Monte-Carlo pi: pi ~ 4*[0]/[1]);
 *   [1] number of pairs = n_local * n / 2;
 *   [2 + b] count of x with x >> 24 == b, b = 0..255.
 * Integer sums, so results are independent of launch shape and of how
 * streams are sharded (the multi-GPU all-reduce is bit-exact).  Launch:
 * V1 / V3 with the default arrays run 14-warp CTAs with one 64 KiB
 * histogram each (dynamic shared memory, set per call with
 * cudaFuncSetAttribute on the current device), other kernels per-warp 1 KiB
 * histograms; the V1 / V3 kernels fall back to the per-warp form when the
 * device's reserved shared memory per block is not 1 KiB.
 * Errors: PRNG_EINVAL if n is odd or a pointer is NULL, PRNG_ESIZE if
 * n >= 2^24 (split the call; V0/V1/V3/V4 are split invariant), PRNG_ECUDA. */
CIPRNG_API int prng_consume(prng_t *h, uint64_t n_per_stream, uint64_t *stats_dev, void *stream);

/* Statistical battery in consumer form (the tests of
 * monobit, block frequency m = 128, runs, serial 2-bit,
 * byte chi-square, 8-lag autocorrelation -- stand in for the BigCrush runs
 * the paper reports).  Runs the same n rounds as prng_generate
 * (identical state evolution) and ADDS integer counts into stats_dev[264]
 * (u64, caller-zeroed).  A stream's bit sequence within the call is its
 * words in round order, each most significant bit first (reading Q31):
 *   [0] one bits            [1] adjacent bit pairs that differ
 *   [2] adjacent pairs 11   [3] bit pairs 8 apart that differ
 *   [4] sum over 128-bit blocks (words 4k..4k+3) of (ones - 64)^2
 *   [5] number of blocks    [6] / [7] first / last bits equal to 1
 *   [8 + b] bytes equal to b, all four bytes of every word.
 * P-values are computed on the host from these counts
 * (paper_1112_5239_b200/battery.py).  Integer sums: independent of launch
 * shape and sharding.  Launch: V1 / V3 with the default arrays run one
 * 28-warp CTA per SM with a 64 KiB byte histogram (dynamic shared memory,
 * the same fallback as prng_consume), other kernels per-warp histograms.
 * Errors: PRNG_EINVAL (NULL), PRNG_ESIZE (n >= 2^20), PRNG_ECUDA. */
CIPRNG_API int prng_battery(prng_t *h, uint64_t n_per_stream, uint64_t *stats_dev, void *stream);

/* Verification digest of one call's output block (reading Q28; a check
 * value defined by this build, the paper has none).  Each stream's row is
 * taken in word pairs (out[s*n + 2j], out[s*n + 2j + 1]), the lone last word
 * of an odd row paired with 0, and
 *   digest_dev[0] += sum over pairs of mix64((hi << 32 | lo) + P * G)
 *   (mod 2^64), P = (first_stream + s) * ceil(n / 2) + j,
 * mix64 = the SplitMix64 finaliser, G = 0x9E3779B97F4A7C15 -- output number
 * P of SplitMix64 seeded with the pair.  Position-aware, additive across
 * shards (rows are whole units), and a bijection of each pair for a fixed
 * position (one wrong word always changes the digest).  out_dev needs 4-byte
 * alignment (8-byte and an even n take the vectorised kernel).
 * Errors: PRNG_EINVAL (NULL), PRNG_ECUDA. */
CIPRNG_API int prng_digest(const uint32_t *out_dev, uint64_t first_stream, uint64_t n_local, uint64_t n,
                uint64_t *digest_dev, void *stream);

/* ---------------------------------------------------------------------- */
/* Blum-Goldwasser and the paper's chaotic variant  */
/* ---------------------------------------------------------------------- */

/* Batch encryption, one independent message per GPU thread.
 * Classic Blum-Goldwasser (chaotic == 0): x_0 = r^2 mod N,
 * c_i = m_i ^ lsb(x_i), x_{i+1} = x_i^2 mod N, y = x_L.
 * Chaotic variant (chaotic != 0, reading Q33): units of
 * Nb = floor(log2(log2 N)) bits, b_i = x_i mod 2^Nb,
 * c_i = m_i ^ (b_0 ^ ... ^ b_i) ^ S0 (the cumulative XOR of Eq. "Oplus").
 * Arguments (device pointers, caller-owned):
 *   N_dev[n_msgs]  public moduli, odd, 3 <= N < 2^63 (N = p q, p, q = 3 mod 4)
 *   S0_dev[n_msgs] the variant's public S0 (< 2^Nb); NULL = all 0; ignored
 *                  by classic BG
 *   r_dev[n_msgs]  the sender's random r, gcd(r, N) = 1
 *   m_dev, c_dev   L units per message, one unit per byte (a bit for
 *                  classic BG, Nb bits for the variant; higher bits of m are
 *                  ignored, those of c are 0), message-major: unit i of
 *                  message k at [k * L + i]
 *   y_dev[n_msgs]  out: y = x_L mod N.  A message whose N or r
 *                  violates the constraints gets y = 0 (never a valid y) and
 *                  no ciphertext.
 * Enqueued on `stream`.  Errors: PRNG_EINVAL (NULL pointers), PRNG_ESIZE,
 * PRNG_ECUDA. */
CIPRNG_API int prng_cbg_encrypt(int chaotic, uint64_t n_msgs, uint64_t L, const uint64_t *N_dev,
                                const uint32_t *S0_dev, const uint64_t *r_dev, const uint8_t *m_dev,
                                uint8_t *c_dev, uint64_t *y_dev, void *stream);

/* Batch decryption with the secret factors: r_p =
 * y^(((p+1)/4)^L) mod p, r_q likewise, x_0 = q (q^-1 mod p) r_p +
 * p (p^-1 mod q) r_q mod N, then the same keystream as encryption (for the
 * variant the cumulative one: reading Q33 -- the paper's "same decryption
 * stage leads to m_i ^ S0" omits the cumulative terms).
 * p_dev, q_dev: primes = 3 (mod 4), p != q, p q < 2^63; c_dev, y_dev as
 * produced by prng_cbg_encrypt; m_dev out.  status_dev (may be NULL): 0 ok,
 * 1 invalid key or y >= N (no plaintext written). */
CIPRNG_API int prng_cbg_decrypt(int chaotic, uint64_t n_msgs, uint64_t L, const uint64_t *p_dev,
                                const uint64_t *q_dev, const uint32_t *S0_dev, const uint8_t *c_dev,
                                const uint64_t *y_dev, uint8_t *m_dev, uint32_t *status_dev, void *stream);

/* ---------------------------------------------------------------------- */
/* Algorithm 1 and the chaos / uniformity checks    */
/* ---------------------------------------------------------------------- */

/* Algorithm 1 "PRNG with chaotic functions" on n_streams
 * independent streams, n_out calls each (reading Q34): per call
 * k = b + XORshift(b), then k + 1 single-cell updates x <- F_f(s, x) with
 * s = XORshift(n) (cells 1..n = bits 0..n-1; F_f replaces bit s-1 of x by
 * bit s-1 of f(x), Def. 1); XORshift(m) = 1 + (Alg. 2 xorshift32() mod m)
 * from the stream's state z, drawn in program order.
 *   f_dev    NULL = vectorial negation (n <= 32), else 2^n u32 table f(x)
 *            (n <= 16), entries < 2^n
 *   z_dev, x_dev [n_streams] u32 xorshift32 states (non-zero) and
 *            configurations, advanced in place
 *   out_dev  [n_streams][n_out] u32: the configuration returned by each call
 * Errors: PRNG_EINVAL (n, b == 0, NULL), PRNG_ESIZE, PRNG_ECUDA. */
CIPRNG_API int prng_alg1_generate(const uint32_t *f_dev, uint32_t n, uint32_t b, uint32_t *z_dev, uint32_t *x_dev,
                                  uint64_t n_streams, uint64_t n_out, uint32_t *out_dev, void *stream);

/* Theorems 1 and 2 for f: B^n -> B^n, n <= 16 (f_dev as above,
 * NULL = negation).  Writes report_dev[3] (u64): [0] vertices of the
 * iteration graph Gamma(f) reachable from 0, [1] vertices from which 0 is
 * reachable, [2] vertices whose in- and out-degree (non-loop arcs) differ.
 * G_f is chaotic (Devaney) iff Gamma(f) is strongly connected iff
 * [0] == [1] == 2^n; the Markov matrix M of Theorem 2 is doubly stochastic
 * iff [2] == 0.  scratch_dev: 2^n bytes, caller-owned.  One CTA;
 * level-synchronous breadth-first search. */
CIPRNG_API int prng_gamma_check(const uint32_t *f_dev, uint32_t n, uint8_t *scratch_dev, uint64_t *report_dev,
                                void *stream);

/* ---------------------------------------------------------------------- */
/* Introspection, checkpoint / test hooks                                 */
/* ---------------------------------------------------------------------- */

typedef struct prng_info_t {
    int32_t variant;
    uint32_t comb_size;
    uint64_t seed, first_stream, n_local;
    uint32_t state_words; /* u32 planes per stream (V0 23, V1 6, V2 18, V3 4, V4 24) */
    int32_t device;
    int32_t store_path;   /* path used by the last prng_generate */
    uint32_t kernel_launches; /* kernels launched by the last call */
} prng_info_t;

CIPRNG_API int prng_get_info(const prng_t *h, prng_info_t *info);

/* State layout (SoA u32 planes; plane k of local stream s at word
 * k*n_local + s):
 *  V0 (23): a.lo a.hi | b0.lo b0.hi .. b3.lo b3.hi | c0.lo c0.hi .. c4.lo c4.hi
 *           | d.lo d.hi | x        (xor64 a; xor128 b; xorwow c and Weyl d)
 *  V1 (6):  xor128 x y z w | x | tp  (tp = this stream's shared cell, Q8)
 *  V2 (18): y1..y8 (BBS states) | m1..m8 (index of each instance's modulus
 *           in the ascending table of the 78 products p*q, p < q primes = 3
 *           mod 4 in [128, 256], Q13) | x | tp
 *  V3 (4):  a.lo a.hi (xor64) | x | tp
 *  V4 (24): V0's 22 generator words | x | tp
 * get/set copy exactly state_words*n_local*4 bytes (else PRNG_ESTATE) and
 * synchronise the device.  set_state validates the content on the host
 * before any copy and returns PRNG_ESTATE (device state untouched) if a V2
 * modulus index m_j >= 78, a V2 state y_j >= its modulus, or any
 * xorshift-family generator of V0/V1/V3/V4 is all zero (a fixed point).  set_state is the checkpoint-resume hook (P:905:
 * the state written back after every kernel is a checkpoint). */
CIPRNG_API int prng_get_state(const prng_t *h, void *host_buf, size_t bytes);
CIPRNG_API int prng_set_state(prng_t *h, const void *host_buf, size_t bytes);

CIPRNG_API const char *prng_strerror(int status);
CIPRNG_API const char *prng_last_cuda_error(void);

/* Host-side exhaustive self-check of the kernels' division-free BBS squarings
 * (P:1209-1211 asks for 32-bit modulus arithmetic only): for every modulus
 * of the table and every y < M, compares Barrett (IMAD.HI quotient), the
 * FP32-quotient form (host emulation of its round-toward-zero steps) and the
 * Montgomery form (entry y*2^32 mod M, one REDC squaring, canonical exit)
 * with y*y % M, and checks the table's derived words (2^32 - M, K, -M^-1).
 * Writes the number of mismatches; runs on the CPU (no GPU). */
CIPRNG_API int prng_selftest_modsq(uint64_t *mismatches);

/* The same exhaustive check executed by a kernel on the current device (the
 * FP32 rounding itself is then the hardware's).  Synchronous; allocates and
 * frees its own device buffers.  Returns PRNG_ECUDA on a CUDA failure (e.g.
 * no GPU), PRNG_EINVAL for a null pointer. */
CIPRNG_API int prng_selftest_modsq_gpu(uint64_t *mismatches);

/* Host-only self-test of the single-stream jump-ahead (PRNG_STORE_JUMP): the
 * minimal polynomials of Listing 1's three generators (xor64, xor128 and
 * xorwow on 64-bit words) and, from seeded states, the state J
 * steps ahead as sum_i c_i S_i (c = z^J mod m) against J plain steps.
 * *mismatches = 0 when every check holds; degrees[3] = the three minimal
 * polynomials' degrees.  No GPU needed. */
CIPRNG_API int prng_selftest_jump(uint64_t *mismatches, uint32_t *degrees);

/* Library build string (compiler, arch). */
CIPRNG_API const char *prng_version(void);

#ifdef __cplusplus
}
#endif

#endif /* CIPRNG_H */
