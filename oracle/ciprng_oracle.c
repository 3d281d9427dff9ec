/*
 * ciprng_oracle.c -- the CPU ORACLE for the chaotic-iteration PRNG hot path
 * of arXiv 1112.5239 (Bahi, Couturier, Guyeux, Heam).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_1112_5239_b200/) never links, imports or calls it,
 * and this file shares no code, header, table or constant generator with the
 * CUDA path: every constant below is re-derived here from the paper or from
 * the DESIGN.md reading it cites.
 *
 * Plain, slow, obviously-correct C99: scalar, single-threaded, no blocking,
 * no fusion, no intrinsics.  Rounds of the neighbour-combined variants are
 * simulated group by group in lockstep, in the order the paper's pseudocode
 * states them.
 *
 * Citations: "P:a-b" = /root/reference/PAPER.md lines a-b; "S:a-b" = SPEC.md;
 * "Qn" = reading n of the ambiguity ledger (restated in
 * DESIGN.md s3).
 *
 * Pinning (what fixes each function other than itself; tests/test_oracle_pins.py):
 *   orc_xor_step          Table 1, P:799-815 (paper's worked example)
 *   orc_xorshift32        Alg. 2; Marsaglia's published example
 *   orc_xor64             Marsaglia 2003 published first output (cited P:845)
 *   orc_xor128_32         Marsaglia 2003 published first output (cited P:951)
 *   orc_xor128_64/xorwow_64  hand-traced tiny-state steps (tests/golden/)
 *   orc_splitmix_word     published SplitMix64 sequence (Q11)
 *   orc_v0_*              hand-traced first output from a tiny state
 *   orc_v1_*              hand-traced C=2 lockstep trace (S:355 tables),
 *                         invariants I1 (prefix-XOR), I2 (self-cancel),
 *                         I3 (group parity), I4 (split invariance)
 *   orc_v2_*              BBS brute force, hand-traced
 *                         C=1 trace, I6 closure, I7 rotation order 8
 *   orc_v3_*, orc_v4_*    (NEXT-1) I2 self-cancel => prefix-XOR of the
 *                         published xor64 / pinned Listing-1 fold, I3 group
 *                         parity, single-cell injection, hand-traced C=2
 *   orc_stats_words       brute-force recount on tiny inputs; pi estimate
 *   orc_digest_words      a verification hash defined by this build (Q28):
 *                         single pairs pinned to the published SplitMix64
 *                         sequence (h = output P of SplitMix64 seeded with
 *                         the pair); shard additivity, injectivity
 *   orc_v*_init_words     word -> state mapping checked field by field
 *   (seeders)             against the published SplitMix64 generator (Q11);
 *                         zero guards reached by injected words and tied to
 *                         Marsaglia's published first outputs; V2 seeds
 *                         recomputed from the words (Q21 incl. the
 *                         rejection loop, reached by injection) and each
 *                         y_j a quadratic residue mod both prime factors
 *                         (Euler's criterion; BBS seeds are squares,
 *                         P:1203-1206)
 *   comb/modulus tables   the CHOICE of seeder and default arrays is this
 *                         build's (Q6, Q11, Q13); the modulus table is pinned
 *                         to P:1212-1214's constraints (primes = 3 mod 4,
 *                         M < 2^16).
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>
#include <stdlib.h>

#define ORC_OK 0
#define ORC_EINVAL (-1)

/* ------------------------------------------------------------------------ */
/* Eq. "Oplus": x^n = x^{n-1} XOR S^n.  The update of every      */
/* variant.  Table 1 is its worked example.                      */
/* ------------------------------------------------------------------------ */
uint64_t orc_xor_step(uint64_t x, uint64_t s) { return x ^ s; }

/* ------------------------------------------------------------------------ */
/* Alg. 2, "An arbitrary round of XORshift", 32-bit, (13,17,5). */
/* Not on the V0-V2 path under reading Q1; kept as the shift-convention pin. */
/* ------------------------------------------------------------------------ */
uint32_t orc_xorshift32(uint32_t *z)
{
    uint32_t v = *z;
    v = v ^ (v << 13);
    v = v ^ (v >> 17);
    v = v ^ (v << 5);
    *z = v;
    return v;
}

/* ------------------------------------------------------------------------ */
/* The three "classical 64-bits PRNGs" of Listing 1, Marsaglia  */
/* 2003 recurrences on 64-bit words (readings Q1-A, Q2, Q3).                 */
/* ------------------------------------------------------------------------ */

/* xorshift == Marsaglia xor64, triple (13, 7, 17) (Q1 reading A). */
uint64_t orc_xor64(uint64_t *a)
{
    uint64_t v = *a;
    v ^= v << 13;
    v ^= v >> 7;
    v ^= v << 17;
    *a = v;
    return v;
}

/* xor128 on u64 words: t=(x^(x<<11)); x=y; y=z; z=w; w=(w^(w>>19))^(t^(t>>8)) (Q2). */
uint64_t orc_xor128_64(uint64_t b[4])
{
    uint64_t t = b[0] ^ (b[0] << 11);
    b[0] = b[1];
    b[1] = b[2];
    b[2] = b[3];
    b[3] = (b[3] ^ (b[3] >> 19)) ^ (t ^ (t >> 8));
    return b[3];
}

/* xorwow on u64 words: t=(x^(x>>2)); x=y; y=z; z=w; w=v;
 * v=(v^(v<<4))^(t^(t<<1)); return (d+=362437)+v;  (Q2, Q3) */
uint64_t orc_xorwow_64(uint64_t c[5], uint64_t *d)
{
    uint64_t t = c[0] ^ (c[0] >> 2);
    c[0] = c[1];
    c[1] = c[2];
    c[2] = c[3];
    c[3] = c[4];
    c[4] = (c[4] ^ (c[4] << 4)) ^ (t ^ (t << 1));
    *d = *d + 362437u;
    return *d + c[4];
}

/* xor128 with "unsigned longs (64 bits) replaced by unsigned integers (32
 * bits)" -- the strategy source of Alg. 4 (reading Q5). */
uint32_t orc_xor128_32(uint32_t b[4])
{
    uint32_t t = b[0] ^ (b[0] << 11);
    b[0] = b[1];
    b[1] = b[2];
    b[2] = b[3];
    b[3] = (b[3] ^ (b[3] >> 19)) ^ (t ^ (t >> 8));
    return b[3];
}

/* ------------------------------------------------------------------------ */
/* Seeder (reading Q11): replaces the host ISAAC initialisation. */
/* W(seed, s, k) = output number 16*s+k+1 of SplitMix64 started at `seed`.   */
/* ------------------------------------------------------------------------ */
uint64_t orc_mix64(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t orc_splitmix_word(uint64_t seed, uint64_t s, uint32_t k)
{
    uint64_t counter = 16u * s + (uint64_t)k + 1u;
    return orc_mix64(seed + 0x9E3779B97F4A7C15ull * counter);
}

static uint32_t lo32(uint64_t v) { return (uint32_t)(v & 0xFFFFFFFFu); }
static uint32_t hi32(uint64_t v) { return (uint32_t)(v >> 32); }

/* ======================================================================== */
/* V0: Listing 1 run per thread == Alg. 3 "naive" kernel.        */
/* ======================================================================== */
typedef struct {
    uint64_t a;     /* xorshift (xor64) state               */
    uint64_t b[4];  /* xor128 state (x, y, z, w)            */
    uint64_t c[5];  /* xorwow shift registers (x, y, z, w, v) */
    uint64_t d;     /* xorwow Weyl counter                  */
    uint32_t x;     /* chaotic-iteration state       */
    uint32_t pad;   /* always 0                             */
} orc_v0_state;

/* The 16 seeder words of stream s: w[k] = W(seed, s, k) (Q11). */
static void seed_words(uint64_t seed, uint64_t s, uint64_t w[16])
{
    uint32_t k;
    for (k = 0; k < 16; k++) w[k] = orc_splitmix_word(seed, s, k);
}

/* Per-stream initial state from the stream's seeder words w[k] = W(s, k)
 * (Q11, Q12): a = w0, b = w1..w4, c = w5..w9, d = w10, x = lo w11; an
 * all-zero generator state (a fixed point of every xorshift) is replaced by
 * Marsaglia's published seeds.  Split from orc_v0_init_one so that tests can
 * inject words that reach the zero guards. */
void orc_v0_init_words(const uint64_t w[16], orc_v0_state *st)
{
    int k;
    memset(st, 0, sizeof(*st));
    st->a = w[0];
    if (st->a == 0) st->a = 88172645463325252ull;              /* zero is a fixed point */
    for (k = 0; k < 4; k++) st->b[k] = w[1 + k];
    if ((st->b[0] | st->b[1] | st->b[2] | st->b[3]) == 0) {
        st->b[0] = 123456789u; st->b[1] = 362436069u; st->b[2] = 521288629u; st->b[3] = 88675123u;
    }
    for (k = 0; k < 5; k++) st->c[k] = w[5 + k];
    if ((st->c[0] | st->c[1] | st->c[2] | st->c[3] | st->c[4]) == 0) {
        st->c[0] = 123456789u; st->c[1] = 362436069u; st->c[2] = 521288629u; st->c[3] = 88675123u;
        st->c[4] = 5783321u;
    }
    st->d = w[10];
    st->x = lo32(w[11]);
}

/* paper_defaults reproduces Listing 1 (x = 123123123) with
 * Marsaglia's published seeds. */
void orc_v0_init_one(uint64_t seed, uint64_t s, int paper_defaults, orc_v0_state *st)
{
    uint64_t w[16];
    if (paper_defaults) {
        memset(st, 0, sizeof(*st));
        st->a = 88172645463325252ull;
        st->b[0] = 123456789u; st->b[1] = 362436069u; st->b[2] = 521288629u; st->b[3] = 88675123u;
        st->c[0] = 123456789u; st->c[1] = 362436069u; st->c[2] = 521288629u; st->c[3] = 88675123u;
        st->c[4] = 5783321u;
        st->d = 6615241u;
        st->x = 123123123u;
        return;
    }
    seed_words(seed, s, w);
    orc_v0_init_words(w, st);
}

/* One call of Listing 1: returns the new x. */
uint32_t orc_v0_next(orc_v0_state *st)
{
    uint64_t t1 = orc_xor64(&st->a);
    uint64_t t2 = orc_xor128_64(st->b);
    uint64_t t3 = orc_xorwow_64(st->c, &st->d);
    uint32_t x = st->x;
    x = x ^ lo32(t1);
    x = x ^ hi32(t2);
    x = x ^ hi32(t3);
    x = x ^ lo32(t2);
    x = x ^ hi32(t1);
    x = x ^ lo32(t3);
    st->x = x;
    return x;
}

/* ======================================================================== */
/* V1: Alg. 4 "improved" kernel, lockstep two-phase (Q7).        */
/* ======================================================================== */
typedef struct {
    uint32_t g[4];  /* xor128-32 state (x, y, z, w) */
    uint32_t x;     /* chaotic-iteration state       */
    uint32_t tp;    /* this thread's shared cell: previous round's t (Q8) */
} orc_v1_state;

/* V1 state from the seeder words: xor128 (a,b,c,d) = lo w0..w3 (all zero ->
 * Marsaglia's seeds), x = lo w4, tp = lo w5 (Q8, Q11). */
void orc_v1_init_words(const uint64_t w[16], orc_v1_state *st)
{
    int k;
    for (k = 0; k < 4; k++) st->g[k] = lo32(w[k]);
    if ((st->g[0] | st->g[1] | st->g[2] | st->g[3]) == 0) {
        st->g[0] = 123456789u; st->g[1] = 362436069u; st->g[2] = 521288629u; st->g[3] = 88675123u;
    }
    st->x = lo32(w[4]);
    st->tp = lo32(w[5]);
}

void orc_v1_init_one(uint64_t seed, uint64_t s, orc_v1_state *st)
{
    uint64_t w[16];
    seed_words(seed, s, w);
    orc_v1_init_words(w, st);
}

/* ======================================================================== */
/* V2: Alg. 5 BBS kernel.                                      */
/* ======================================================================== */
typedef struct {
    uint32_t y[8];  /* BBS internal states bbs1..bbs8                 */
    uint32_t m[8];  /* index of each instance's modulus in orc_moduli */
    uint32_t x;     /* chaotic-iteration state                        */
    uint32_t tp;    /* shared cell (previous round's t)               */
} orc_v2_state;

/* Modulus table (Q13): "prime numbers around 256 that are congruent to 3
 * modulus 4" with M = p*q < 2^16.  Primes p = 3 mod 4 in
 * [128, 256]; all products p < q, ascending. */
static uint32_t orc_moduli_tab[128];
static int orc_moduli_n = 0;

static int is_prime(uint32_t v)
{
    uint32_t d;
    if (v < 2) return 0;
    for (d = 2; d * d <= v; d++)
        if (v % d == 0) return 0;
    return 1;
}

static void build_moduli(void)
{
    uint32_t primes[64];
    int np = 0, i, j, n = 0;
    uint32_t v;
    if (orc_moduli_n) return;
    for (v = 128; v <= 256; v++)
        if (is_prime(v) && v % 4 == 3) primes[np++] = v;
    for (i = 0; i < np; i++)
        for (j = i + 1; j < np; j++) orc_moduli_tab[n++] = primes[i] * primes[j];
    /* insertion sort, ascending */
    for (i = 1; i < n; i++) {
        uint32_t key = orc_moduli_tab[i];
        j = i - 1;
        while (j >= 0 && orc_moduli_tab[j] > key) { orc_moduli_tab[j + 1] = orc_moduli_tab[j]; j--; }
        orc_moduli_tab[j + 1] = key;
    }
    orc_moduli_n = n;
}

int orc_moduli(uint32_t *out, int cap)
{
    int i;
    build_moduli();
    for (i = 0; i < orc_moduli_n && i < cap; i++) out[i] = orc_moduli_tab[i];
    return orc_moduli_n;
}

static uint32_t gcd32(uint32_t a, uint32_t b)
{
    while (b) { uint32_t t = a % b; a = b; b = t; }
    return a;
}

/* One BBS step x_{n+1} = x_n^2 mod M; x < M < 2^16 so x^2 < 2^32. */
uint32_t orc_bbs_step(uint32_t y, uint32_t M) { return (y * y) % M; }

/* Q21 seed from the seeder words: instance j takes modulus index
 * m_j = hi(w_j) mod 78 and r = 2 + lo(w_j) mod (M-3), stepped (wrapping to
 * 2) until gcd(r, M) = 1 and r^2 mod M > 1; its state is the quadratic
 * residue y_j = r^2 mod M (BBS seeds are squares; cf. the
 * x_0 = r^2 mod N of P:1344).  x = lo w8, tp = lo w9. */
void orc_v2_init_words(const uint64_t w[16], orc_v2_state *st)
{
    int j;
    build_moduli();
    for (j = 0; j < 8; j++) {
        uint32_t mi = hi32(w[j]) % (uint32_t)orc_moduli_n;
        uint32_t M = orc_moduli_tab[mi];
        uint32_t r = 2u + lo32(w[j]) % (M - 3u);
        while (gcd32(r, M) != 1u || (r * r) % M <= 1u) r = (r == M - 2u) ? 2u : r + 1u;
        st->y[j] = (r * r) % M;
        st->m[j] = mi;
    }
    st->x = lo32(w[8]);
    st->tp = lo32(w[9]);
}

void orc_v2_init_one(uint64_t seed, uint64_t s, orc_v2_state *st)
{
    uint64_t w[16];
    seed_words(seed, s, w);
    orc_v2_init_words(w, st);
}

/* ======================================================================== */
/* V3 and V4: Alg. 4's neighbour combination          */
/* with other strategy sources.                                  */
/*  V3: the xor64 of the paper's "optimized versions" ("the    */
/*      optimized versions use the xor64 described in [Marsaglia2003]").    */
/*      Reading Q29: Alg. 4's t is 32-bit ("a 32-bits xor-like PRNG */
/*      has been chosen"), so t = xor64() is C's conversion of the 64-bit   */
/*      output: its low 32 bits.                                            */
/*  V4: Listing 1's three generators and six-word fold as the  */
/*      source: t = lo(t1)^hi(t2)^hi(t3)^lo(t2)^hi(t1)^lo(t3) (reading Q30). */
/* ======================================================================== */
typedef struct {
    uint64_t a;     /* xor64 state                            */
    uint32_t x;     /* chaotic-iteration state                */
    uint32_t tp;    /* shared cell: previous round's t (Q8)   */
} orc_v3_state;

typedef struct {
    uint64_t a;     /* xorshift (xor64) state                 */
    uint64_t b[4];  /* xor128 state                           */
    uint64_t c[5];  /* xorwow shift registers                 */
    uint64_t d;     /* xorwow Weyl counter                    */
    uint32_t x;     /* chaotic-iteration state                */
    uint32_t tp;    /* shared cell                            */
} orc_v4_state;

/* Seeds (Q11 extended): V3 a = W(s,0) (0 -> Marsaglia's 88172645463325252),
 * x = lo W(s,1), tp = lo W(s,2).  V4: the generator words exactly as V0
 * (W(s,0..10) with V0's zero guards), x = lo W(s,11), tp = lo W(s,12). */
void orc_v3_init_words(const uint64_t w[16], orc_v3_state *st)
{
    st->a = w[0];
    if (st->a == 0) st->a = 88172645463325252ull;
    st->x = lo32(w[1]);
    st->tp = lo32(w[2]);
}

void orc_v3_init_one(uint64_t seed, uint64_t s, orc_v3_state *st)
{
    uint64_t w[16];
    seed_words(seed, s, w);
    orc_v3_init_words(w, st);
}

void orc_v4_init_words(const uint64_t w[16], orc_v4_state *st)
{
    orc_v0_state g;
    int k;
    orc_v0_init_words(w, &g);
    st->a = g.a;
    for (k = 0; k < 4; k++) st->b[k] = g.b[k];
    for (k = 0; k < 5; k++) st->c[k] = g.c[k];
    st->d = g.d;
    st->x = lo32(w[11]);
    st->tp = lo32(w[12]);
}

void orc_v4_init_one(uint64_t seed, uint64_t s, orc_v4_state *st)
{
    uint64_t w[16];
    seed_words(seed, s, w);
    orc_v4_init_words(w, st);
}

/* The strategy draws ("t = xor-like()"). */
uint32_t orc_v3_draw(orc_v3_state *st) { return lo32(orc_xor64(&st->a)); }

uint32_t orc_v4_draw(orc_v4_state *st)
{
    uint64_t t1 = orc_xor64(&st->a);
    uint64_t t2 = orc_xor128_64(st->b);
    uint64_t t3 = orc_xorwow_64(st->c, &st->d);
    return lo32(t1) ^ hi32(t2) ^ hi32(t3) ^ lo32(t2) ^ hi32(t1) ^ lo32(t3);
}

/* ======================================================================== */
/* Grid-level entry points (the oracle's mirror of the C-ABI).              */
/* variant: 0 = V0, 1 = V1, 2 = V2.  states: array of n_local per-stream    */
/* structs of the variant's type.  Output is stream-major out[s*n + i] (Q9). */
/* ======================================================================== */
size_t orc_state_size(int variant)
{
    if (variant == 0) return sizeof(orc_v0_state);
    if (variant == 1) return sizeof(orc_v1_state);
    if (variant == 2) return sizeof(orc_v2_state);
    if (variant == 3) return sizeof(orc_v3_state);
    if (variant == 4) return sizeof(orc_v4_state);
    return 0;
}

int orc_grid_init(int variant, uint64_t seed, uint64_t first_stream, uint64_t n_local,
                  int paper_defaults, void *states)
{
    uint64_t s;
    if (variant == 0) {
        orc_v0_state *st = (orc_v0_state *)states;
        if (paper_defaults && !(first_stream == 0 && n_local == 1)) return ORC_EINVAL;
        for (s = 0; s < n_local; s++) orc_v0_init_one(seed, first_stream + s, paper_defaults, &st[s]);
        return ORC_OK;
    }
    if (paper_defaults) return ORC_EINVAL;
    if (variant == 1) {
        orc_v1_state *st = (orc_v1_state *)states;
        for (s = 0; s < n_local; s++) orc_v1_init_one(seed, first_stream + s, &st[s]);
        return ORC_OK;
    }
    if (variant == 2) {
        orc_v2_state *st = (orc_v2_state *)states;
        for (s = 0; s < n_local; s++) orc_v2_init_one(seed, first_stream + s, &st[s]);
        return ORC_OK;
    }
    if (variant == 3) {
        orc_v3_state *st = (orc_v3_state *)states;
        for (s = 0; s < n_local; s++) orc_v3_init_one(seed, first_stream + s, &st[s]);
        return ORC_OK;
    }
    if (variant == 4) {
        orc_v4_state *st = (orc_v4_state *)states;
        for (s = 0; s < n_local; s++) orc_v4_init_one(seed, first_stream + s, &st[s]);
        return ORC_OK;
    }
    return ORC_EINVAL;
}

/* Test hook: one stream's state from 16 injected seeder words (the word ->
 * state mapping of Q11/Q21 without the SplitMix64 step), so that pins can
 * reach the zero guards and the Q21 rejection loop. */
int orc_init_from_words(int variant, const uint64_t *w, void *state)
{
    if (!w || !state) return ORC_EINVAL;
    if (variant == 0) { orc_v0_init_words(w, (orc_v0_state *)state); return ORC_OK; }
    if (variant == 1) { orc_v1_init_words(w, (orc_v1_state *)state); return ORC_OK; }
    if (variant == 2) { orc_v2_init_words(w, (orc_v2_state *)state); return ORC_OK; }
    if (variant == 3) { orc_v3_init_words(w, (orc_v3_state *)state); return ORC_OK; }
    if (variant == 4) { orc_v4_init_words(w, (orc_v4_state *)state); return ORC_OK; }
    return ORC_EINVAL;
}

/* Default combination arrays for C = 32 (reading Q6): the paper never prints
 * array_comb1/2 or the 16 BBS arrangement arrays. */
static void default_comb_v1(uint32_t l, uint32_t *c1, uint32_t *c2)
{
    *c1 = (l + 1u) % 32u;
    *c2 = (l + 17u) % 32u;
}

static uint32_t default_comb_v2(uint32_t a, uint32_t l)
{
    if (a < 8u) return (l + 1u + a) % 32u;
    return (l + 17u + (a - 8u)) % 32u;
}

/* V0 generate: each stream runs Listing 1 n times (Alg. 3). */
static void v0_generate(orc_v0_state *st, uint64_t n_local, uint64_t n, uint32_t *out)
{
    uint64_t s, i;
    for (s = 0; s < n_local; s++)
        for (i = 0; i < n; i++) out[s * n + i] = orc_v0_next(&st[s]);
}

/* V1 generate (Alg. 4), per group of C streams, lockstep:
 *   offset = threadIdx % C; o1 = threadIdx - offset + array_comb1[offset];
 *   o2 likewise with array_comb2;
 *   per round: t = xor-like(); t ^= shmem[o1] ^ shmem[o2]; shmem[tid] = t;
 *   x ^= t; store x.
 * Two-phase (Q7): every lane reads the previous round's shmem before any
 * lane writes. */
static int v1_generate(orc_v1_state *st, uint64_t n_local, uint32_t C, const uint8_t *comb,
                       uint64_t n, uint32_t *out)
{
    uint64_t g0, i;
    uint32_t l;
    uint32_t gval[32], tnew[32], o1[32], o2[32];
    if (C == 0 || C > 32 || n_local % C) return ORC_EINVAL;
    if (comb == NULL && C != 32) return ORC_EINVAL;
    for (l = 0; l < C; l++) {
        if (comb) { o1[l] = comb[l]; o2[l] = comb[C + l]; }
        else default_comb_v1(l, &o1[l], &o2[l]);
        if (o1[l] >= C || o2[l] >= C) return ORC_EINVAL;
    }
    for (g0 = 0; g0 < n_local; g0 += C) {
        orc_v1_state *grp = &st[g0];
        for (i = 0; i < n; i++) {
            /* phase 1: every thread draws its xor-like number */
            for (l = 0; l < C; l++) gval[l] = orc_xor128_32(grp[l].g);
            /* phase 2: combine with the previous round's shared cells */
            for (l = 0; l < C; l++) tnew[l] = gval[l] ^ grp[o1[l]].tp ^ grp[o2[l]].tp;
            /* phase 3: commit shared cells, chaotic-iteration update, store */
            for (l = 0; l < C; l++) {
                grp[l].tp = tnew[l];
                grp[l].x = orc_xor_step(grp[l].x, tnew[l]);
                out[(g0 + l) * n + i] = grp[l].x;
            }
        }
    }
    return ORC_OK;
}

/* V2 generate (Alg. 5), per group of C streams, lockstep.
 * o1, o2 chosen once per call from the call-entry states of bbs1, bbs2
 * (Q15: array_comb[8 + (bbs2 & 7)], Q16).  Per round: 8 squarings give 8
 * nibbles; bbs3 and bbs7 give two shifts of at most 3 bits,
 * filled with exactly `shift` low bits of new bbs1 / bbs2 draws
 * (Q17, Q18); then the combination and update as in V1.
 * At the end of the call the 8 (state, modulus) pairs rotate: instance j
 * is stored in place j+1, instance 8 in place 1 (Q19, Q20). */
static int v2_generate(orc_v2_state *st, uint64_t n_local, uint32_t C, const uint8_t *comb,
                       uint64_t n, uint32_t *out)
{
    static const uint32_t array_shift[4] = {0u, 1u, 3u, 7u};
    uint64_t g0, i;
    uint32_t l, a;
    uint32_t tnew[32], o1[32], o2[32];
    uint32_t tab[16][32];
    build_moduli();
    if (C == 0 || C > 32 || n_local % C) return ORC_EINVAL;
    if (comb == NULL && C != 32) return ORC_EINVAL;
    for (a = 0; a < 16; a++)
        for (l = 0; l < C; l++) {
            tab[a][l] = comb ? comb[a * C + l] : default_comb_v2(a, l);
            if (tab[a][l] >= C) return ORC_EINVAL;
        }
    if (n == 0) return ORC_OK; /* no launch, no rotation (Q20) */
    for (g0 = 0; g0 < n_local; g0 += C) {
        orc_v2_state *grp = &st[g0];
        for (l = 0; l < C; l++) {
            o1[l] = tab[grp[l].y[0] & 7u][l];
            o2[l] = tab[8u + (grp[l].y[1] & 7u)][l];
        }
        for (i = 0; i < n; i++) {
            for (l = 0; l < C; l++) {
                orc_v2_state *p = &grp[l];
                uint32_t t = 0, shift, j;
                for (j = 0; j < 8; j++) {
                    p->y[j] = orc_bbs_step(p->y[j], orc_moduli_tab[p->m[j]]);
                    t = (t << 4) | (p->y[j] & 15u);
                }
                p->y[2] = orc_bbs_step(p->y[2], orc_moduli_tab[p->m[2]]);
                shift = p->y[2] & 3u;
                t = t << shift;
                p->y[0] = orc_bbs_step(p->y[0], orc_moduli_tab[p->m[0]]);
                t = t | (p->y[0] & array_shift[shift]);
                p->y[6] = orc_bbs_step(p->y[6], orc_moduli_tab[p->m[6]]);
                shift = p->y[6] & 3u;
                t = t << shift;
                p->y[1] = orc_bbs_step(p->y[1], orc_moduli_tab[p->m[1]]);
                t = t | (p->y[1] & array_shift[shift]);
                tnew[l] = t;
            }
            for (l = 0; l < C; l++) tnew[l] = tnew[l] ^ grp[o1[l]].tp ^ grp[o2[l]].tp;
            for (l = 0; l < C; l++) {
                grp[l].tp = tnew[l];
                grp[l].x = orc_xor_step(grp[l].x, tnew[l]);
                out[(g0 + l) * n + i] = grp[l].x;
            }
        }
        /* rotation: place j+1 <- instance j, place 1 <- instance 8 */
        for (l = 0; l < C; l++) {
            orc_v2_state *p = &grp[l];
            uint32_t y7 = p->y[7], m7 = p->m[7];
            int j;
            for (j = 7; j > 0; j--) { p->y[j] = p->y[j - 1]; p->m[j] = p->m[j - 1]; }
            p->y[0] = y7;
            p->m[0] = m7;
        }
    }
    return ORC_OK;
}

/* V3 / V4 generate: Alg. 4 exactly as v1_generate above (same default
 * arrays, Q6; same two-phase lockstep, Q7), only the draw of phase 1 comes
 * from the variant's source. */
static int v34_generate(int variant, void *states, uint64_t n_local, uint32_t C, const uint8_t *comb,
                        uint64_t n, uint32_t *out)
{
    uint64_t g0, i;
    uint32_t l;
    uint32_t gval[32], tnew[32], o1[32], o2[32];
    orc_v3_state *s3 = (orc_v3_state *)states;
    orc_v4_state *s4 = (orc_v4_state *)states;
    if (C == 0 || C > 32 || n_local % C) return ORC_EINVAL;
    if (comb == NULL && C != 32) return ORC_EINVAL;
    for (l = 0; l < C; l++) {
        if (comb) { o1[l] = comb[l]; o2[l] = comb[C + l]; }
        else default_comb_v1(l, &o1[l], &o2[l]);
        if (o1[l] >= C || o2[l] >= C) return ORC_EINVAL;
    }
    for (g0 = 0; g0 < n_local; g0 += C) {
        for (i = 0; i < n; i++) {
            /* phase 1: every thread draws its strategy source */
            for (l = 0; l < C; l++)
                gval[l] = variant == 3 ? orc_v3_draw(&s3[g0 + l]) : orc_v4_draw(&s4[g0 + l]);
            /* phase 2: combine with the previous round's shared cells */
            for (l = 0; l < C; l++) {
                uint32_t tp1 = variant == 3 ? s3[g0 + o1[l]].tp : s4[g0 + o1[l]].tp;
                uint32_t tp2 = variant == 3 ? s3[g0 + o2[l]].tp : s4[g0 + o2[l]].tp;
                tnew[l] = gval[l] ^ tp1 ^ tp2;
            }
            /* phase 3: commit shared cells, chaotic-iteration update, store */
            for (l = 0; l < C; l++) {
                uint32_t *tp = variant == 3 ? &s3[g0 + l].tp : &s4[g0 + l].tp;
                uint32_t *x = variant == 3 ? &s3[g0 + l].x : &s4[g0 + l].x;
                *tp = tnew[l];
                *x = orc_xor_step(*x, tnew[l]);
                out[(g0 + l) * n + i] = *x;
            }
        }
    }
    return ORC_OK;
}

int orc_grid_generate(int variant, void *states, uint64_t n_local, uint32_t C,
                      const uint8_t *comb, uint64_t n, uint32_t *out)
{
    if (variant == 0) { v0_generate((orc_v0_state *)states, n_local, n, out); return ORC_OK; }
    if (variant == 1) return v1_generate((orc_v1_state *)states, n_local, C, comb, n, out);
    if (variant == 2) return v2_generate((orc_v2_state *)states, n_local, C, comb, n, out);
    if (variant == 3 || variant == 4) return v34_generate(variant, states, n_local, C, comb, n, out);
    return ORC_EINVAL;
}

/* ======================================================================== */
/* Consumer statistics (reading Q24; the paper only says numbers can be      */
/* "consumed directly after generation").                       */
/* stats[0] += #pairs with u^2 + v^2 < 2^64, u = x_{2k}, v = x_{2k+1} of one */
/* stream within one call; stats[1] += #pairs; stats[2 + (x >> 24)] += 1.    */
/* ======================================================================== */
int orc_stats_words(const uint32_t *out, uint64_t n_local, uint64_t n, uint64_t *stats)
{
    uint64_t s, i;
    if (n % 2) return ORC_EINVAL;
    for (s = 0; s < n_local; s++) {
        for (i = 0; i < n; i++) stats[2 + (out[s * n + i] >> 24)] += 1;
        for (i = 0; i + 1 < n; i += 2) {
            uint64_t u = out[s * n + i], v = out[s * n + i + 1];
            uint64_t uu = u * u, vv = v * v;
            stats[1] += 1;
            if (vv <= ~uu) stats[0] += 1; /* u^2 + v^2 <= 2^64 - 1 */
        }
    }
    return ORC_OK;
}

/* ======================================================================== */
/* Statistical battery counts (monobit, */
/* block frequency m = 128, runs, serial 2-bit, byte chi-square, 8-lag       */
/* autocorrelation -- the desk-scale stand-in for the BigCrush runs of       */
/* P:851-853).  Reading Q31: the bit sequence of a stream within one call is  */
/* its words x_0 .. x_{n-1} in round order, each word most significant bit   */
/* first; sequences never continue across streams or calls.  Plain bit-by-  */
/* bit loops.  Accumulated (u64) into stats[264]:                            */
/*   [0] ones            [1] adjacent pairs that differ   [2] adjacent 11    */
/*   [3] pairs 8 apart that differ   [4] sum over 128-bit blocks (4 words at */
/*   round index 4k..4k+3) of (ones in block - 64)^2   [5] number of blocks  */
/*   [6] first bits equal to 1   [7] last bits equal to 1                    */
/*   [8 + b] bytes equal to b over all four bytes of every word              */
/* ======================================================================== */
#define ORC_BATTERY_WORDS 264

static uint32_t bit_at(const uint32_t *w, uint64_t j) /* j-th bit, MSB first */
{
    return (w[j / 32] >> (31u - (uint32_t)(j % 32))) & 1u;
}

int orc_battery_words(const uint32_t *out, uint64_t n_local, uint64_t n, uint64_t *stats)
{
    uint64_t s, j, k;
    for (s = 0; s < n_local; s++) {
        const uint32_t *w = out + s * n;
        uint64_t N = 32u * n;
        if (n == 0) continue;
        for (j = 0; j < N; j++) {
            uint32_t b = bit_at(w, j);
            stats[0] += b;
            if (j + 1 < N) {
                uint32_t c = bit_at(w, j + 1);
                stats[1] += (b != c);
                stats[2] += (b == 1u && c == 1u);
            }
            if (j + 8 < N) stats[3] += (b != bit_at(w, j + 8));
        }
        for (k = 0; k + 4 <= n; k += 4) {
            int64_t ones = 0, d;
            for (j = 32u * k; j < 32u * (k + 4); j++) ones += bit_at(w, j);
            d = ones - 64;
            stats[4] += (uint64_t)(d * d);
            stats[5] += 1;
        }
        stats[6] += bit_at(w, 0);
        stats[7] += bit_at(w, N - 1);
        for (k = 0; k < n; k++) {
            stats[8 + (w[k] & 0xFFu)] += 1;
            stats[8 + ((w[k] >> 8) & 0xFFu)] += 1;
            stats[8 + ((w[k] >> 16) & 0xFFu)] += 1;
            stats[8 + (w[k] >> 24)] += 1;
        }
    }
    return ORC_OK;
}

/* ======================================================================== */
/* NEXT-3: Blum-Goldwasser and the paper's chaotic variant     */
/* (P:1368-1386), on moduli N < 2^63 (unsigned __int128 products).           */
/* Units are one byte each: bits for classic BG (b_i = lsb x_i),     */
/* blocks of Nb = floor(log2(log2 N)) bits for the variant (P:1371-1372;     */
/* reading Q33: b_i = x_i mod 2^Nb, c_i = m_i ^ (b_0 ^ .. ^ b_i) ^ S0,       */
/* decryption with the same cumulative keystream).                          */
/* ======================================================================== */
uint64_t orc_modmul(uint64_t a, uint64_t b, uint64_t m)
{
    return (uint64_t)(((unsigned __int128)a * b) % m);
}

uint64_t orc_modpow(uint64_t a, uint64_t e, uint64_t m)
{
    uint64_t r = 1 % m;
    a %= m;
    while (e) {
        if (e & 1u) r = orc_modmul(r, a, m);
        a = orc_modmul(a, a, m);
        e >>= 1;
    }
    return r;
}

/* extended Euclid; ORC_EINVAL if gcd(a, m) != 1 */
int orc_modinv(uint64_t a, uint64_t m, uint64_t *inv)
{
    __int128 t = 0, nt = 1, r = (__int128)m, nr = (__int128)(a % m), q, tmp;
    while (nr != 0) {
        q = r / nr;
        tmp = t - q * nt; t = nt; nt = tmp;
        tmp = r - q * nr; r = nr; nr = tmp;
    }
    if (r != 1) return ORC_EINVAL;
    if (t < 0) t += (__int128)m;
    *inv = (uint64_t)t;
    return ORC_OK;
}

static uint64_t gcd64(uint64_t a, uint64_t b)
{
    while (b) { uint64_t t = a % b; a = b; b = t; }
    return a;
}

/* Nb = floor(log2(log2 N)) = the largest t with N >= 2^(2^t). */
uint32_t orc_bg_unit_bits(uint64_t N)
{
    uint32_t t = 0;
    /* 2^(2^(t+1)) for t + 1 <= 5 fits in 64 bits; N < 2^63 < 2^(2^6) */
    while (t < 5 && N >= (1ull << (1u << (t + 1)))) t++;
    return t;
}

/* chaotic != 0: the variant; else classic BG.  m, c: L units.  Returns
 * ORC_EINVAL if N is even, N < 3, N >= 2^63 or gcd(r, N) != 1 (the paper's
 * r in [1, N] must be a unit, else it leaks a factor). */
int orc_cbg_encrypt(int chaotic, uint64_t N, uint32_t S0, uint64_t r, uint64_t L, const uint8_t *m, uint8_t *c,
                    uint64_t *y)
{
    uint64_t x, i;
    uint32_t Nb = orc_bg_unit_bits(N), mask = (1u << Nb) - 1u, B = 0;
    if (N < 3 || !(N & 1u) || (N >> 63) || gcd64(r % N, N) != 1) return ORC_EINVAL;
    x = orc_modmul(r, r, N);                       /* x_0 = r^2 mod N */
    for (i = 0; i < L; i++) {
        if (chaotic) {
            B ^= (uint32_t)(x & mask);                 /* b_0 ^ ... ^ b_i */
            c[i] = (uint8_t)((m[i] ^ B ^ S0) & mask);
        } else {
            c[i] = (uint8_t)((m[i] ^ (uint32_t)(x & 1u)) & 1u);  /* lsb of x_i */
        }
        x = orc_modmul(x, x, N);                   /* x_{i+1} = x_i^2 mod N */
    }
    *y = x;                                        /* y = x_0^(2^L) mod N */
    return ORC_OK;
}

/* Decryption: r_p = y^(((p+1)/4)^L) mod p, r_q likewise,
 * x_0 = q (q^-1 mod p) r_p + p (p^-1 mod q) r_q mod N, regenerate the
 * keystream.  Exponents are reduced mod p-1 (Fermat). */
int orc_cbg_decrypt(int chaotic, uint64_t p, uint64_t q, uint32_t S0, uint64_t L, const uint8_t *c, uint64_t y,
                    uint8_t *m)
{
    uint64_t N = p * q, ep, eq, rp, rq, ip, iq, x, i;
    uint32_t Nb, mask, B = 0;
    if (p < 3 || q < 3 || p == q || (p & 3u) != 3u || (q & 3u) != 3u) return ORC_EINVAL;
    if ((unsigned __int128)p * q >= ((unsigned __int128)1 << 63) || y >= N) return ORC_EINVAL;
    if (orc_modinv(q % p, p, &iq) || orc_modinv(p % q, q, &ip)) return ORC_EINVAL;
    ep = orc_modpow((p + 1) / 4, L, p - 1);
    eq = orc_modpow((q + 1) / 4, L, q - 1);
    rp = orc_modpow(y % p, ep, p);
    rq = orc_modpow(y % q, eq, q);
    x = (orc_modmul(orc_modmul(q, iq, N), rp, N) + orc_modmul(orc_modmul(p, ip, N), rq, N)) % N;
    Nb = orc_bg_unit_bits(N);
    mask = (1u << Nb) - 1u;
    for (i = 0; i < L; i++) {
        if (chaotic) {
            B ^= (uint32_t)(x & mask);
            m[i] = (uint8_t)((c[i] ^ B ^ S0) & mask);
        } else {
            m[i] = (uint8_t)((c[i] ^ (uint32_t)(x & 1u)) & 1u);
        }
        x = orc_modmul(x, x, N);
    }
    return ORC_OK;
}

/* ======================================================================== */
/* NEXT-4: Algorithm 1 "PRNG with chaotic functions" and the     */
/* chaos / uniformity checks of Theorems 1-2.                   */
/* Reading Q34: cells i in [1, n] are bits i-1; F_f(i, x) replaces bit i-1   */
/* of x by bit i-1 of f(x) (Def. 1); XORshift(m) = 1 + (xorshift32() mod m)  */
/* from Alg. 2's generator, one state per stream, drawn in      */
/* program order (first for k, then one per iteration); k = b + XORshift(b)  */
/* and the loop "for i = 0, ..., k" runs k + 1 iterations.  f = NULL is the  */
/* vectorial negation; otherwise a table of 2^n entries.        */
/* ======================================================================== */
static uint32_t xorshift_range(uint32_t *z, uint32_t m) { return 1u + orc_xorshift32(z) % m; }

static uint32_t apply_single(const uint32_t *f, uint32_t n, uint32_t i, uint32_t x)
{
    uint32_t fx = f ? f[x] : (~x & (n == 32 ? 0xFFFFFFFFu : ((1u << n) - 1u)));
    uint32_t bit = 1u << (i - 1u);
    return (x & ~bit) | (fx & bit);
}

/* One call of Algorithm 1 per stream, repeated n_out times: out[s*n_out + j]
 * is the configuration returned by the j-th call.  z: xorshift32 states,
 * x: configurations (both advanced in place). */
int orc_alg1_generate(const uint32_t *f, uint32_t n, uint32_t b, uint32_t *z, uint32_t *x, uint64_t n_streams,
                      uint64_t n_out, uint32_t *out)
{
    uint64_t s, j;
    uint32_t i, k;
    if (n == 0 || n > 32 || (f && n > 16) || b == 0) return ORC_EINVAL;
    for (s = 0; s < n_streams; s++) {
        for (j = 0; j < n_out; j++) {
            k = b + xorshift_range(&z[s], b);
            for (i = 0; i <= k; i++)
                x[s] = apply_single(f, n, xorshift_range(&z[s], n), x[s]);
            out[s * n_out + j] = x[s];
        }
    }
    return ORC_OK;
}

/* Gamma(f): an arc x -> F_f(i, x) for every cell i.  Counts its
 * strongly connected components (plain iterative Kosaraju over 2^n vertices)
 * and checks Theorem 2's doubly-stochastic condition: with M_ij = Mc_ij / n
 * off the diagonal and M_ii = 1 - (1/n) sum_j Mc_ij, the rows sum to 1 by
 * construction and column j sums to 1 - outdeg(j)/n + indeg(j)/n, so M is
 * doubly stochastic iff every vertex has equal in- and out-degree counting
 * non-loop arcs.  report[0] = #SCC, report[1] = 1 if doubly stochastic,
 * report[2] = #vertices with indeg != outdeg. */
int orc_gamma_check(const uint32_t *f, uint32_t n, uint64_t *report)
{
    uint32_t V, v, i, w, top, cnt = 0;
    uint32_t *order, *stack, *comp, *indeg, *outdeg, *it, nord = 0;
    unsigned char *seen;
    if (n == 0 || n > 16) return ORC_EINVAL;
    V = 1u << n;
    order = (uint32_t *)malloc(V * sizeof(uint32_t));
    stack = (uint32_t *)malloc(V * sizeof(uint32_t));
    comp = (uint32_t *)malloc(V * sizeof(uint32_t));
    indeg = (uint32_t *)calloc(V, sizeof(uint32_t));
    outdeg = (uint32_t *)calloc(V, sizeof(uint32_t));
    it = (uint32_t *)calloc(V, sizeof(uint32_t));
    seen = (unsigned char *)calloc(V, 1);
    for (v = 0; v < V; v++)
        for (i = 1; i <= n; i++) {
            w = apply_single(f, n, i, v);
            if (w != v) { outdeg[v]++; indeg[w]++; }
        }
    /* pass 1: DFS finishing order on Gamma(f) */
    for (v = 0; v < V; v++) {
        if (seen[v]) continue;
        top = 0; stack[top++] = v; seen[v] = 1; it[v] = 1;
        while (top) {
            uint32_t u = stack[top - 1];
            if (it[u] <= n) {
                w = apply_single(f, n, it[u], u);
                it[u]++;
                if (!seen[w]) { seen[w] = 1; it[w] = 1; stack[top++] = w; }
            } else {
                order[nord++] = u;
                top--;
            }
        }
    }
    /* pass 2: DFS on the transpose in reverse finishing order; the transpose
     * arcs into u are found by scanning the n candidate predecessors u with
     * bit i-1 flipped or kept (F_f(i, p) differs from p only in bit i-1). */
    for (v = 0; v < V; v++) comp[v] = 0xFFFFFFFFu;
    while (nord) {
        v = order[--nord];
        if (comp[v] != 0xFFFFFFFFu) continue;
        top = 0; stack[top++] = v; comp[v] = cnt;
        while (top) {
            uint32_t u = stack[--top];
            for (i = 1; i <= n; i++) {
                uint32_t cand[2], c;
                cand[0] = u; cand[1] = u ^ (1u << (i - 1u));
                for (c = 0; c < 2; c++) {
                    uint32_t pz = cand[c];
                    if (apply_single(f, n, i, pz) == u && comp[pz] == 0xFFFFFFFFu) {
                        comp[pz] = cnt;
                        stack[top++] = pz;
                    }
                }
            }
        }
        cnt++;
    }
    report[0] = cnt;
    report[2] = 0;
    for (v = 0; v < V; v++) report[2] += (indeg[v] != outdeg[v]);
    report[1] = report[2] == 0;
    free(order); free(stack); free(comp); free(indeg); free(outdeg); free(it); free(seen);
    return ORC_OK;
}

/* Reachability form of Theorem 1's test, used for GPU parity: report[0] =
 * vertices reachable from vertex 0 in Gamma(f), report[1] = vertices from
 * which vertex 0 is reachable, report[2] = vertices with in-degree !=
 * out-degree (non-loop arcs).  Gamma(f) is strongly connected iff
 * report[0] == report[1] == 2^n; Theorem 2's M is doubly stochastic iff
 * report[2] == 0.  Plain breadth-first search with a queue. */
int orc_gamma_reach(const uint32_t *f, uint32_t n, uint64_t *report)
{
    uint32_t V, v, i, head, tail, dir;
    uint32_t *queue, *indeg, *outdeg;
    unsigned char *seen;
    if (n == 0 || n > 16) return ORC_EINVAL;
    V = 1u << n;
    queue = (uint32_t *)malloc(V * sizeof(uint32_t));
    indeg = (uint32_t *)calloc(V, sizeof(uint32_t));
    outdeg = (uint32_t *)calloc(V, sizeof(uint32_t));
    seen = (unsigned char *)malloc(V);
    for (dir = 0; dir < 2; dir++) {
        memset(seen, 0, V);
        head = tail = 0;
        queue[tail++] = 0;
        seen[0] = 1;
        while (head < tail) {
            uint32_t u = queue[head++];
            for (i = 1; i <= n; i++) {
                if (dir == 0) { /* arcs u -> F_f(i, u) */
                    uint32_t w = apply_single(f, n, i, u);
                    if (!seen[w]) { seen[w] = 1; queue[tail++] = w; }
                } else {        /* arcs p -> u: p in {u, u ^ bit(i-1)} with F_f(i, p) == u */
                    uint32_t cand[2], c;
                    cand[0] = u; cand[1] = u ^ (1u << (i - 1u));
                    for (c = 0; c < 2; c++)
                        if (apply_single(f, n, i, cand[c]) == u && !seen[cand[c]]) {
                            seen[cand[c]] = 1;
                            queue[tail++] = cand[c];
                        }
                }
            }
        }
        report[dir] = tail;
    }
    for (v = 0; v < V; v++)
        for (i = 1; i <= n; i++) {
            uint32_t w = apply_single(f, n, i, v);
            if (w != v) { outdeg[v]++; indeg[w]++; }
        }
    report[2] = 0;
    for (v = 0; v < V; v++) report[2] += (indeg[v] != outdeg[v]);
    free(queue); free(indeg); free(outdeg); free(seen);
    return ORC_OK;
}

/* Verification digest (reading Q28, r2 definition): each stream's row is
 * taken in pairs (x_2j, x_2j+1), the lone last word of an odd row paired
 * with 0, and the digest is the sum mod 2^64 over pairs of
 * orc_mix64((x_2j+1 << 32 | x_2j) + P * 0x9E3779B97F4A7C15), with
 * P = (first_stream + s) * ceil(n / 2) + j -- output number P of SplitMix64
 * seeded with the pair (the finaliser and increment of orc_splitmix_word). */
uint64_t orc_digest_words(const uint32_t *out, uint64_t first_stream, uint64_t n_local, uint64_t n)
{
    uint64_t s, j, acc = 0, hn = (n + 1) / 2;
    for (s = 0; s < n_local; s++)
        for (j = 0; j < hn; j++) {
            uint64_t lo = out[s * n + 2 * j];
            uint64_t hi = (2 * j + 1 < n) ? out[s * n + 2 * j + 1] : 0;
            uint64_t P = (first_stream + s) * hn + j;
            acc += orc_mix64(((hi << 32) | lo) + P * 0x9E3779B97F4A7C15ull);
        }
    return acc;
}
