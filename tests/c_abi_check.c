/* c_abi_check.c -- the C ABI used from plain C99 (no Python, no CUDA API):
 * include/ciprng.h must compile as C, libciprng.so must link and run.
 *
 *   host mode (no GPU): version, every status string, the host self-tests
 *   (exhaustive BBS squaring, jump-ahead algebra), argument errors that are
 *   rejected before any device work.
 *   gpu mode: prng_create / prng_generate_host / prng_emit-free round trip
 *   for V1 and V0 (one stream: the jump-ahead path), checked word for word
 *   against the C oracle (oracle/ciprng_oracle.c, linked as liboracle.so --
 *   test infrastructure; the product library never sees it).
 *
 * Built and run by tests/test_abi.py (host) and tests/test_c_abi_gpu.py.
 * Exit status 0 = every check passed; prints "C ABI OK <mode>". */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "ciprng.h"

/* the oracle's C entry points (oracle/ciprng_oracle.c) */
int orc_grid_init(int variant, uint64_t seed, uint64_t first_stream, uint64_t n_local, int paper_defaults,
                  void *states);
int orc_grid_generate(int variant, void *states, uint64_t n_local, uint32_t C, const uint8_t *comb, uint64_t n,
                      uint32_t *out);

static int failures = 0;
#define CHECK(cond, ...)                      \
    do {                                      \
        if (!(cond)) {                        \
            fprintf(stderr, "FAIL: " __VA_ARGS__); \
            fprintf(stderr, "\n");            \
            ++failures;                       \
        }                                     \
    } while (0)

static int host_checks(void) {
    uint64_t bad = 1;
    uint32_t deg[3] = {0, 0, 0};
    prng_t *h = NULL;
    int st;
    CHECK(prng_version() && strstr(prng_version(), "sm_100a"), "version string");
    for (st = PRNG_OK; st >= PRNG_EIO; --st) CHECK(strcmp(prng_strerror(st), "unknown status") != 0, "strerror %d", st);
    CHECK(prng_selftest_modsq(&bad) == PRNG_OK && bad == 0, "modsq selftest (%llu)", (unsigned long long)bad);
    bad = 1;
    CHECK(prng_selftest_jump(&bad, deg) == PRNG_OK && bad == 0, "jump selftest (%llu)", (unsigned long long)bad);
    CHECK(deg[0] == 64 && deg[1] == 253 && deg[2] == 320, "minimal polynomial degrees %u %u %u", deg[0], deg[1],
          deg[2]);
    /* rejected before touching a device */
    CHECK(prng_create(1, 32, 7, &h) == PRNG_EINVAL && h == NULL, "unknown variant");
    CHECK(prng_create(1, 0, PRNG_V1_XOR128_COMB, &h) == PRNG_EINVAL, "zero streams");
    CHECK(prng_create(1, 33, PRNG_V1_XOR128_COMB, &h) == PRNG_EINVAL, "incomplete group");
    CHECK(prng_create(1, 32, PRNG_V1_XOR128_COMB, NULL) == PRNG_EINVAL, "NULL out");
    CHECK(prng_generate(NULL, 4, NULL, NULL) == PRNG_EINVAL, "NULL handle");
    CHECK(prng_destroy(NULL) == PRNG_OK, "destroy NULL");
    return failures;
}

static int compare_with_oracle(int variant, uint64_t seed, uint64_t S, uint64_t n, int paper_defaults) {
    prng_config cfg;
    prng_t *h = NULL;
    size_t words = (size_t)S * n, k;
    uint32_t *got = malloc(words * 4), *ref = malloc(words * 4);
    void *states = calloc((size_t)S, 24 * 4); /* >= the oracle's largest per-stream struct */
    int call, rc;
    memset(&cfg, 0, sizeof(cfg));
    cfg.paper_defaults = paper_defaults;
    rc = prng_create_shard(seed, 0, S, variant, &cfg, &h);
    CHECK(rc == PRNG_OK, "create V%d: %s", variant, prng_strerror(rc));
    if (rc != PRNG_OK) return failures;
    CHECK(orc_grid_init(variant, seed, 0, S, paper_defaults, states) == 0, "oracle init");
    for (call = 0; call < 2; ++call) {
        rc = prng_generate_host(h, n, got, NULL);
        CHECK(rc == PRNG_OK, "generate_host V%d: %s %s", variant, prng_strerror(rc), prng_last_cuda_error());
        orc_grid_generate(variant, states, S, 32, NULL, n, ref);
        for (k = 0; k < words; ++k)
            if (got[k] != ref[k]) {
                CHECK(0, "V%d call %d word %zu: gpu %u oracle %u", variant, call, k, got[k], ref[k]);
                break;
            }
    }
    prng_destroy(h);
    free(got);
    free(ref);
    free(states);
    return failures;
}

int main(int argc, char **argv) {
    const int gpu = argc > 1 && strcmp(argv[1], "gpu") == 0;
    host_checks();
    if (gpu) {
        compare_with_oracle(PRNG_V1_XOR128_COMB, 0x0123456789ABCDEFull, 4096, 128, 0);
        compare_with_oracle(PRNG_V2_BBS_COMB, 7, 1024, 64, 0);
        compare_with_oracle(PRNG_V0_XORLIKE3, 0, 1, 100000, 1); /* one stream: jump-ahead path */
    }
    if (failures) {
        fprintf(stderr, "%d check(s) failed\n", failures);
        return 1;
    }
    printf("C ABI OK %s\n", gpu ? "gpu" : "host");
    return 0;
}
