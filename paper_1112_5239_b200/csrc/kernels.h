// kernels.h -- host-side launchers of the sm_100a kernels (internal).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

namespace ciprng {

struct GenArgs;

// Words per entry of the V2 modulus table (api.cu modulus_table()).
constexpr int kModWords = 8;

// L2 residency of the handle's state planes (set by api.cu around each
// launch): the state is read and written once per call (48 B/stream for V1)
// while the output streams past it, so it is marked persisting in L2 and the
// output is written evict-first -- across back-to-back calls the state then
// never travels to HBM.  base == nullptr: no window.
struct L2Window {
    void *base = nullptr;
    size_t bytes = 0;
    float hit = 0.f;  // fraction of the window that may persist (carve-out / window)
};
extern thread_local L2Window g_l2win;

// Launch with programmatic stream serialization (see device.cuh pdl_wait);
// falls back to a plain launch when disabled (CIPRNG_PDL=0).
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    unsigned na = 0;
    if (pdl_enabled()) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (g_l2win.base != nullptr) {
        at[na].id = cudaLaunchAttributeAccessPolicyWindow;
        at[na].val.accessPolicyWindow.base_ptr = g_l2win.base;
        at[na].val.accessPolicyWindow.num_bytes = g_l2win.bytes;
        at[na].val.accessPolicyWindow.hitRatio = g_l2win.hit;
        at[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        at[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Blocks of `kern` that are resident at once on the device (occupancy x SMs):
// the unit of the consumer / battery grids (persistent_grid below; sized from
// the occupancy API because registers limit the consumer to 7 CTAs/SM).
int resident_blocks(const void *kern, int threads, size_t smem);
// True when the current device reserves exactly StatsSinkCta::kResv (1 KiB)
// of shared memory per block, i.e. dynamic shared memory starts at window
// offset 0x400 as the CTA-histogram consumers' immediate-offset atomics assume.
constexpr int kCtaHistResvBytes = 1024;
bool cta_hist_ok();
// Grid of the per-warp-histogram consumer / battery kernels (V0, V2, the
// general kernels; the CTA-histogram ones use launch_cta_hist below): k
// waves of resident CTAs (k = 0:
// one tile per warp, no cap; CIPRNG_NVCC_EXTRA=-DCIPRNG_PGRID_WAVES=k for
// experiments).  Measured (consumers, 2^20 streams, L2 flushed,
// profiles/experiments/s42_consume_grid_waves.jsonl), k = 1 / 2 / 3 / 4 / 0:
// V1 1.669 / 1.687 / 1.693 / 1.690 / 1.689e12, V3 1.104 / 1.153 / 1.153 /
// 1.152 / 1.151e12, V2 2.61 / 2.70 / 2.70 / 2.68 / 2.67e11 numbers/s -- a
// single persistent wave leaves SMs idle behind the slowest warps.
#ifndef CIPRNG_PGRID_WAVES
#define CIPRNG_PGRID_WAVES 3
#endif
template <typename... KArgs>
inline int persistent_grid(void (*kern)(KArgs...), int threads, size_t smem, uint64_t blocks_needed) {
    const int r = CIPRNG_PGRID_WAVES == 0 ? 0x7FFFFFFF
                                          : CIPRNG_PGRID_WAVES * resident_blocks(reinterpret_cast<const void *>(kern),
                                                                                 threads, smem);
    const uint64_t b = blocks_needed < (uint64_t)r ? blocks_needed : (uint64_t)r;
    return (int)(b ? b : 1);
}

// Grid of the CTA-histogram consumers (sinks.cuh StatsSinkCta): k waves of
// resident CTAs (default 1: 2 x 14 warps per SM take the tiles round-robin),
// but never so few CTAs that a u32 histogram word could reach 2^31
// increments -- a word takes at most one increment per round from each warp
// of its CTA, i.e. tiles-per-warp x warps x n (n < 2^24 host-checked, so one
// tile per warp always fits).
#ifndef CIPRNG_V1C_CTA_WAVES
#define CIPRNG_V1C_CTA_WAVES 1
#endif
template <typename... KArgs, typename... Args>
inline void launch_cta_hist(void (*kern)(KArgs...), int wpb, size_t smem, uint64_t tiles, uint64_t n, cudaStream_t st,
                            Args &&...args) {
    // the 64 KiB opt-in: per (kernel, device), set on every call (a host
    // attribute write; a static flag here would be shared by every kernel of
    // the same signature, and the template instantiation is per signature)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const uint64_t need = (tiles + wpb - 1) / wpb;
    uint64_t grid = (uint64_t)CIPRNG_V1C_CTA_WAVES * resident_blocks(reinterpret_cast<const void *>(kern), 32 * wpb, smem);
    if (grid == 0 || grid > need) grid = need;
    while (grid < need && ((tiles + grid * wpb - 1) / (grid * wpb)) * (uint64_t)wpb * n >= (1ull << 31)) grid *= 2;
    if (grid > need) grid = need;
    launch_k(kern, dim3((unsigned)grid), dim3(32 * wpb), smem, st, std::forward<Args>(args)...);
}

struct InitArgs {
    uint32_t *state;
    uint64_t n_local;
    uint64_t seed;
    uint64_t first_stream;
    int variant;
    int paper_defaults;
    const uint32_t *mod;  // V2: [n_mod][kModWords] = {invMf, mu, 2^32 - M, K, M, Mp, R2, 0} (api.cu)
    uint32_t n_mod;
};

// Minimum-CTAs-per-SM operand of the generator kernels' launch bounds: 1
// (explicit) relaxes ptxas' register budget, 0 leaves its default.  Chosen
// per instantiation from B200 measurements (profiles/experiments/s44_launch_bounds.jsonl,
// both budgets measured for every kernel): 1 for the V1 and V3 TMA store
// kernels (+0.3 %, +1.4 %), the V0 consumer (+1.8 %) and the V4 store
// (+0.7 %); 0 for the V1 / V3 consumers (-1.1 %, -2.9 % with 1) and the V0
// store (-2.5 %).  -DCIPRNG_EXP_LB_MIN1 forces 1 everywhere (experiments).
#ifdef CIPRNG_EXP_LB_MIN1
constexpr bool kLbForceMin1 = true;
#else
constexpr bool kLbForceMin1 = false;
#endif

// V3 TMA store kernel shape (experiment knobs through CIPRNG_NVCC_EXTRA):
// box width in rounds (8, 16 or 32) and warps per CTA.  Measured (C2 shape,
// L2 flushed, profiles/experiments/s41_v3_box_shape.jsonl): 32-round boxes,
// 1 warp per CTA 1.236e12 numbers/s; 2 warps 1.219e12; 16-round boxes
// 1.17-1.20e12; 8-round 1.11e12.
#ifndef CIPRNG_V3_COLS
#define CIPRNG_V3_COLS 32
#endif
#ifndef CIPRNG_V3_WPB
#define CIPRNG_V3_WPB 1
#endif

// Tuning of the V1 fast store kernel (defaults chosen from B200 measurements,
// overridable for experiments with CIPRNG_V1_COLS / _WPB / _GRID).
struct V1Tuning {
    int cols = 32;        // TMA box width in rounds: 8, 16, 32 (2-D boxes) or
                          // 64, 128 (3-D band boxes, needs n % 32 == 0)
    int wpb = 4;          // warps per CTA (c32 w4 0.992 vs w2 0.979 of copy peak, profiles/experiments/s16)
    int grid_blocks = 0;  // 2-D kernels: 0 = one 64-stream tile per warp, > 0 = grid cap
    int bufs = 2;            // c32: shared-memory boxes per warp (1, 2 or 3)
    bool smem_stg = false;   // DIRECT store path via a shared-memory transpose + coalesced STG.128
    int tiles_per_warp = 1;  // 2-D kernels without a cap: grid = tiles / (wpb * tiles_per_warp)
    bool l2_prefetch = false; // 2-D TMA kernel: bulk-prefetch the next wave's state into L2 (+0.3 % flushed, -1.3 % steady: off, s18)
    int grid_mode = 0;    // band kernels: 0 = one tile per warp, -1 = persistent at
                          // full occupancy, k > 0 = persistent with k CTAs per SM
    bool shape_set = false;  // cols / wpb given by the environment: no per-n choice
};

// mode: 0 = store (direct), 1 = store (TMA tiles, V1 fast only), 2 = consume
int launch_init(const InitArgs &a, cudaStream_t st);
int launch_v0(const GenArgs &a, int mode, cudaStream_t st);
int launch_v1(const GenArgs &a, bool fast, int mode, const CUtensorMap *tmap, cudaStream_t st,
              const V1Tuning &tune);
int launch_v2(const GenArgs &a, int mode, cudaStream_t st, int kind = -1);
int launch_modsq_check(const uint32_t *mod, uint32_t n_mod, unsigned long long *bad, cudaStream_t st);
int launch_v3(const GenArgs &a, bool fast, int mode, const CUtensorMap *tmap, cudaStream_t st);
int launch_v4(const GenArgs &a, int mode, cudaStream_t st);
int launch_cbg(bool encrypt, int chaotic, uint64_t n_msgs, uint64_t L, const uint64_t *a0, const uint64_t *a1,
               const uint32_t *S0, const uint8_t *in, uint8_t *out, uint64_t *y, uint32_t *status, cudaStream_t st);
int launch_alg1(const uint32_t *f, uint32_t n, uint32_t b, uint32_t *z, uint32_t *x, uint64_t n_streams,
                uint64_t n_out, uint32_t *out, cudaStream_t st);
int launch_gamma(const uint32_t *f, uint32_t n, uint8_t *mark, unsigned long long *report, cudaStream_t st);
int launch_digest(const uint32_t *out, uint64_t first_stream, uint64_t n_local, uint64_t n, uint64_t *digest,
                  cudaStream_t st, int grid);
// v0_jump.cu: one V0 stream split over the GPU by GF(2) jump-ahead + XOR
// scan (C1).  The plan (jump polynomials for one (L, B)) lives in the handle.
#ifndef CIPRNG_JUMP_THREADS  // experiment knob
#define CIPRNG_JUMP_THREADS 128
#endif
// 128 threads per CTA: 25.2 us per C1 call; 256: 26.6 us (profiles/experiments/s62;
// bit-sweep era 34.8 vs 28.8); with the one-level jump 128 / 160 / 192 / 256:
// 20.5 / 21.2 / 21.4 / 20.7 us (s76).  Fewer than 128 is not supported (64 produced
// wrong words in s62: the kernel's per-CTA setup assumes at least 4 warps).
constexpr int kJumpThreads = CIPRNG_JUMP_THREADS;
static_assert(kJumpThreads >= 128 && kJumpThreads % 32 == 0, "v0_jump_kernel needs >= 4 warps per CTA");
constexpr int kJumpPolyWords = 6;
// One-level jump (default): every segment jumps straight from the chunk
// start with its own host polynomial z^((b T + t) L) -- no block-start pass,
// no second Krylov window build: 24.6 -> 20.5 us per C1 call, the per-shape
// plan 5 -> 70 ms of host time (profiles/experiments/s74).  0 = the two-level
// jump (block start, then segment) for comparison.
#ifndef CIPRNG_JUMP_ONE_LEVEL
#define CIPRNG_JUMP_ONE_LEVEL 1
#endif
#define kJumpOneLevel CIPRNG_JUMP_ONE_LEVEL
constexpr int kJumpMaxDeg[3] = {64, 256, 320};  // state bits of xor64, xor128-64, xorwow-64
constexpr uint32_t kJumpMaxL = 64;              // rounds per segment (shared-memory staging)
constexpr uint64_t kJumpMinN = 4096;            // below this the one-thread chain is as fast
constexpr uint64_t kJumpMaxStreams = 16;        // streams per handle the split path takes (grid rows)
struct V0JumpPlan {
    uint64_t *poly = nullptr;   // jump polynomials (v0_jump.cu)
    uint32_t *flags = nullptr;  // [B] look-back flags, then [B] block aggregates
    uint32_t L = 0, B = 0, epoch = 0, streams = 0;
    uint64_t n = 0;    // rounds of the call the launch shape was chosen for
    size_t smem = 0;
};
bool v0_jump_available();
int v0_jump_selftest(uint64_t *mismatches, uint32_t *degrees);  // host only
// >= 1: launches enqueued; -1..-3: not applicable / nothing enqueued (the
// caller falls back to the one-thread kernel); -4: a later chunk failed to
// launch after earlier chunks ran (the call fails, PRNG_ECUDA)
int v0_jump_launch(V0JumpPlan &p, uint32_t *state, uint64_t n_local, uint32_t *out, uint64_t n, cudaStream_t st);
void v0_jump_free(V0JumpPlan &p);

// emit.cu: format 1 = hex lines (9 B per word), 2 = bit lines (33 B per word)
int launch_format(const uint32_t *words, uint64_t count, int format, uint8_t *text, cudaStream_t st);

}  // namespace ciprng
