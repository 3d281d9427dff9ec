// api.cu -- the C ABI of include/ciprng.h: argument checking, device state
// ownership, kernel-path selection and the pipelined device->host path.
#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>
#include <cstdio>
#include <cstdlib>
#include <cerrno>
#include <cstring>
#include <unistd.h>
#include <vector>

#include "../../include/ciprng.h"
#include "device.cuh"
#include "kernels.h"

#define CIPRNG_STR_(x) #x
#define CIPRNG_STR(x) CIPRNG_STR_(x)

using namespace ciprng;

namespace {

thread_local char g_cuda_err[256] = "no error";

int cuda_fail(cudaError_t e) {
    std::snprintf(g_cuda_err, sizeof(g_cuda_err), "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
    return PRNG_ECUDA;
}
#define CK(expr)                                   \
    do {                                           \
        cudaError_t e_ = (expr);                   \
        if (e_ != cudaSuccess) return cuda_fail(e_); \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// Modulus table of V2 (reading Q13), built here independently of any other
// component: primes p = 3 (mod 4) in [128, 256] by a sieve, products p < q
// ascending, each as one 32-byte entry (kModWords words)
//   {invMf = bits of RZ(1/M) as float, mu = floor(2^32 / M), 2^32 - M,
//    K = 0x4B000000 * M mod 2^32, M, Mp = -M^{-1} mod 2^32, R2 = 2^64 mod M, 0}
// so one 128-bit load gives a BBS instance everything both squarings need
// (barrett_sq: mu, 2^32 - M; fbarrett_sq: invMf, 2^32 - M, K; device.cuh);
// the second 128-bit half serves the Montgomery alternative (mont_sq: M, Mp, R2);
// the negated modulus is stored rather than derived so each squaring ends in
// one IMAD + one VIADDMNMX.
static uint32_t rz_recip_bits(uint32_t M) {
    int k = 0;  // 2^23 <= floor(2^k / M) < 2^24: then RZ(1/M) = floor(2^k / M) * 2^-k
    while (((1ull << k) / M) < (1ull << 23)) ++k;
    const uint32_t m = (uint32_t)((1ull << k) / M);
    return ((uint32_t)(127 + 23 - k) << 23) | (m & 0x7FFFFFu);
}

std::vector<uint32_t> modulus_table() {
    std::vector<bool> composite(257, false);
    std::vector<uint32_t> primes;
    for (uint32_t v = 2; v <= 256; ++v) {
        if (composite[v]) continue;
        for (uint32_t w = v * v; w <= 256; w += v) composite[w] = true;
        if (v >= 128 && (v & 3u) == 3u) primes.push_back(v);
    }
    std::vector<uint32_t> Ms;
    for (size_t i = 0; i < primes.size(); ++i)
        for (size_t k = i + 1; k < primes.size(); ++k) Ms.push_back(primes[i] * primes[k]);
    std::sort(Ms.begin(), Ms.end());
    std::vector<uint32_t> tab;
    for (uint32_t M : Ms) {
        uint32_t inv = M;  // Newton: M*M = 1 (mod 8) for odd M; each step doubles the valid bits
        for (int k = 0; k < 4; ++k) inv *= 2u - M * inv;
        const uint32_t R2 = (uint32_t)((((unsigned __int128)1) << 64) % M);
        const uint32_t e[kModWords] = {rz_recip_bits(M), (uint32_t)((1ull << 32) / M), 0u - M,
                                       0x4B000000u * M, M, 0u - inv, R2, 0u};
        tab.insert(tab.end(), e, e + kModWords);
    }
    return tab;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                   const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    // resolved once, thread-safely (function-local static initialisation)
    static const EncodeTiledFn fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<EncodeTiledFn>(p);
        return static_cast<EncodeTiledFn>(nullptr);
    }();
    return fn;
}

constexpr int kStateWords[5] = {23, 6, 18, 4, 24};

}  // namespace

thread_local ciprng::L2Window ciprng::g_l2win;

int ciprng::resident_blocks(const void *kern, int threads, size_t smem) {
    static std::mutex mu;
    static std::map<std::tuple<const void *, int, size_t, int>, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    const auto key = std::make_tuple(kern, threads, smem, dev);
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    int sms = 148, per = 1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, threads, smem) != cudaSuccess || per < 1) per = 1;
    cudaGetLastError();
    return cache[key] = per * sms;
}

static bool env_on(const char *name, bool dflt);

bool ciprng::cta_hist_ok() {
    static std::mutex mu;
    static std::map<int, bool> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    int resv = -1;
    if (cudaDeviceGetAttribute(&resv, cudaDevAttrReservedSharedMemoryPerBlock, dev) != cudaSuccess) resv = -1;
    cudaGetLastError();
    // CIPRNG_CTA_HIST=0 forces the per-warp histograms (tests of the fallback)
    return cache[dev] = (resv == kCtaHistResvBytes) && env_on("CIPRNG_CTA_HIST", true);
}

static bool env_on(const char *name, bool dflt) {
    const char *v = std::getenv(name);
    if (!v || !v[0]) return dflt;
    return v[0] != '0';
}

bool ciprng::pdl_enabled() {
    static const bool on = [] {
        const char *v = std::getenv("CIPRNG_PDL");
        return !(v && v[0] == '0');
    }();
    return on;
}

struct prng_s {
    int variant = 0;
    uint64_t seed = 0, first = 0, n_local = 0;
    uint32_t C = 32;
    bool default_tables = true;
    int device = 0;
    int store_path = PRNG_STORE_AUTO;
    CombTables comb{};
    uint32_t *state = nullptr;
    uint32_t *mod = nullptr;  // V2 modulus table, n_mod entries of kModWords words
    uint32_t n_mod = 0;
    int num_sms = 148;
    // Evict-first output stores (default; CIPRNG_EVICT_FIRST=0 disables) and an
    // optional persisting-L2 window over the state planes (CIPRNG_L2PERSIST=1;
    // measured slower than evict-first alone on B200, gpurun_out/s11).
    size_t l2win_bytes = 0;
    float l2win_hit = 0.f;
    bool evict_first = true;
    bool state_last = true;
    V1Tuning v1tune;
    int v2_kind = -1;  // V2 store kernel instantiation (CIPRNG_V2_KIND, experiments; -1 = default)
    // last call info
    int last_path = 0;
    uint32_t last_launches = 0;
    // TMA descriptor cache
    struct TmEntry {
        const void *ptr = nullptr;
        uint64_t n = 0, rows = 0;
        int cols = 0;
        CUtensorMap map;
        bool ok = false;
    } tm[4];
    int tm_next = 0;
    // host pipeline
    uint32_t *staging[2] = {nullptr, nullptr};
    size_t staging_words = 0;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_gen[2] = {nullptr, nullptr}, ev_copy[2] = {nullptr, nullptr};
    // emitter (prng_emit): device text buffers and pinned host buffers
    uint8_t *text[2] = {nullptr, nullptr};
    size_t text_bytes = 0;
    uint8_t *pinned[2] = {nullptr, nullptr};
    size_t pinned_bytes = 0;
    // V0 single-stream jump-ahead plan (v0_jump.cu); CIPRNG_V0_JUMP=0 disables
    V0JumpPlan jump;
    bool jump_on = true;
};

namespace {

const CUtensorMap *tensor_map(prng_t *h, const uint32_t *out, uint64_t n, uint64_t rows, int cols) {
    for (auto &e : h->tm)
        if (e.ok && e.ptr == out && e.n == n && e.rows == rows && e.cols == cols) return &e.map;
    EncodeTiledFn fn = encode_fn();
    if (!fn) return nullptr;
    auto &e = h->tm[h->tm_next];
    h->tm_next = (h->tm_next + 1) & 3;
    cuuint64_t gdim[2] = {n, rows};
    cuuint64_t gstride[1] = {n * 4};
    if (cols >= 64) {
        // 3-D band view {32 words, rows, n/32 bands}; box {32, 64, cols/32}
        cuuint64_t gdim3[3] = {32, rows, n / 32};
        cuuint64_t gstride3[2] = {n * 4, 128};
        cuuint32_t box3[3] = {32, 64, (cuuint32_t)(cols / 32)};
        cuuint32_t estr3[3] = {1, 1, 1};
        CUresult r3 = fn(&e.map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<uint32_t *>(out), gdim3, gstride3,
                         box3, estr3, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        e.ok = (r3 == CUDA_SUCCESS);
        e.cols = cols;
        e.ptr = out;
        e.n = n;
        e.rows = rows;
        return e.ok ? &e.map : nullptr;
    }
    // box = cols rounds x 64 streams; swizzle span = the box row (cols * 4 B)
    cuuint32_t box[2] = {(cuuint32_t)cols, 64};
    cuuint32_t estr[2] = {1, 1};
    const CUtensorMapSwizzle sw = cols == 8 ? CU_TENSOR_MAP_SWIZZLE_32B
                                  : cols == 32 ? CU_TENSOR_MAP_SWIZZLE_128B
                                               : CU_TENSOR_MAP_SWIZZLE_64B;
    CUresult r = fn(&e.map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<uint32_t *>(out), gdim, gstride, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    e.ok = (r == CUDA_SUCCESS);
    e.cols = cols;
    e.ptr = out;
    e.n = n;
    e.rows = rows;
    return e.ok ? &e.map : nullptr;
}

// Enqueue one pass over local streams [s_begin, s_begin + s_count).
// mode 0 = store to out, 2 = consume into stats.
int run_pass(prng_t *h, uint64_t n, uint64_t s_begin, uint64_t s_count, uint32_t *out, uint64_t *stats, int mode,
             cudaStream_t st) {
    GenArgs a;
    std::memset(&a, 0, sizeof(a));
    a.state = h->state;
    a.n_local = h->n_local;
    a.s_begin = s_begin;
    a.s_count = s_count;
    a.n = n;
    a.out = out;
    a.stats = stats;
    a.mod = h->mod;
    a.C = h->C;
    a.comb = h->comb;
    a.vec = (out != nullptr && (n % 4 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0)) ? 1u : 0u;
    a.evict_first = h->evict_first ? 1u : 0u;
    a.state_last = h->state_last ? 1u : 0u;
    struct WindowScope {  // the state's L2 access-policy window for this pass's launches
        explicit WindowScope(const prng_t *hh) {
            g_l2win.base = hh->l2win_bytes ? hh->state : nullptr;
            g_l2win.bytes = hh->l2win_bytes;
            g_l2win.hit = hh->l2win_hit;
        }
        ~WindowScope() { g_l2win = L2Window(); }
    } window_scope(h);
    int launches = 0;
    int path = PRNG_STORE_DIRECT;
    if (h->variant == 0) {
        int jl = -1;
        if (mode == 0 && h->jump_on && h->n_local <= kJumpMaxStreams && s_begin == 0 && s_count == h->n_local &&
            n >= kJumpMinN)
            jl = v0_jump_launch(h->jump, h->state, h->n_local, out, n, st);
        if (jl == -4) return cuda_fail(cudaErrorLaunchFailure);
        if (jl > 0) path = PRNG_STORE_JUMP;
        launches = jl > 0 ? jl : launch_v0(a, mode, st);
    } else if (h->variant == 1) {
        const bool fast = h->default_tables && h->C == 32;
        int kmode = mode;
        const CUtensorMap *tm = nullptr;
        V1Tuning tune = h->v1tune;
        // Box shape by n (profiles/experiments/s35_band_by_n.jsonl, 2^20
        // streams, L2 flushed): 2-D 32-round boxes (128-byte row pieces 4n
        // bytes apart) win at n = 128 (1.51e12 vs 1.30e12) but lose ground as
        // the row stride grows (n = 1024: 1.33e12); 3-D band boxes of 64
        // rounds x 64 rows, 2 warps per CTA, write 256-byte row pieces and
        // stay at 1.51-1.64e12 for every n >= 192.
        if (!tune.shape_set && n >= 192 && n % 32 == 0) {
            tune.cols = 64;
            tune.wpb = 2;
        }
        if (tune.cols >= 64 && n % 32 != 0) tune.cols = 32;  // band boxes need whole 32-round bands
        if (mode == 0 && fast) {
            const bool tma_ok = a.vec && n < (1ull << 31) && s_count < (1ull << 31);
            if (h->store_path == PRNG_STORE_TMA && reinterpret_cast<uintptr_t>(out) % 16 != 0) return PRNG_EALIGN;
            if (h->store_path != PRNG_STORE_DIRECT && tma_ok) {
                tm = tensor_map(h, out, n, s_count, tune.cols);
                if (tm) {
                    kmode = 1;
                    path = PRNG_STORE_TMA;
                }
            }
            // no TMA descriptor (misaligned rows, n % 4 != 0): the staged
            // shared-memory + coalesced STG path unless DIRECT was requested
            if (kmode == 0 && h->store_path != PRNG_STORE_DIRECT) kmode = 4;
        }
        launches = launch_v1(a, fast, kmode, tm, st, tune);
    } else if (h->variant == 2) {
        launches = launch_v2(a, mode, st, h->v2_kind);
    } else if (h->variant == 3) {
        const bool fast = h->default_tables && h->C == 32;
        int kmode = mode;
        const CUtensorMap *tm = nullptr;
        if (mode == 0 && fast) {
            const bool tma_ok = a.vec && n < (1ull << 31) && s_count < (1ull << 31);
            if (h->store_path == PRNG_STORE_TMA && reinterpret_cast<uintptr_t>(out) % 16 != 0) return PRNG_EALIGN;
            if (h->store_path != PRNG_STORE_DIRECT && tma_ok) {
                tm = tensor_map(h, out, n, s_count, CIPRNG_V3_COLS);
                if (tm) {
                    kmode = 1;
                    path = PRNG_STORE_TMA;
                }
            }
            if (kmode == 0 && h->store_path != PRNG_STORE_DIRECT) kmode = 4;  // staged fallback
        }
        launches = launch_v3(a, fast, kmode, tm, st);
    } else {
        launches = launch_v4(a, mode, st);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e);
    h->last_launches += launches;
    h->last_path = path;
    return PRNG_OK;
}

bool pow2_le32(uint32_t c) { return c >= 1 && c <= 32 && (c & (c - 1)) == 0; }

}  // namespace

extern "C" {

int prng_create(uint64_t seed, uint64_t n_streams, int variant, prng_t **out) {
    return prng_create_shard(seed, 0, n_streams, variant, nullptr, out);
}

int prng_create_shard(uint64_t seed, uint64_t first_stream, uint64_t n_local, int variant, const prng_config *cfg,
                      prng_t **out) {
    if (out == nullptr) return PRNG_EINVAL;
    *out = nullptr;
    if (variant < 0 || variant > 4 || n_local == 0) return PRNG_EINVAL;
    uint32_t C = 32;
    const uint8_t *comb = nullptr;
    int paper_defaults = 0, store_path = PRNG_STORE_AUTO;
    if (cfg) {
        if (cfg->comb_size) C = cfg->comb_size;
        comb = cfg->comb;
        paper_defaults = cfg->paper_defaults;
        store_path = cfg->store_path;
    }
    if (store_path < 0 || store_path > 2) return PRNG_EINVAL;
    if (paper_defaults && !(variant == 0 && first_stream == 0 && n_local == 1)) return PRNG_EINVAL;
    if (n_local > (1ull << 40)) return PRNG_ESIZE;
    prng_t *h = new (std::nothrow) prng_t();
    if (!h) return PRNG_ENOMEM;
    h->variant = variant;
    h->seed = seed;
    h->first = first_stream;
    h->n_local = n_local;
    h->store_path = store_path;
    if (variant != 0) {
        if (!pow2_le32(C) || first_stream % C || n_local % C || (comb == nullptr && C != 32)) {
            delete h;
            return PRNG_EINVAL;
        }
        const int ntab = variant == 2 ? 16 : 2;
        for (int t = 0; t < ntab; ++t)
            for (uint32_t l = 0; l < C; ++l) {
                uint32_t v;
                if (comb) {
                    v = comb[t * C + l];
                    if (v >= C) {
                        delete h;
                        return PRNG_EINVAL;
                    }
                } else if (variant != 2) {  // V1, V3, V4: Alg. 4's two arrays
                    v = (t == 0) ? (l + 1u) % 32u : (l + 17u) % 32u;  // Q6
                } else {
                    v = (t < 8) ? (l + 1u + t) % 32u : (l + 17u + (t - 8)) % 32u;  // Q6
                }
                h->comb.t[t][l] = (uint8_t)v;
            }
        h->C = C;
        h->default_tables = (comb == nullptr);
    }
    int rc = PRNG_OK;
    cudaError_t e = cudaGetDevice(&h->device);
    if (e != cudaSuccess) {
        delete h;
        return cuda_fail(e);
    }
    cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device);
    // experiment overrides of the V1 store kernel shape
    if (const char *v = std::getenv("CIPRNG_V1_COLS")) {
        int c = std::atoi(v);
        if (c == 8 || c == 16 || c == 32 || c == 64 || c == 128) h->v1tune.cols = c;
        h->v1tune.shape_set = true;
    }
    if (const char *v = std::getenv("CIPRNG_V1_PERSIST")) h->v1tune.grid_mode = std::atoi(v);
    if (const char *v = std::getenv("CIPRNG_V1_WPB")) {
        int w = std::atoi(v);
        if (w >= 1 && w <= 8) h->v1tune.wpb = w;
        h->v1tune.shape_set = true;
    }
    for (const char *knob : {"CIPRNG_V1_PERSIST", "CIPRNG_V1_BUFS", "CIPRNG_V1_TPW", "CIPRNG_V1_GRID", "CIPRNG_V1_PF"})
        if (const char *v = std::getenv(knob); v && v[0]) h->v1tune.shape_set = true;
    if (const char *v = std::getenv("CIPRNG_V2_KIND")) h->v2_kind = std::atoi(v);
    h->v1tune.l2_prefetch = env_on("CIPRNG_V1_PF", false);
    h->jump_on = env_on("CIPRNG_V0_JUMP", true);
    h->v1tune.smem_stg = env_on("CIPRNG_V1_SMEM_STG", false);
    if (const char *v = std::getenv("CIPRNG_V1_BUFS")) {
        int b = std::atoi(v);
        if (b >= 1 && b <= 3) h->v1tune.bufs = b;
    }
    if (const char *v = std::getenv("CIPRNG_V1_TPW")) {
        int t = std::atoi(v);
        if (t >= 1 && t <= 64) h->v1tune.tiles_per_warp = t;
    }
    if (const char *v = std::getenv("CIPRNG_V1_GRID")) {
        int b = std::atoi(v);
        if (b > 0) h->v1tune.grid_blocks = b * h->num_sms;
    }
    const size_t words = (size_t)kStateWords[variant] * n_local;
    e = cudaMalloc(&h->state, words * 4);
    if (e != cudaSuccess) {
        cuda_fail(e);
        delete h;
        return PRNG_ENOMEM;
    }
    {
        // evict-last only pays while the planes are a small part of L2 (V1 24
        // MiB, V3 16 MiB at 2^20 streams); for V0/V2/V4's 72-96 MiB it evicts
        // useful lines (measured: V2 -11 %, gpurun_out/r1f)
        int l2 = 0;
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, h->device);
        h->state_last = env_on("CIPRNG_STATE_EVICT_LAST", true) && l2 > 0 && words * 4 <= (size_t)l2 / 4;
    }
    // Evict-first output stores pay only while they protect L2-resident state
    // planes: with the planes kept (2^20 V1 streams) +2-5 %, with planes
    // larger than the L2 budget (2^22-2^23 streams, C4 on one GPU) they cost
    // 3-4 % (profiles/experiments/s38_evict_first_by_state.jsonl)
    h->evict_first = env_on("CIPRNG_EVICT_FIRST", h->state_last);
    if (env_on("CIPRNG_L2PERSIST", false)) {
        // persisting-L2 carve-out (device-wide limit; only ever raised) sized
        // to the state planes, and a launch window covering them
        int max_persist = 0, max_window = 0;
        cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, h->device);
        cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, h->device);
        if (max_persist > 0 && max_window > 0) {
            size_t cur = 0;
            cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
            const size_t want = std::min(words * 4, (size_t)max_persist);
            if (cur < want) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
            cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
            h->l2win_bytes = std::min(words * 4, (size_t)max_window);
            h->l2win_hit = h->l2win_bytes ? std::min(1.0f, (float)cur / (float)h->l2win_bytes) : 0.f;
        }
        cudaGetLastError();  // the policy is an optimisation: never fail creation on it
    }
    std::vector<uint32_t> tab = modulus_table();
    h->n_mod = (uint32_t)(tab.size() / kModWords);
    e = cudaMalloc(&h->mod, tab.size() * 4);
    if (e == cudaSuccess) e = cudaMemcpy(h->mod, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        rc = cuda_fail(e);
        prng_destroy(h);
        return rc;
    }
    InitArgs ia;
    ia.state = h->state;
    ia.n_local = n_local;
    ia.seed = seed;
    ia.first_stream = first_stream;
    ia.variant = variant;
    ia.paper_defaults = paper_defaults;
    ia.mod = h->mod;
    ia.n_mod = h->n_mod;
    launch_init(ia, 0);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        rc = cuda_fail(e);
        prng_destroy(h);
        return rc;
    }
    *out = h;
    return PRNG_OK;
}

int prng_destroy(prng_t *h) {
    if (!h) return PRNG_OK;
    DeviceGuard g(h->device);
    if (h->copy_stream) cudaStreamSynchronize(h->copy_stream);
    cudaFree(h->state);
    cudaFree(h->mod);
    v0_jump_free(h->jump);
    cudaFree(h->staging[0]);
    cudaFree(h->staging[1]);
    for (int b = 0; b < 2; ++b) {
        cudaFree(h->text[b]);
        if (h->pinned[b]) cudaFreeHost(h->pinned[b]);
    }
    for (int b = 0; b < 2; ++b) {
        if (h->ev_gen[b]) cudaEventDestroy(h->ev_gen[b]);
        if (h->ev_copy[b]) cudaEventDestroy(h->ev_copy[b]);
    }
    if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
    delete h;
    return PRNG_OK;
}

// Device staging (two chunk buffers of `words` u32) and the copy stream +
// events of the host pipelines (prng_generate_host, prng_emit).
static int ensure_pipeline(prng_t *h, size_t words) {
    if (words > h->staging_words) {
        for (int b = 0; b < 2; ++b) {
            cudaFree(h->staging[b]);
            h->staging[b] = nullptr;
        }
        h->staging_words = 0;
        for (int b = 0; b < 2; ++b) {
            cudaError_t e = cudaMalloc(&h->staging[b], words * 4);
            if (e != cudaSuccess) {
                cuda_fail(e);
                return PRNG_ENOMEM;
            }
        }
        h->staging_words = words;
    }
    if (!h->copy_stream) {
        CK(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
        for (int b = 0; b < 2; ++b) {
            CK(cudaEventCreateWithFlags(&h->ev_gen[b], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&h->ev_copy[b], cudaEventDisableTiming));
        }
    }
    return PRNG_OK;
}

static int check_size(const prng_t *h, uint64_t n) {
    if (n && h->n_local > SIZE_MAX / 4 / n) return PRNG_ESIZE;
    return PRNG_OK;
}

int prng_generate(prng_t *h, uint64_t n_per_stream, uint32_t *out_dev, void *stream) {
    if (!h) return PRNG_EINVAL;
    h->last_launches = 0;
    if (n_per_stream == 0) return PRNG_OK;  // no words to write: out_dev may be NULL
    if (!out_dev) return PRNG_EINVAL;
    int rc = check_size(h, n_per_stream);
    if (rc) return rc;
    DeviceGuard g(h->device);
    return run_pass(h, n_per_stream, 0, h->n_local, out_dev, nullptr, 0, (cudaStream_t)stream);
}

int prng_generate_host(prng_t *h, uint64_t n_per_stream, uint32_t *out_host, void *stream) {
    if (!h) return PRNG_EINVAL;
    h->last_launches = 0;
    if (n_per_stream == 0) return PRNG_OK;
    if (!out_host) return PRNG_EINVAL;
    int rc = check_size(h, n_per_stream);
    if (rc) return rc;
    DeviceGuard g(h->device);
    cudaStream_t st = (cudaStream_t)stream;
    // chunk = whole 64-stream tiles, about 64 MiB of output
    const uint64_t row_bytes = n_per_stream * 4;
    uint64_t rows = (64ull << 20) / row_bytes;
    rows = std::max<uint64_t>(64, rows / 64 * 64);
    if (rows > h->n_local) rows = h->n_local;
    rc = ensure_pipeline(h, (size_t)rows * n_per_stream);
    if (rc) return rc;
    uint32_t launches = 0;
    uint64_t chunk = 0;
    for (uint64_t r0 = 0; r0 < h->n_local; r0 += rows, ++chunk) {
        const int b = (int)(chunk & 1);
        const uint64_t cnt = std::min<uint64_t>(rows, h->n_local - r0);
        if (chunk >= 2) CK(cudaStreamWaitEvent(st, h->ev_copy[b], 0));
        h->last_launches = 0;
        rc = run_pass(h, n_per_stream, r0, cnt, h->staging[b], nullptr, 0, st);
        if (rc) return rc;
        launches += h->last_launches;
        CK(cudaEventRecord(h->ev_gen[b], st));
        CK(cudaStreamWaitEvent(h->copy_stream, h->ev_gen[b], 0));
        CK(cudaMemcpyAsync(out_host + r0 * n_per_stream, h->staging[b], cnt * row_bytes, cudaMemcpyDeviceToHost,
                           h->copy_stream));
        CK(cudaEventRecord(h->ev_copy[b], h->copy_stream));
    }
    h->last_launches = launches;
    CK(cudaStreamSynchronize(h->copy_stream));
    CK(cudaStreamSynchronize(st));
    return PRNG_OK;
}

static bool write_all(int fd, const uint8_t *p, size_t len) {
    while (len) {
        const ssize_t k = ::write(fd, p, len);
        if (k < 0) {
            if (errno == EINTR) continue;
            return false;
        }
        p += k;
        len -= (size_t)k;
    }
    return true;
}

int prng_emit(prng_t *h, uint64_t n_per_stream, int fd, int format, uint64_t *bytes_written, void *stream) {
    if (bytes_written) *bytes_written = 0;
    if (!h || fd < 0 || format < PRNG_EMIT_RAW_LE32 || format > PRNG_EMIT_BITS) return PRNG_EINVAL;
    h->last_launches = 0;
    if (n_per_stream == 0) return PRNG_OK;
    const uint64_t bpw = format == PRNG_EMIT_RAW_LE32 ? 4 : format == PRNG_EMIT_HEX ? 9 : 33;
    if (h->n_local > SIZE_MAX / bpw / n_per_stream) return PRNG_ESIZE;
    DeviceGuard g(h->device);
    cudaStream_t st = (cudaStream_t)stream;
    // chunk = whole 64-stream tiles, about 64 MiB of serialised bytes
    uint64_t rows = (64ull << 20) / (n_per_stream * bpw);
    rows = std::max<uint64_t>(64, rows / 64 * 64);
    if (rows > h->n_local) rows = h->n_local;
    const size_t words = (size_t)rows * n_per_stream, bytes = words * bpw;
    int rc = ensure_pipeline(h, words);
    if (rc) return rc;
    if (format != PRNG_EMIT_RAW_LE32 && bytes > h->text_bytes) {
        for (int b = 0; b < 2; ++b) {
            cudaFree(h->text[b]);
            h->text[b] = nullptr;
        }
        h->text_bytes = 0;
        for (int b = 0; b < 2; ++b)
            if (cudaMalloc(&h->text[b], bytes) != cudaSuccess) return PRNG_ENOMEM;
        h->text_bytes = bytes;
    }
    if (bytes > h->pinned_bytes) {
        for (int b = 0; b < 2; ++b) {
            if (h->pinned[b]) cudaFreeHost(h->pinned[b]);
            h->pinned[b] = nullptr;
        }
        h->pinned_bytes = 0;
        for (int b = 0; b < 2; ++b)
            if (cudaHostAlloc(reinterpret_cast<void **>(&h->pinned[b]), bytes, cudaHostAllocDefault) != cudaSuccess)
                return PRNG_ENOMEM;
        h->pinned_bytes = bytes;
    }
    // chunk c: generate (+ format) on `stream`, copy to pinned[c & 1] on the
    // copy stream; meanwhile the host writes chunk c - 1.  Every chunk is
    // generated even after a write failure, so the handle's state always
    // advances by the whole call (like prng_generate).
    uint32_t launches = 0;
    uint64_t written = 0, pend_bytes = 0;
    bool io_ok = true;
    int pend = -1;  // buffer of the chunk waiting to be written
    uint64_t chunk = 0;
    for (uint64_t r0 = 0; r0 < h->n_local; r0 += rows, ++chunk) {
        const int b = (int)(chunk & 1);
        const uint64_t cnt = std::min<uint64_t>(rows, h->n_local - r0);
        if (chunk >= 2) CK(cudaStreamWaitEvent(st, h->ev_copy[b], 0));
        h->last_launches = 0;
        rc = run_pass(h, n_per_stream, r0, cnt, h->staging[b], nullptr, 0, st);
        if (rc) return rc;
        launches += h->last_launches;
        const uint8_t *src = reinterpret_cast<const uint8_t *>(h->staging[b]);
        if (format != PRNG_EMIT_RAW_LE32) {
            launches += launch_format(h->staging[b], cnt * n_per_stream, format, h->text[b], st);
            CK(cudaGetLastError());
            src = h->text[b];
        }
        CK(cudaEventRecord(h->ev_gen[b], st));
        CK(cudaStreamWaitEvent(h->copy_stream, h->ev_gen[b], 0));
        CK(cudaMemcpyAsync(h->pinned[b], src, cnt * n_per_stream * bpw, cudaMemcpyDeviceToHost, h->copy_stream));
        CK(cudaEventRecord(h->ev_copy[b], h->copy_stream));
        if (pend >= 0) {
            CK(cudaEventSynchronize(h->ev_copy[pend]));
            if (io_ok && (io_ok = write_all(fd, h->pinned[pend], pend_bytes))) written += pend_bytes;
        }
        pend = b;
        pend_bytes = cnt * n_per_stream * bpw;
    }
    CK(cudaEventSynchronize(h->ev_copy[pend]));
    if (io_ok && (io_ok = write_all(fd, h->pinned[pend], pend_bytes))) written += pend_bytes;
    CK(cudaStreamSynchronize(st));
    h->last_launches = launches;
    if (bytes_written) *bytes_written = written;
    return io_ok ? PRNG_OK : PRNG_EIO;
}

int prng_consume(prng_t *h, uint64_t n_per_stream, uint64_t *stats_dev, void *stream) {
    if (!h || !stats_dev || (n_per_stream & 1)) return PRNG_EINVAL;
    h->last_launches = 0;
    if (n_per_stream == 0) return PRNG_OK;
    if (n_per_stream >= (1ull << 24)) return PRNG_ESIZE;  // u32 tile counters (sinks.cuh)
    DeviceGuard g(h->device);
    return run_pass(h, n_per_stream, 0, h->n_local, nullptr, stats_dev, 2, (cudaStream_t)stream);
}

int prng_battery(prng_t *h, uint64_t n_per_stream, uint64_t *stats_dev, void *stream) {
    if (!h || !stats_dev) return PRNG_EINVAL;
    h->last_launches = 0;
    if (n_per_stream == 0) return PRNG_OK;
    if (n_per_stream >= (1ull << 20)) return PRNG_ESIZE;  // u32 tile counters (sinks.cuh)
    DeviceGuard g(h->device);
    return run_pass(h, n_per_stream, 0, h->n_local, nullptr, stats_dev, 3, (cudaStream_t)stream);
}

int prng_digest(const uint32_t *out_dev, uint64_t first_stream, uint64_t n_local, uint64_t n, uint64_t *digest_dev,
                void *stream) {
    if (!out_dev || !digest_dev) return PRNG_EINVAL;
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    launch_digest(out_dev, first_stream, n_local, n, digest_dev, (cudaStream_t)stream, sms * 8);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PRNG_OK : cuda_fail(e);
}

int prng_cbg_encrypt(int chaotic, uint64_t n_msgs, uint64_t L, const uint64_t *N_dev, const uint32_t *S0_dev,
                     const uint64_t *r_dev, const uint8_t *m_dev, uint8_t *c_dev, uint64_t *y_dev, void *stream) {
    if (n_msgs == 0) return PRNG_OK;
    if (!N_dev || !r_dev || !y_dev || (L && (!m_dev || !c_dev))) return PRNG_EINVAL;
    if (L && n_msgs > SIZE_MAX / L) return PRNG_ESIZE;
    launch_cbg(true, chaotic, n_msgs, L, N_dev, r_dev, S0_dev, m_dev, c_dev, y_dev, nullptr, (cudaStream_t)stream);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PRNG_OK : cuda_fail(e);
}

int prng_cbg_decrypt(int chaotic, uint64_t n_msgs, uint64_t L, const uint64_t *p_dev, const uint64_t *q_dev,
                     const uint32_t *S0_dev, const uint8_t *c_dev, const uint64_t *y_dev, uint8_t *m_dev,
                     uint32_t *status_dev, void *stream) {
    if (n_msgs == 0) return PRNG_OK;
    if (!p_dev || !q_dev || !y_dev || (L && (!m_dev || !c_dev))) return PRNG_EINVAL;
    if (L && n_msgs > SIZE_MAX / L) return PRNG_ESIZE;
    launch_cbg(false, chaotic, n_msgs, L, p_dev, q_dev, S0_dev, c_dev, m_dev, const_cast<uint64_t *>(y_dev),
               status_dev, (cudaStream_t)stream);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PRNG_OK : cuda_fail(e);
}

int prng_alg1_generate(const uint32_t *f_dev, uint32_t n, uint32_t b, uint32_t *z_dev, uint32_t *x_dev,
                       uint64_t n_streams, uint64_t n_out, uint32_t *out_dev, void *stream) {
    if (n == 0 || n > 32 || (f_dev && n > 16) || b == 0) return PRNG_EINVAL;
    if (n_streams == 0 || n_out == 0) return PRNG_OK;
    if (!z_dev || !x_dev || !out_dev) return PRNG_EINVAL;
    if (n_streams > SIZE_MAX / 4 / n_out) return PRNG_ESIZE;
    launch_alg1(f_dev, n, b, z_dev, x_dev, n_streams, n_out, out_dev, (cudaStream_t)stream);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PRNG_OK : cuda_fail(e);
}

int prng_gamma_check(const uint32_t *f_dev, uint32_t n, uint8_t *scratch_dev, uint64_t *report_dev, void *stream) {
    if (n == 0 || n > 16 || !scratch_dev || !report_dev) return PRNG_EINVAL;
    launch_gamma(f_dev, n, scratch_dev, reinterpret_cast<unsigned long long *>(report_dev), (cudaStream_t)stream);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PRNG_OK : cuda_fail(e);
}

int prng_get_info(const prng_t *h, prng_info_t *info) {
    if (!h || !info) return PRNG_EINVAL;
    info->variant = h->variant;
    info->comb_size = h->C;
    info->seed = h->seed;
    info->first_stream = h->first;
    info->n_local = h->n_local;
    info->state_words = (uint32_t)kStateWords[h->variant];
    info->device = h->device;
    info->store_path = h->last_path;
    info->kernel_launches = h->last_launches;
    return PRNG_OK;
}

int prng_get_state(const prng_t *h, void *host_buf, size_t bytes) {
    if (!h || !host_buf) return PRNG_EINVAL;
    const size_t need = (size_t)kStateWords[h->variant] * h->n_local * 4;
    if (bytes != need) return PRNG_ESTATE;
    DeviceGuard g(h->device);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(host_buf, h->state, need, cudaMemcpyDeviceToHost));
    return PRNG_OK;
}

/* Content check of a checkpoint before it reaches the device (the buffer is
 * already on the host): a V2 modulus index must address the table and each
 * BBS state must be a residue of its modulus (the kernels' Barrett squaring
 * assumes y < M < 2^16, and an index past the table would read out of
 * bounds); no xorshift-family generator may be all zero (a fixed point). */
static bool state_valid(const prng_t *h, const uint32_t *st) {
    const uint64_t L = h->n_local;
    auto w = [&](int plane, uint64_t s) { return st[(uint64_t)plane * L + s]; };
    auto zero = [&](int p0, int np, uint64_t s) {
        uint32_t o = 0;
        for (int p = p0; p < p0 + np; ++p) o |= w(p, s);
        return o == 0;
    };
    std::vector<uint32_t> tab;
    if (h->variant == PRNG_V2_BBS_COMB) tab = modulus_table();
    for (uint64_t s = 0; s < L; ++s) {
        switch (h->variant) {
            case PRNG_V0_XORLIKE3:
            case PRNG_V4_XORLIKE3_COMB:
                if (zero(0, 2, s) || zero(2, 8, s) || zero(10, 10, s)) return false;
                break;
            case PRNG_V1_XOR128_COMB:
                if (zero(0, 4, s)) return false;
                break;
            case PRNG_V3_XOR64_COMB:
                if (zero(0, 2, s)) return false;
                break;
            case PRNG_V2_BBS_COMB:
                for (int j = 0; j < 8; ++j) {
                    const uint32_t m = w(8 + j, s);
                    if (m >= h->n_mod || w(j, s) >= tab[(size_t)m * kModWords + 4]) return false;
                }
                break;
            default:
                return false;
        }
    }
    return true;
}

int prng_set_state(prng_t *h, const void *host_buf, size_t bytes) {
    if (!h || !host_buf) return PRNG_EINVAL;
    const size_t need = (size_t)kStateWords[h->variant] * h->n_local * 4;
    if (bytes != need) return PRNG_ESTATE;
    if (!state_valid(h, (const uint32_t *)host_buf)) return PRNG_ESTATE;
    DeviceGuard g(h->device);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h->state, host_buf, need, cudaMemcpyHostToDevice));
    return PRNG_OK;
}

const char *prng_strerror(int status) {
    switch (status) {
        case PRNG_OK: return "ok";
        case PRNG_EINVAL: return "invalid argument or configuration";
        case PRNG_ENOMEM: return "out of memory";
        case PRNG_ECUDA: return "CUDA error (see prng_last_cuda_error)";
        case PRNG_EALIGN: return "output pointer not 16-byte aligned";
        case PRNG_ESIZE: return "size overflow";
        case PRNG_ESTATE: return "state buffer size mismatch or invalid state content";
        case PRNG_EIO: return "write to the output sink failed (see errno)";
        default: return "unknown status";
    }
}

const char *prng_last_cuda_error(void) { return g_cuda_err; }

int prng_selftest_modsq(uint64_t *mismatches) {
    if (!mismatches) return PRNG_EINVAL;
    std::vector<uint32_t> tab = modulus_table();
    uint64_t bad = 0;
    for (size_t k = 0; k + kModWords <= tab.size(); k += kModWords) {
        const uint32_t invMf = tab[k], mu = tab[k + 1], nM = tab[k + 2], K = tab[k + 3], M = tab[k + 4];
        const uint32_t Mp = tab[k + 5], R2 = tab[k + 6];
        if (nM != 0u - M || K != 0x4B000000u * M || M * Mp != 0xFFFFFFFFu) ++bad;
        for (uint32_t y = 0; y < M; ++y) {
            const uint32_t ref = (y * y) % M;
            if (barrett_sq(y, nM, mu) != ref) ++bad;
            if (fbarrett_sq(y, nM, K, invMf) != ref) ++bad;
            uint32_t yh = mont_enter(y, M, Mp, R2);
            if (yh != (uint32_t)(((uint64_t)y << 32) % M) || mont_sq(yh, M, Mp) != ref ||
                yh != (uint32_t)(((uint64_t)ref << 32) % M))
                ++bad;
        }
    }
    *mismatches = bad;
    return PRNG_OK;
}

int prng_selftest_jump(uint64_t *mismatches, uint32_t *degrees) {
    if (!mismatches || !degrees) return PRNG_EINVAL;
    return v0_jump_selftest(mismatches, degrees);
}

int prng_selftest_modsq_gpu(uint64_t *mismatches) {
    if (!mismatches) return PRNG_EINVAL;
    std::vector<uint32_t> tab = modulus_table();
    uint32_t *mod = nullptr;
    unsigned long long *bad = nullptr;
    cudaError_t e = cudaMalloc(&mod, tab.size() * 4);
    if (e == cudaSuccess) e = cudaMalloc(&bad, sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemcpy(mod, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemset(bad, 0, sizeof(unsigned long long));
    if (e == cudaSuccess) {
        launch_modsq_check(mod, (uint32_t)(tab.size() / kModWords), bad, 0);
        e = cudaGetLastError();
    }
    unsigned long long host = 0;
    if (e == cudaSuccess) e = cudaMemcpy(&host, bad, sizeof(host), cudaMemcpyDeviceToHost);
    cudaFree(mod);
    cudaFree(bad);
    if (e != cudaSuccess) return cuda_fail(e);
    *mismatches = host;
    return PRNG_OK;
}

const char *prng_version(void) {
    return "ciprng 0.1 (sm_100a; nvcc " CIPRNG_STR(__CUDACC_VER_MAJOR__) "." CIPRNG_STR(__CUDACC_VER_MINOR__) ")";
}

}  // extern "C"
