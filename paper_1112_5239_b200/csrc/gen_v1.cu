// gen_v1.cu -- V1: Alg. 4 "improved" kernel on sm_100a.
//
// Per stream (= paper thread): one 32-bit xor128 (Q5), the
// chaotic-iteration state x and the shared cell tp (the previous round's t,
// Q7/Q8).  Per round:  t = xor128() ^ tp[o1] ^ tp[o2];  tp = t;  x ^= t;
// emit x.  A combination group (C streams) never
// straddles a warp, so the exchange of shared cells is a register shuffle:
// no shared memory, no barrier, and the paper's unsynchronised shmem
// read/write becomes the two-phase semantics of reading Q7 by construction.
//
// Two kernels:
//  * v1_general_kernel -- any C | 32, any arrays: one lane per stream,
//    2 SHFL per number.
//  * v1_fast_kernel -- the default C = 32 arrays comb1 = l+1, comb2 = l+17
//    (Q6).  Because o2 = o1 + 16, lane j of a 16-lane half-warp owns streams
//    j and j+16 of a group; both need tp[j+1] ^ tp[j+17] = u[j+1] with
//    u[j] = tp[j] ^ tp[j+16] local to lane j, and u after a round is
//    g[j] ^ g[j+16] (the neighbour term cancels).  One SHFL per 2 numbers,
//    3 LOP3 per 2 numbers on top of the xor128 steps.  Stores either direct
//    (128-bit STG of 4-round buffers) or through a per-warp shared-memory
//    tile written to HBM by a 2-D TMA bulk tensor store.
#include "device.cuh"
#include "kernels.h"
#include "sinks.cuh"

namespace ciprng {

// ===================================================================== general
template <class Sink>
__global__ void __launch_bounds__(256) v1_general_kernel(GenArgs a) {
    Sink sink(a);
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t C = a.C;
    const uint32_t off = lane % C, gbase = lane - off;
    const uint32_t src1 = gbase + a.comb.t[0][off];
    const uint32_t src2 = gbase + a.comb.t[1][off];
    const uint64_t n_tiles = (a.s_count + 31) / 32;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    uint32_t *P = a.state;
    const uint64_t L = a.n_local;

    for (uint64_t tile = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); tile < n_tiles;
         tile += warps) {
        const uint64_t row = tile * 32 + lane;
        const bool valid = row < a.s_count;
        const uint64_t s = a.s_begin + row;
        uint32_t g0 = 0, g1 = 0, g2 = 0, g3 = 0, x = 0, tp = 0;
        if (valid) {
            g0 = P[0 * L + s]; g1 = P[1 * L + s]; g2 = P[2 * L + s]; g3 = P[3 * L + s];
            x = P[4 * L + s]; tp = P[5 * L + s];
        }
        sink.begin_tile();
        uint64_t i = 0;
        for (; i + 4 <= a.n; i += 4) {
            uint32_t t, o0, o1, o2, o3;
            g0 = xor128_f(g0, g3);
            t = g0 ^ __shfl_sync(kFull, tp, src1) ^ __shfl_sync(kFull, tp, src2);
            tp = t; x ^= t; o0 = x;
            g1 = xor128_f(g1, g0);
            t = g1 ^ __shfl_sync(kFull, tp, src1) ^ __shfl_sync(kFull, tp, src2);
            tp = t; x ^= t; o1 = x;
            g2 = xor128_f(g2, g1);
            t = g2 ^ __shfl_sync(kFull, tp, src1) ^ __shfl_sync(kFull, tp, src2);
            tp = t; x ^= t; o2 = x;
            g3 = xor128_f(g3, g2);
            t = g3 ^ __shfl_sync(kFull, tp, src1) ^ __shfl_sync(kFull, tp, src2);
            tp = t; x ^= t; o3 = x;
            sink.put4(row, i, o0, o1, o2, o3, valid);
        }
        for (; i < a.n; ++i) {  // ragged tail: plain step with register moves
            uint32_t g = xor128_f(g0, g3);
            g0 = g1; g1 = g2; g2 = g3; g3 = g;
            uint32_t t = g ^ __shfl_sync(kFull, tp, src1) ^ __shfl_sync(kFull, tp, src2);
            tp = t; x ^= t;
            sink.put1(row, i, x, valid);
        }
        if (valid) {
            P[0 * L + s] = g0; P[1 * L + s] = g1; P[2 * L + s] = g2; P[3 * L + s] = g3;
            P[4 * L + s] = x; P[5 * L + s] = tp;
        }
    }
    sink.finish(a);
}

// ======================================================================== fast
// Tile = 64 streams (2 groups) per warp; lane L: half h = L >> 4 (group),
// j = L & 15, owns rows rA = 32h + j and rB = rA + 16 of the tile.
constexpr int kFastTileRows = 64;
constexpr int kTmaCols = 16;                                   // rounds per TMA box
constexpr int kTmaTileBytes = kFastTileRows * kTmaCols * 4;    // 4 KiB
constexpr int kTmaWarpBytes = 2 * kTmaTileBytes;               // double buffer

// byte offset of 16-byte chunk c (0..3) of row r (0..63) in a 64-byte-row
// tile written with CU_TENSOR_MAP_SWIZZLE_64B (16-byte chunk index XOR
// address bits [7:8]); conflict-free for 8 consecutive rows.
__device__ __forceinline__ uint32_t swz64(uint32_t r, uint32_t c) { return r * 64u + ((c ^ ((r >> 1) & 3u)) << 4); }

template <class Sink, bool kTma>
__global__ void __launch_bounds__(128) v1_fast_kernel(GenArgs a, const __grid_constant__ CUtensorMap tmap) {
    Sink sink(a);
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t h = lane >> 4, j = lane & 15u;
    const uint32_t src = (j + 1u) & 15u;  // width-16 shuffle source
    const uint64_t n_tiles = (a.s_count + kFastTileRows - 1) / kFastTileRows;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    uint32_t *P = a.state;
    const uint64_t L = a.n_local;
    const uint32_t rA_t = 32u * h + j, rB_t = rA_t + 16u;  // rows within the tile

    uint32_t wsmem = 0;
    if constexpr (kTma) {
        extern __shared__ __align__(1024) uint8_t smem_dyn[];
        // swizzled TMA boxes need 1 KiB-aligned shared addresses
        const uint32_t base = (smem_u32(smem_dyn) + 1023u) & ~1023u;
        wsmem = base + (threadIdx.x >> 5) * kTmaWarpBytes;
    }
    uint32_t tma_issued = 0;  // tiles issued by this warp (lane 0 tracks groups)

    for (uint64_t tile = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); tile < n_tiles;
         tile += warps) {
        const uint64_t row0 = tile * kFastTileRows;
        const bool valid = row0 + 32u * h < a.s_count;  // s_count % 32 == 0
        const uint64_t rA = row0 + rA_t, rB = row0 + rB_t;
        const uint64_t sA = a.s_begin + rA, sB = a.s_begin + rB;
        uint32_t a0 = 0, a1 = 0, a2 = 0, a3 = 0, xA = 0, tpA = 0;
        uint32_t b0 = 0, b1 = 0, b2 = 0, b3 = 0, xB = 0, tpB = 0;
        if (valid) {
            a0 = P[0 * L + sA]; a1 = P[1 * L + sA]; a2 = P[2 * L + sA]; a3 = P[3 * L + sA];
            xA = P[4 * L + sA]; tpA = P[5 * L + sA];
            b0 = P[0 * L + sB]; b1 = P[1 * L + sB]; b2 = P[2 * L + sB]; b3 = P[3 * L + sB];
            xB = P[4 * L + sB]; tpB = P[5 * L + sB];
        }
        sink.begin_tile();
        uint32_t u = tpA ^ tpB;  // u[j] = tp[j] ^ tp[j+16]
        uint32_t nb = 0;

#define CIPRNG_V1_ROUND(GA, GA3, GB, GB3, OA, OB)        \
    GA = xor128_f(GA, GA3);                              \
    GB = xor128_f(GB, GB3);                              \
    nb = __shfl_sync(kFull, u, src, 16);                 \
    xA ^= GA ^ nb;                                       \
    xB ^= GB ^ nb;                                       \
    u = GA ^ GB;                                         \
    OA = xA;                                             \
    OB = xB;

        uint64_t i = 0;
        if constexpr (kTma) {
            // rounds in boxes of kTmaCols; n % 4 == 0 guaranteed by the host
            for (uint64_t i0 = 0; i0 < a.n; i0 += kTmaCols) {
                const uint32_t buf = wsmem + (tma_issued & 1u) * kTmaTileBytes;
                if (tma_issued >= 2) {
                    if (lane == 0) bulk_wait_read<1>();
                    __syncwarp();
                }
#pragma unroll
                for (uint32_t q = 0; q < kTmaCols / 4; ++q) {
                    if (i0 + 4 * q < a.n) {
                        uint32_t oA0, oA1, oA2, oA3, oB0, oB1, oB2, oB3;
                        CIPRNG_V1_ROUND(a0, a3, b0, b3, oA0, oB0)
                        CIPRNG_V1_ROUND(a1, a0, b1, b0, oA1, oB1)
                        CIPRNG_V1_ROUND(a2, a1, b2, b1, oA2, oB2)
                        CIPRNG_V1_ROUND(a3, a2, b3, b2, oA3, oB3)
                        st_shared_v4(buf + swz64(rA_t, q), oA0, oA1, oA2, oA3);
                        st_shared_v4(buf + swz64(rB_t, q), oB0, oB1, oB2, oB3);
                    }
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    tma_store_2d(&tmap, buf, (int)i0, (int)row0);
                    bulk_commit();
                }
                ++tma_issued;
            }
            i = a.n;
        } else {
            for (; i + 4 <= a.n; i += 4) {
                uint32_t oA0, oA1, oA2, oA3, oB0, oB1, oB2, oB3;
                CIPRNG_V1_ROUND(a0, a3, b0, b3, oA0, oB0)
                CIPRNG_V1_ROUND(a1, a0, b1, b0, oA1, oB1)
                CIPRNG_V1_ROUND(a2, a1, b2, b1, oA2, oB2)
                CIPRNG_V1_ROUND(a3, a2, b3, b2, oA3, oB3)
                sink.put4(rA, i, oA0, oA1, oA2, oA3, valid);
                sink.put4(rB, i, oB0, oB1, oB2, oB3, valid);
            }
            for (; i < a.n; ++i) {  // ragged tail
                uint32_t gA = xor128_f(a0, a3), gB = xor128_f(b0, b3);
                a0 = a1; a1 = a2; a2 = a3; a3 = gA;
                b0 = b1; b1 = b2; b2 = b3; b3 = gB;
                nb = __shfl_sync(kFull, u, src, 16);
                xA ^= gA ^ nb;
                xB ^= gB ^ nb;
                u = gA ^ gB;
                sink.put1(rA, i, xA, valid, 0);
                sink.put1(rB, i, xB, valid, 1);
            }
        }
#undef CIPRNG_V1_ROUND
        if (valid) {
            if (a.n > 0) {
                // last round's t: t = g ^ nb; g is the newest ring entry (a3 after
                // whole blocks; the tail shifts it into a3 as well)
                tpA = a3 ^ nb;
                tpB = b3 ^ nb;
            }
            P[0 * L + sA] = a0; P[1 * L + sA] = a1; P[2 * L + sA] = a2; P[3 * L + sA] = a3;
            P[4 * L + sA] = xA; P[5 * L + sA] = tpA;
            P[0 * L + sB] = b0; P[1 * L + sB] = b1; P[2 * L + sB] = b2; P[3 * L + sB] = b3;
            P[4 * L + sB] = xB; P[5 * L + sB] = tpB;
        }
    }
    if constexpr (kTma) {
        if (lane == 0) bulk_wait<0>();
        __syncwarp();
    }
    sink.finish(a);
}

// ===================================================================== launch
static int blocks_for(uint64_t warps_needed, int warps_per_block, int cap_blocks) {
    uint64_t b = (warps_needed + warps_per_block - 1) / warps_per_block;
    if (cap_blocks > 0 && b > (uint64_t)cap_blocks) b = cap_blocks;
    if (b == 0) b = 1;
    return (int)b;
}

int launch_v1(const GenArgs &a, bool fast, int mode, const CUtensorMap *tmap, cudaStream_t st,
              int persistent_blocks) {
    // mode: 0 store-direct, 1 store-tma, 2 consume
    if (a.s_count == 0) return 0;
    if (fast) {
        const uint64_t tiles = (a.s_count + kFastTileRows - 1) / kFastTileRows;
        const int wpb = 4;
        CUtensorMap dummy;
        if (tmap == nullptr) tmap = &dummy;
        if (mode == 0) {
            int grid = blocks_for(tiles, wpb, 0);
            v1_fast_kernel<StoreSink, false><<<grid, 32 * wpb, 0, st>>>(a, *tmap);
        } else if (mode == 1) {
            int grid = blocks_for(tiles, wpb, 0);
            size_t smem = (size_t)wpb * kTmaWarpBytes + 1024;  // + alignment slack
            v1_fast_kernel<StoreSink, true><<<grid, 32 * wpb, smem, st>>>(a, *tmap);
        } else {
            int grid = blocks_for(tiles, wpb, persistent_blocks);
            v1_fast_kernel<StatsSink, false><<<grid, 32 * wpb, wpb * StatsSink::kSmemBytesPerWarp, st>>>(a, *tmap);
        }
    } else {
        const uint64_t tiles = (a.s_count + 31) / 32;
        const int wpb = 8;
        if (mode == 2) {
            int grid = blocks_for(tiles, wpb, persistent_blocks);
            v1_general_kernel<StatsSink><<<grid, 32 * wpb, wpb * StatsSink::kSmemBytesPerWarp, st>>>(a);
        } else {
            int grid = blocks_for(tiles, wpb, 0);
            v1_general_kernel<StoreSink><<<grid, 32 * wpb, 0, st>>>(a);
        }
    }
    return 1;
}

}  // namespace ciprng
