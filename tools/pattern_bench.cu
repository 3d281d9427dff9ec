// pattern_bench.cu -- HBM write-pattern microbenchmark (tools only, not the
// product): the V1 TMA tile-store address pattern with NO generator compute,
// versus a coalesced STG.128 fill, to separate pattern limits from compute
// limits.  Build: nvcc -shared -Xcompiler -fPIC -gencode
// arch=compute_100a,code=sm_100a tools/pattern_bench.cu -o tools/libpattern.so
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int kCols>
__global__ void __launch_bounds__(256) tma_pattern(const __grid_constant__ CUtensorMap tmap, uint64_t rows, uint64_t n) {
    constexpr uint32_t kTile = 64 * kCols * 4;
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t base = ((smem_u32(smem) + 1023u) & ~1023u) + (threadIdx.x >> 5) * 2 * kTile;
    // fill both buffers once
    for (uint32_t o = lane * 16; o < 2 * kTile; o += 512)
        asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(base + o), "r"(o) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    const uint64_t tiles = rows / 64;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    uint32_t issued = 0;
    for (uint64_t t = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < tiles; t += warps) {
        for (uint64_t i0 = 0; i0 < n; i0 += kCols) {
            if (lane == 0) {
                if (issued >= 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                                 reinterpret_cast<uint64_t>(&tmap)),
                             "r"(base + (issued & 1) * kTile), "r"((int)i0), "r"((int)(t * 64))
                             : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            ++issued;
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// 3-D box {32 words, 64 rows, kBands}: one TMA op writes kBands*128 B of
// each of 64 consecutive rows (rows are n*4 bytes apart in global).
template <int kBands, int kBufs>
__global__ void __launch_bounds__(256) tma3d_pattern(const __grid_constant__ CUtensorMap tmap, uint64_t rows, uint64_t n) {
    constexpr uint32_t kTile = 64 * 32 * 4 * kBands;
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t base = ((smem_u32(smem) + 1023u) & ~1023u) + (threadIdx.x >> 5) * kBufs * kTile;
    for (uint32_t o = lane * 16; o < kBufs * kTile; o += 512)
        asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(base + o), "r"(o) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    const uint64_t tiles = rows / 64;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    uint32_t issued = 0;
    for (uint64_t t = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < tiles; t += warps) {
        for (uint64_t b0 = 0; b0 < n / 32; b0 += kBands) {
            if (lane == 0) {
                if (issued >= kBufs) {
                    if (kBufs == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                    else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                }
                asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                                 reinterpret_cast<uint64_t>(&tmap)),
                             "r"(base + (issued % kBufs) * kTile), "r"(0), "r"((int)(t * 64)), "r"((int)b0)
                             : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            ++issued;
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// contiguous 1-D bulk copies: each warp writes its tile (64 rows x n words,
// contiguous) in kChunk-byte pieces
template <int kChunk>
__global__ void __launch_bounds__(256) bulk1d_pattern(uint8_t *out, uint64_t rows, uint64_t n) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t base = ((smem_u32(smem) + 1023u) & ~1023u) + (threadIdx.x >> 5) * 2 * kChunk;
    const uint64_t tiles = rows / 64, tile_bytes = 64 * n * 4;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    uint32_t issued = 0;
    for (uint64_t t = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < tiles; t += warps) {
        for (uint64_t o = 0; o < tile_bytes; o += kChunk) {
            if (lane == 0) {
                if (issued >= 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + t * tile_bytes + o),
                             "r"(base + (issued & 1) * kChunk), "n"(kChunk)
                             : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            ++issued;
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void stg_fill(uint4 *p, uint64_t n16) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n16; k += stride)
        p[k] = make_uint4((uint32_t)k, 1, 2, 3);
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

extern "C" __attribute__((visibility("default"))) float pattern_run(int which, void *out, uint64_t rows, uint64_t n,
                                                                   int cols, int wpb, int blocks_per_sm, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    CUtensorMap map;
    void *fnp0 = nullptr;
    {
        cudaDriverEntryPointQueryResult q0;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp0, cudaEnableDefault, &q0);
    }
    if (which == 2) {  // 3-D band map, cols = bands per op
        cuuint64_t gdim[3] = {32, rows, n / 32};
        cuuint64_t gstr[2] = {n * 4, 128};
        cuuint32_t box[3] = {32, 64, (cuuint32_t)cols};
        cuuint32_t es[3] = {1, 1, 1};
        CUresult r = ((EncodeFn)fnp0)(&map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, out, gdim, gstr, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { fprintf(stderr, "encode3d failed %d\n", (int)r); return -2.f; }
    }
    if (which == 0) {
        void *fnp = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
        cuuint64_t gdim[2] = {n, rows};
        cuuint64_t gstr[1] = {n * 4};
        cuuint32_t box[2] = {(cuuint32_t)cols, 64};
        cuuint32_t es[2] = {1, 1};
        CUtensorMapSwizzle sw = cols == 8 ? CU_TENSOR_MAP_SWIZZLE_32B
                                : cols == 32 ? CU_TENSOR_MAP_SWIZZLE_128B
                                             : CU_TENSOR_MAP_SWIZZLE_64B;
        ((EncodeFn)fnp)(&map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, out, gdim, gstr, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    auto launch = [&]() {
        if (which == 0) {
            uint64_t warps = rows / 64;
            int grid = (int)((warps + wpb - 1) / wpb);
            if (blocks_per_sm > 0 && grid > blocks_per_sm * sms) grid = blocks_per_sm * sms;
            size_t smem = (size_t)wpb * 2 * 64 * cols * 4 + 1024;
            if (cols == 8) {
                cudaFuncSetAttribute(tma_pattern<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                tma_pattern<8><<<grid, 32 * wpb, smem>>>(map, rows, n);
            } else if (cols == 16) {
                cudaFuncSetAttribute(tma_pattern<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                tma_pattern<16><<<grid, 32 * wpb, smem>>>(map, rows, n);
            } else {
                cudaFuncSetAttribute(tma_pattern<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                tma_pattern<32><<<grid, 32 * wpb, smem>>>(map, rows, n);
            }
        } else if (which == 2) {
            uint64_t warps = rows / 64;
            int grid = (int)((warps + wpb - 1) / wpb);
            if (blocks_per_sm > 0 && grid > blocks_per_sm * sms) grid = blocks_per_sm * sms;
            const int bufs = (cols >= 4) ? 1 : 2;
            size_t smem = (size_t)wpb * bufs * 64 * 32 * 4 * cols + 1024;
#define L3(B, F)                                                                                           \
    if (cols == B) {                                                                                       \
        cudaFuncSetAttribute(tma3d_pattern<B, F>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        tma3d_pattern<B, F><<<grid, 32 * wpb, smem>>>(map, rows, n);                                       \
    }
            L3(1, 2) L3(2, 2) L3(4, 1)
#undef L3
        } else if (which == 3) {
            uint64_t warps = rows / 64;
            int grid = (int)((warps + wpb - 1) / wpb);
            if (blocks_per_sm > 0 && grid > blocks_per_sm * sms) grid = blocks_per_sm * sms;
            size_t smem = (size_t)wpb * 2 * 16384 + 1024;
            cudaFuncSetAttribute(bulk1d_pattern<16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            bulk1d_pattern<16384><<<grid, 32 * wpb, smem>>>((uint8_t *)out, rows, n);
        } else {
            stg_fill<<<sms * 8, 256>>>((uint4 *)out, rows * n / 4);
        }
    };
    for (int r = 0; r < 3; ++r) launch();
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        fprintf(stderr, "pattern_run: %s\n", cudaGetErrorString(e));
        return -1.f;
    }
    return ms / reps;
}
