// pipe_bench.cu -- issue/pipe throughput microbenchmarks on sm_100a, used to
// choose how the BBS squaring (V2) and the xor-like shifts are split across
// the ALU, heavy-FMA and FP64 pipes.  Each thread runs 8 independent chains
// of one instruction kind; the result is lane-ops per clock per SM.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC tools/pipe_bench.cu -o tools/libpipe.so
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define ITERS 2048

template <int K>
__global__ void kbench(uint32_t *sink, double *dsink, uint32_t c, double dc) {
    uint32_t a[8];
    double d[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        a[j] = threadIdx.x * 7u + j;
        d[j] = (double)(threadIdx.x + j);
    }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (K == 0) {  // IMAD (lo)
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(c), "r"(a[(j + 1) & 7]));
            } else if (K == 1) {  // IMAD.HI
                asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(c), "r"(a[(j + 1) & 7]));
            } else if (K == 2) {  // LOP3
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[j]) : "r"(c), "r"(a[(j + 1) & 7]));
            } else if (K == 3) {  // DFMA
                asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d[j]) : "d"(dc), "d"(d[(j + 1) & 7]));
            } else if (K == 4) {  // IMAD.HI + DFMA interleaved (1:1)
                asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(c), "r"(a[(j + 1) & 7]));
                asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d[j]) : "d"(dc), "d"(d[(j + 1) & 7]));
            } else if (K == 5) {  // IMAD lo + LOP3 (1:1)
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(c), "r"(a[(j + 1) & 7]));
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[(j + 4) & 7]) : "r"(c), "r"(a[(j + 5) & 7]));
            } else if (K == 6) {  // FFMA
                float f = __int_as_float(a[j]);
                asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(f) : "f"(1.0001f));
                a[j] = __float_as_int(f);
            } else if (K == 7) {  // IMAD lo + FFMA (1:1): do FP32 ops use the heavy pipe?
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(c), "r"(a[(j + 1) & 7]));
                float f = __int_as_float(a[(j + 4) & 7]);
                asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(f) : "f"(1.0001f));
                a[(j + 4) & 7] = __float_as_int(f);
            } else if (K == 8) {  // DMUL
                asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(d[j]) : "d"(dc));
            } else if (K == 9) {  // DFMA + LOP3 (1:1)
                asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d[j]) : "d"(dc), "d"(d[(j + 1) & 7]));
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[j]) : "r"(c), "r"(a[(j + 1) & 7]));
            } else if (K == 10) {  // SHF (funnel)
                asm volatile("shf.l.wrap.b32 %0, %0, %1, 13;" : "+r"(a[j]) : "r"(a[(j + 1) & 7]));
            } else if (K == 11) {  // IMAD.WIDE
                uint64_t w;
                asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(w) : "r"(a[j]), "r"(c));
                a[j] = (uint32_t)w ^ (uint32_t)(w >> 32);
            }
        }
    }
    uint32_t acc = 0;
    double dacc = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        acc ^= a[j];
        dacc += d[j];
    }
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    dsink[blockIdx.x * blockDim.x + threadIdx.x] = dacc;
}

typedef void (*KFn)(uint32_t *, double *, uint32_t, double);
static KFn kernels[] = {kbench<0>, kbench<1>, kbench<2>, kbench<3>, kbench<4>, kbench<5>,
                        kbench<6>, kbench<7>, kbench<8>, kbench<9>, kbench<10>, kbench<11>};

// returns milliseconds for one launch of kind k (after warm-up)
extern "C" float pipe_run(int k, int blocks, int threads) {
    uint32_t *s;
    double *ds;
    cudaMalloc(&s, (size_t)blocks * threads * 4);
    cudaMalloc(&ds, (size_t)blocks * threads * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    kernels[k]<<<blocks, threads>>>(s, ds, 0x9E3779B9u, 1.0000001);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) kernels[k]<<<blocks, threads>>>(s, ds, 0x9E3779B9u, 1.0000001);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaFree(s);
    cudaFree(ds);
    return ms / 5;
}

extern "C" int pipe_iters() { return ITERS; }
