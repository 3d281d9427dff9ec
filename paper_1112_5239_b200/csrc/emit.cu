// emit.cu -- serialisation of generated words for external test batteries
// (SURVEY s8(b) raw-LE32 sink; "raw little-endian 32-bit words
// to file or standard output", S:642-650 emit(..., format in {raw-le32, hex,
// bits}); the paper ran DieHARD / TestU01 BigCrush on its outputs).
//
// raw-le32 needs no kernel: the device words ARE little-endian u32, so the
// chunk is copied as is.  hex and bits are text: one line per word, built
// on the GPU so the host only copies and writes.  Bit order for "bits" is
// the battery's (reading Q31): most significant bit first.
#include "device.cuh"
#include "kernels.h"

namespace ciprng {

// hex: 8 lowercase digits + '\n' (9 bytes per word); bits: 32 '0'/'1' + '\n'
// (33 bytes per word).  One thread per word; each writes its own line.
__global__ void __launch_bounds__(256) format_kernel(const uint32_t *__restrict__ words, uint64_t count, int format,
                                                     uint8_t *__restrict__ text) {
    pdl_launch_dependents();
    pdl_wait();
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count; k += stride) {
        const uint32_t w = words[k];
        if (format == 1) {
            uint8_t *p = text + 9 * k;
#pragma unroll
            for (int d = 0; d < 8; ++d) {
                const uint32_t nib = (w >> (28 - 4 * d)) & 15u;
                p[d] = (uint8_t)(nib < 10 ? '0' + nib : 'a' + nib - 10);
            }
            p[8] = '\n';
        } else {
            uint8_t *p = text + 33 * k;
#pragma unroll
            for (int b = 0; b < 32; ++b) p[b] = (uint8_t)('0' + ((w >> (31 - b)) & 1u));
            p[32] = '\n';
        }
    }
}

int launch_format(const uint32_t *words, uint64_t count, int format, uint8_t *text, cudaStream_t st) {
    if (count == 0) return 0;
    uint64_t blocks = (count + 255) / 256;
    if (blocks > 148u * 16u) blocks = 148u * 16u;
    launch_k(format_kernel, dim3((int)blocks), dim3(256), 0, st, words, count, format, text);
    return 1;
}

}  // namespace ciprng
