// kernels.h -- host-side launchers of the sm_100a kernels (internal).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace ciprng {

struct GenArgs;

struct InitArgs {
    uint32_t *state;
    uint64_t n_local;
    uint64_t seed;
    uint64_t first_stream;
    int variant;
    int paper_defaults;
    const uint32_t *mod;  // V2: [n_mod][2] = {M, mu}
    uint32_t n_mod;
};

// mode: 0 = store (direct), 1 = store (TMA tiles, V1 fast only), 2 = consume
int launch_init(const InitArgs &a, cudaStream_t st);
int launch_v0(const GenArgs &a, int mode, cudaStream_t st, int persistent_blocks);
int launch_v1(const GenArgs &a, bool fast, int mode, const CUtensorMap *tmap, cudaStream_t st,
              int persistent_blocks);
int launch_v2(const GenArgs &a, int mode, cudaStream_t st, int persistent_blocks);
int launch_digest(const uint32_t *out, uint64_t first_stream, uint64_t n_local, uint64_t n, uint64_t *digest,
                  cudaStream_t st, int grid);

}  // namespace ciprng
