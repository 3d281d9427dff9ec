// bg.cu -- SURVEY s8(f) NEXT-3: batch Blum-Goldwasser encryption /
// decryption and the paper's chaotic variant
// (P:1368-1386), one message per thread.
//
// Per message (reading Q33): x_0 = r^2 mod N; unit i uses x_i, then
// x_{i+1} = x_i^2 mod N; classic: c_i = m_i ^ lsb(x_i);
// chaotic: b_i = x_i mod 2^Nb with Nb = floor(log2(log2 N)),
// c_i = m_i ^ (b_0 ^ ... ^ b_i) ^ S0; y = x_L.
// Decryption recovers x_0 from y with the secret factors:
// r_p = y^(((p+1)/4)^L mod (p-1)) mod p, likewise r_q, CRT, then replays the
// keystream with the same cumulative XOR.
//
// Moduli are odd and < 2^63, so the squaring chain runs in 64-bit Montgomery
// form (R = 2^64): one Montgomery product and one reduction-to-canonical per
// unit.  The O(log) setup of decryption uses 128-bit % (a few hundred
// operations per message).  Units are bytes; each thread moves its message
// 16 units at a time (128-bit loads/stores) when the layout allows.
#include "device.cuh"
#include "kernels.h"

namespace ciprng {

struct Mont64 {
    uint64_t N, Ninv;  // Ninv = -N^-1 mod 2^64
    __device__ __forceinline__ explicit Mont64(uint64_t n) : N(n) {
        uint64_t x = n;  // n * x == 1 mod 2^3 for odd n; Newton doubles the bits
#pragma unroll
        for (int k = 0; k < 5; ++k) x *= 2 - n * x;
        Ninv = 0 - x;
    }
    // a * b * 2^-64 mod N for a, b < N < 2^63
    __device__ __forceinline__ uint64_t mul(uint64_t a, uint64_t b) const {
        const uint64_t lo = a * b, hi = __umul64hi(a, b);
        const uint64_t m = lo * Ninv;
        uint64_t t = hi + __umul64hi(m, N) + (lo != 0);  // (T + m N) / 2^64, < 2N
        return t >= N ? t - N : t;
    }
    // a * 2^-64 mod N (leave Montgomery form)
    __device__ __forceinline__ uint64_t redc(uint64_t a) const {
        const uint64_t m = a * Ninv;
        uint64_t t = __umul64hi(m, N) + (a != 0);
        return t >= N ? t - N : t;
    }
    // x * 2^64 mod N (enter Montgomery form): 64 modular doublings of x
    __device__ __forceinline__ uint64_t to(uint64_t x) const {
        uint64_t v = x % N;
        for (int k = 0; k < 64; ++k) {
            v <<= 1;  // v < N < 2^63: no overflow
            if (v >= N) v -= N;
        }
        return v;
    }
};

__device__ __forceinline__ uint64_t mulmod128(uint64_t a, uint64_t b, uint64_t m) {
    return (uint64_t)(((unsigned __int128)a * b) % m);
}
__device__ uint64_t powmod128(uint64_t a, uint64_t e, uint64_t m) {
    uint64_t r = 1 % m;
    a %= m;
    while (e) {
        if (e & 1) r = mulmod128(r, a, m);
        a = mulmod128(a, a, m);
        e >>= 1;
    }
    return r;
}
__device__ bool invmod128(uint64_t a, uint64_t m, uint64_t &inv) {
    __int128 t = 0, nt = 1, r = m, nr = a % m;
    while (nr != 0) {
        const __int128 q = r / nr;
        __int128 tmp = t - q * nt;
        t = nt;
        nt = tmp;
        tmp = r - q * nr;
        r = nr;
        nr = tmp;
    }
    if (r != 1) return false;
    if (t < 0) t += m;
    inv = (uint64_t)t;
    return true;
}
__device__ __forceinline__ uint64_t gcd64(uint64_t a, uint64_t b) {
    while (b) {
        const uint64_t t = a % b;
        a = b;
        b = t;
    }
    return a;
}
// Nb = floor(log2(log2 N)) = the largest t with N >= 2^(2^t)
__device__ __forceinline__ uint32_t unit_bits(uint64_t N) {
    uint32_t t = 0;
    while (t < 5 && N >= (1ull << (1u << (t + 1)))) ++t;
    return t;
}

// XOR the keystream of x_0 (canonical) into L units: out = in ^ key.
// chaotic: key_i = (b_0 ^ .. ^ b_i) ^ S0 masked to Nb bits; classic: lsb(x_i).
__device__ void keystream_xor(const Mont64 &M, uint64_t x0, bool chaotic, uint32_t S0, uint64_t L, const uint8_t *in,
                              uint8_t *out, uint64_t *x_end) {
    const uint32_t mask = chaotic ? ((1u << unit_bits(M.N)) - 1u) : 1u;
    uint64_t xm = M.to(x0), x = x0;
    uint32_t B = 0;
    auto key = [&]() -> uint32_t {  // key of the current x, then step x
        uint32_t k;
        if (chaotic) {
            B ^= (uint32_t)x & mask;
            k = (B ^ S0) & mask;
        } else {
            k = (uint32_t)x & 1u;
        }
        xm = M.mul(xm, xm);
        x = M.redc(xm);
        return k;
    };
    uint64_t i = 0;
    const bool vec = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15u) == 0;
    if (vec) {
        for (; i + 16 <= L; i += 16) {
            const uint4 v = *reinterpret_cast<const uint4 *>(in + i);
            uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint32_t k = key();
                k |= key() << 8;
                k |= key() << 16;
                k |= key() << 24;
                w[q] = (w[q] ^ k) & (mask * 0x01010101u);
            }
            *reinterpret_cast<uint4 *>(out + i) = make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
    for (; i < L; ++i) out[i] = (uint8_t)((in[i] ^ key()) & mask);
    if (x_end) *x_end = x;
}

// relaxed register budget (explicit minimum of 1 CTA/SM): +2 % encryption
// throughput (profiles/experiments/s47_misc_launch_bounds.jsonl)
__global__ void __launch_bounds__(256, 1) cbg_encrypt_kernel(int chaotic, uint64_t n_msgs, uint64_t L,
                                                          const uint64_t *Ns, const uint32_t *S0s,
                                                          const uint64_t *rs, const uint8_t *m, uint8_t *c,
                                                          uint64_t *y) {
    pdl_launch_dependents();
    pdl_wait();
    const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n_msgs) return;
    const uint64_t N = Ns[k], r = rs[k];
    if (N < 3 || !(N & 1) || (N >> 63) || gcd64(r % N, N) != 1) {  // invalid: flag y = 0
        y[k] = 0;
        return;
    }
    const Mont64 M(N);
    const uint64_t x0 = mulmod128(r, r, N);
    keystream_xor(M, x0, chaotic != 0, S0s ? S0s[k] : 0u, L, m + k * L, c + k * L, y + k);
}

__global__ void __launch_bounds__(256, 1) cbg_decrypt_kernel(int chaotic, uint64_t n_msgs, uint64_t L,
                                                          const uint64_t *ps, const uint64_t *qs,
                                                          const uint32_t *S0s, const uint8_t *c,
                                                          const uint64_t *ys, uint8_t *m, uint32_t *status) {
    pdl_launch_dependents();
    pdl_wait();
    const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n_msgs) return;
    const uint64_t p = ps[k], q = qs[k], y = ys[k];
    const unsigned __int128 N128 = (unsigned __int128)p * q;
    uint64_t ip = 0, iq = 0;
    if (p < 3 || q < 3 || p == q || (p & 3) != 3 || (q & 3) != 3 || (N128 >> 63) != 0 || y >= (uint64_t)N128 ||
        !invmod128(q % p, p, iq) || !invmod128(p % q, q, ip)) {
        if (status) status[k] = 1u;
        return;
    }
    const uint64_t N = (uint64_t)N128;
    const uint64_t ep = powmod128((p + 1) / 4, L, p - 1), eq = powmod128((q + 1) / 4, L, q - 1);
    const uint64_t rp = powmod128(y % p, ep, p), rq = powmod128(y % q, eq, q);
    const uint64_t x0 = (mulmod128(mulmod128(q, iq, N), rp, N) + mulmod128(mulmod128(p, ip, N), rq, N)) % N;
    if (status) status[k] = 0u;
    keystream_xor(Mont64(N), x0, chaotic != 0, S0s ? S0s[k] : 0u, L, c + k * L, m + k * L, nullptr);
}

int launch_cbg(bool encrypt, int chaotic, uint64_t n_msgs, uint64_t L, const uint64_t *a0, const uint64_t *a1,
               const uint32_t *S0, const uint8_t *in, uint8_t *out, uint64_t *y, uint32_t *status,
               cudaStream_t st) {
    if (n_msgs == 0) return 0;
    const int threads = 128;
    const dim3 grid((unsigned)((n_msgs + threads - 1) / threads));
    if (encrypt)
        launch_k(cbg_encrypt_kernel, grid, dim3(threads), 0, st, chaotic, n_msgs, L, a0, S0, a1, in, out, y);
    else
        launch_k(cbg_decrypt_kernel, grid, dim3(threads), 0, st, chaotic, n_msgs, L, a0, a1, S0, in,
                 (const uint64_t *)y, out, status);
    return 1;
}

}  // namespace ciprng
