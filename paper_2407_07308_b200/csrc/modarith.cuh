// modarith.cuh -- 64-bit modular arithmetic for sm_100a (primes q < 2^62).
// Residues are canonical in [0, q) at every kernel boundary (bit-exact contract, R3).
#pragma once
#include <cstdint>

#define BC_DEV __device__ __forceinline__

namespace bc {

// Per-modulus constants: q, Barrett mu = floor(2^(2b) / q) with b = bitlength(q), shift b.
struct Mod {
    uint64_t q;
    uint64_t mu;
    uint32_t b;
    uint32_t pad;
};

BC_DEV uint64_t add_mod(uint64_t a, uint64_t b, uint64_t q) {
    uint64_t s = a + b;
    return s >= q ? s - q : s;
}
BC_DEV uint64_t sub_mod(uint64_t a, uint64_t b, uint64_t q) { return a >= b ? a - b : a + q - b; }
BC_DEV uint64_t neg_mod(uint64_t a, uint64_t q) { return a ? q - a : 0; }

// Shoup: w' = floor(w * 2^64 / q); returns x*w mod q for any x < 2^64 (q < 2^63).
BC_DEV uint64_t mul_shoup(uint64_t x, uint64_t w, uint64_t wp, uint64_t q) {
    uint64_t hi = __umul64hi(x, wp);
    uint64_t r = x * w - hi * q;
    return r >= q ? r - q : r;
}
// lazy variant: result in [0, 2q)
BC_DEV uint64_t mul_shoup_lazy(uint64_t x, uint64_t w, uint64_t wp, uint64_t q) {
    uint64_t hi = __umul64hi(x, wp);
    return x * w - hi * q;
}

// Barrett for a*b with a, b < q < 2^62: x = a*b < 2^(2b); x1 = x >> (b-1) < 2^(b+1);
// qhat = (x1 * mu) >> (b+1) <= floor(x/q), error <= 2.
BC_DEV uint64_t mul_mod(uint64_t a, uint64_t b, const Mod &M) {
    uint64_t lo = a * b;
    uint64_t hi = __umul64hi(a, b);
    uint32_t s = M.b - 1;
    uint64_t x1 = (lo >> s) | (hi << (64 - s));
    uint64_t plo = x1 * M.mu;
    uint64_t phi = __umul64hi(x1, M.mu);
    uint32_t t = M.b + 1;
    uint64_t qhat = (plo >> t) | (phi << (64 - t));
    uint64_t r = lo - qhat * M.q;
    if (r >= M.q) r -= M.q;
    if (r >= M.q) r -= M.q;
    return r;
}

// reduce an arbitrary 64-bit value mod q (q < 2^62): x < 2^64 < 2^(2b) since b >= 33
BC_DEV uint64_t reduce64(uint64_t x, const Mod &M) {
    uint32_t s = M.b - 1;
    uint64_t x1 = x >> s;
    uint64_t plo = x1 * M.mu;
    uint64_t phi = __umul64hi(x1, M.mu);
    uint32_t t = M.b + 1;
    uint64_t qhat = (plo >> t) | (phi << (64 - t));
    uint64_t r = x - qhat * M.q;
    if (r >= M.q) r -= M.q;
    if (r >= M.q) r -= M.q;
    return r;
}

// signed small integer -> residue
BC_DEV uint64_t from_signed(int64_t v, uint64_t q) {
    if (v >= 0) return (uint64_t)v % q;
    uint64_t a = (uint64_t)(-v) % q;
    return a ? q - a : 0;
}

}  // namespace bc
