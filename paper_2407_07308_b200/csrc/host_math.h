// host_math.h -- host-side number theory and slot algebra of the product path.
// Independent implementation (shares no code with oracle/).  Definitions: DESIGN.md §3
// readings R1 (prime chain), R2 (omega), R5 (slot algebra), R6 (integer encoding).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace bc {

typedef unsigned __int128 u128;

inline uint64_t mulmod_h(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)((u128)a * b % q); }
uint64_t powmod_h(uint64_t a, uint64_t e, uint64_t q);
uint64_t invmod_h(uint64_t a, uint64_t q);          // q prime
uint64_t invmod_h_any(uint64_t a, uint64_t m);      // gcd(a, m) = 1, any m
bool is_prime_u64(uint64_t n);
std::vector<uint64_t> prime_factors(uint64_t n);     // distinct, trial division
uint64_t gcd_u64(uint64_t a, uint64_t b);
uint64_t mult_order(uint64_t a, uint64_t m);

// R1: `count` smallest primes >= max(2^(bits-1), after+1), q = 1 mod modulus.
std::vector<uint64_t> prime_chain(uint64_t modulus, int bits, int count, uint64_t after, uint64_t exclude);
// R2: omega = h^((q-1)/m) for the smallest h >= 2 giving exact order m.
uint64_t root_of_order(uint64_t order, uint64_t q);

// Phi_m over Z, coefficients low -> high (length phi(m)+1).
std::vector<int64_t> cyclotomic(uint32_t m);

// ---- F_p polynomials (low -> high) ----
typedef std::vector<int64_t> Poly;
Poly p_trim(Poly a);
Poly p_mul(const Poly &a, const Poly &b, int64_t p);
Poly p_mod(const Poly &a, const Poly &b, int64_t p);
Poly p_divexact(const Poly &a, const Poly &b, int64_t p);

// ---- F_{p^D} = F_p[X]/G ----
struct GF {
    int64_t p;
    int D;
    Poly G;  // monic, degree D
    std::vector<int64_t> mul(const std::vector<int64_t> &a, const std::vector<int64_t> &b) const;
    std::vector<int64_t> pow(std::vector<int64_t> a, unsigned __int128 e) const;
    std::vector<int64_t> one() const;
    bool is_one(const std::vector<int64_t> &a) const;
};

struct SlotAlgebra {
    int64_t p;
    uint32_t m, n, D, S;
    GF gf;
    std::vector<int64_t> zeta;          // D coefficients
    uint32_t g;                          // slot generator (rotations; rows of S1 slots)
    uint32_t S1 = 0, g2 = 1, S2 = 1;     // hypercube: slot s = j*S1 + i <-> g^i g2^j (cyclic: S1 = S)
    std::vector<uint32_t> t;             // t_s
    uint32_t words_per_row(uint32_t l) const { return S1 / l; }
    uint32_t word_slot(uint32_t w, uint32_t l) const { return (w / (S1 / l)) * S1 + (w % (S1 / l)) * l; }
    std::vector<int64_t> zpow;           // [m][D]: zeta^e
    std::vector<std::vector<int64_t>> E0;  // [D][n]: slot-0 idempotent basis, E0_i(zeta) = X^i
    std::vector<std::vector<int64_t>> kappa;  // [d*D][D]: kappa_{i,k} = mu_i^{p^k} (F_{p^D} values)
    std::string error;
    bool build(int64_t p, uint32_t m, const std::vector<int64_t> &phi, uint32_t dmax);
};

}  // namespace bc
