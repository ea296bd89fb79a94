// host_math.cpp -- host number theory and slot algebra (product path; see host_math.h).
#include "host_math.h"

#include <algorithm>
#include <set>
#include <stdexcept>

namespace bc {

uint64_t powmod_h(uint64_t a, uint64_t e, uint64_t q) {
    uint64_t r = 1 % q;
    a %= q;
    while (e) {
        if (e & 1) r = mulmod_h(r, a, q);
        a = mulmod_h(a, a, q);
        e >>= 1;
    }
    return r;
}

uint64_t invmod_h(uint64_t a, uint64_t q) { return powmod_h(a, q - 2, q); }

uint64_t invmod_h_any(uint64_t a, uint64_t m) {
    int64_t t = 0, nt = 1, r = (int64_t)m, nr = (int64_t)(a % m);
    while (nr) {
        int64_t qq = r / nr, tmp;
        tmp = t - qq * nt; t = nt; nt = tmp;
        tmp = r - qq * nr; r = nr; nr = tmp;
    }
    if (r != 1) throw std::runtime_error("invmod_h_any: not invertible");
    return (uint64_t)(t < 0 ? t + (int64_t)m : t);
}

uint64_t gcd_u64(uint64_t a, uint64_t b) {
    while (b) { uint64_t t = a % b; a = b; b = t; }
    return a;
}

bool is_prime_u64(uint64_t n) {
    if (n < 2) return false;
    static const uint64_t bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    for (uint64_t b : bases) if (n % b == 0) return n == b;
    uint64_t d = n - 1;
    int s = 0;
    while ((d & 1) == 0) { d >>= 1; ++s; }
    for (uint64_t a : bases) {
        uint64_t x = powmod_h(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool comp = true;
        for (int r = 1; r < s; ++r) {
            x = mulmod_h(x, x, n);
            if (x == n - 1) { comp = false; break; }
        }
        if (comp) return false;
    }
    return true;
}

std::vector<uint64_t> prime_factors(uint64_t n) {
    std::vector<uint64_t> f;
    for (uint64_t d = 2; d * d <= n; ++d) {
        if (n % d == 0) { f.push_back(d); while (n % d == 0) n /= d; }
    }
    if (n > 1) f.push_back(n);
    return f;
}

uint64_t mult_order(uint64_t a, uint64_t m) {
    uint64_t k = 1, x = a % m;
    while (x != 1) { x = x * a % m; ++k; }
    return k;
}

std::vector<uint64_t> prime_chain(uint64_t modulus, int bits, int count, uint64_t after, uint64_t exclude) {
    uint64_t start = std::max<uint64_t>(1ull << (bits - 1), after + 1);
    uint64_t q = start + ((modulus - (start - 1) % modulus) % modulus);  // q = 1 mod modulus, q >= start
    std::vector<uint64_t> out;
    while ((int)out.size() < count) {
        if (q >= (1ull << 62)) throw std::runtime_error("NotEnoughPrimes below 2^62");
        if (q != exclude && is_prime_u64(q)) out.push_back(q);
        q += modulus;
    }
    return out;
}

uint64_t root_of_order(uint64_t order, uint64_t q) {
    if ((q - 1) % order) throw std::runtime_error("OrderNotDividing");
    std::vector<uint64_t> pf = prime_factors(order);
    for (uint64_t h = 2;; ++h) {
        uint64_t w = powmod_h(h, (q - 1) / order, q);
        bool ok = true;
        for (uint64_t r : pf) if (powmod_h(w, order / r, q) == 1) { ok = false; break; }
        if (ok) return w;
    }
}

// Phi_m = prod_{d | m} (x^d - 1)^{mu(m/d)}: multiply by the mu=+1 binomials, then divide
// exactly by the mu=-1 binomials (both sparse operations).
static int mobius(uint32_t n) {
    int k = 0;
    for (uint32_t d = 2; d * d <= n; ++d) {
        if (n % d == 0) {
            n /= d;
            if (n % d == 0) return 0;
            ++k;
        }
    }
    if (n > 1) ++k;
    return (k & 1) ? -1 : 1;
}

std::vector<int64_t> cyclotomic(uint32_t m) {
    std::vector<int64_t> poly{1};
    std::vector<uint32_t> dens;
    for (uint32_t d = 1; d <= m; ++d) {
        if (m % d) continue;
        int mu = mobius(m / d);
        if (mu == 1) {  // poly *= (x^d - 1)
            std::vector<int64_t> r(poly.size() + d, 0);
            for (size_t i = 0; i < poly.size(); ++i) { r[i + d] += poly[i]; r[i] -= poly[i]; }
            poly.swap(r);
        } else if (mu == -1) {
            dens.push_back(d);
        }
    }
    for (uint32_t d : dens) {  // poly /= (x^d - 1): q_k = -(a_k) + q_{k-d}... synthetic division
        size_t deg = poly.size() - 1;
        std::vector<int64_t> qt(deg - d + 1, 0);
        std::vector<int64_t> a = poly;
        for (size_t k = deg; k >= d; --k) {
            int64_t c = a[k];
            qt[k - d] = c;
            a[k] -= c;
            a[k - d] += c;
            if (k == d) break;
        }
        for (size_t k = 0; k < d; ++k) if (a[k] != 0) throw std::runtime_error("cyclotomic: inexact");
        poly.swap(qt);
    }
    return poly;
}

// ---------------------------------------------------------------- F_p polynomials
Poly p_trim(Poly a) {
    while (a.size() > 1 && a.back() == 0) a.pop_back();
    return a;
}

Poly p_mul(const Poly &a, const Poly &b, int64_t p) {
    Poly r(a.size() + b.size() - 1, 0);
    for (size_t i = 0; i < a.size(); ++i) {
        if (!a[i]) continue;
        for (size_t j = 0; j < b.size(); ++j) r[i + j] = (r[i + j] + a[i] * b[j]) % p;
    }
    return p_trim(r);
}

Poly p_mod(const Poly &a0, const Poly &b0, int64_t p) {
    Poly a = a0, b = p_trim(b0);
    for (auto &x : a) x = ((x % p) + p) % p;
    size_t db = b.size() - 1;
    if (a.size() <= db) return p_trim(a);
    int64_t inv = (int64_t)powmod_h((uint64_t)((b[db] % p + p) % p), p - 2, p);
    for (size_t k = a.size() - 1; k >= db; --k) {
        int64_t c = a[k] * inv % p;
        if (c) for (size_t j = 0; j <= db; ++j) a[k - db + j] = ((a[k - db + j] - c * b[j]) % p + p) % p;
        if (k == db) break;
    }
    a.resize(std::max<size_t>(db, 1));
    return p_trim(a);
}

Poly p_divexact(const Poly &a0, const Poly &b, int64_t p) {  // b monic
    Poly a = a0;
    for (auto &x : a) x = ((x % p) + p) % p;
    size_t db = b.size() - 1;
    Poly qt(a.size() - db, 0);
    for (size_t k = a.size() - 1; k >= db; --k) {
        int64_t c = a[k];
        qt[k - db] = c;
        if (c) for (size_t j = 0; j <= db; ++j) a[k - db + j] = ((a[k - db + j] - c * b[j]) % p + p) % p;
        if (k == db) break;
    }
    for (size_t k = 0; k < db; ++k) if (a[k]) throw std::runtime_error("p_divexact: remainder");
    return qt;
}

static Poly p_powmod(Poly base, uint64_t e, const Poly &mod, int64_t p) {
    Poly r{1};
    base = p_mod(base, mod, p);
    while (e) {
        if (e & 1) r = p_mod(p_mul(r, base, p), mod, p);
        base = p_mod(p_mul(base, base, p), mod, p);
        e >>= 1;
    }
    return r;
}

static Poly p_sub(Poly a, Poly b, int64_t p) {
    size_t n = std::max(a.size(), b.size());
    a.resize(n, 0); b.resize(n, 0);
    for (size_t i = 0; i < n; ++i) a[i] = ((a[i] - b[i]) % p + p) % p;
    return p_trim(a);
}

static Poly p_gcd(Poly a, Poly b, int64_t p) {
    a = p_trim(a); b = p_trim(b);
    while (!(b.size() == 1 && b[0] == 0)) { Poly r = p_mod(a, b, p); a = b; b = r; }
    return a;
}

// Rabin: X^{p^D} = X mod G and gcd(X^{p^{D/r}} - X, G) = 1 for every prime r | D.
static bool irreducible(const Poly &G, int64_t p) {
    int D = (int)G.size() - 1;
    Poly X{0, 1};
    auto frob = [&](int k) { Poly y = X; for (int i = 0; i < k; ++i) y = p_powmod(y, p, G, p); return y; };
    if (p_sub(frob(D), X, p) != Poly{0}) return false;
    for (uint64_t r : prime_factors(D)) {
        Poly g = p_gcd(G, p_sub(frob(D / (int)r), X, p), p);
        if (g.size() > 1) return false;
    }
    return true;
}

// ---------------------------------------------------------------- F_{p^D}
std::vector<int64_t> GF::one() const { std::vector<int64_t> e(D, 0); e[0] = 1; return e; }
bool GF::is_one(const std::vector<int64_t> &a) const {
    for (int i = 0; i < D; ++i) if (a[i] != (i == 0)) return false;
    return true;
}
std::vector<int64_t> GF::mul(const std::vector<int64_t> &a, const std::vector<int64_t> &b) const {
    std::vector<int64_t> r(2 * D - 1, 0);
    for (int i = 0; i < D; ++i) {
        if (!a[i]) continue;
        for (int j = 0; j < D; ++j) r[i + j] = (r[i + j] + a[i] * b[j]) % p;
    }
    for (int k = 2 * D - 2; k >= D; --k) {
        int64_t c = r[k];
        if (!c) continue;
        for (int j = 0; j < D; ++j) r[k - D + j] = ((r[k - D + j] - c * G[j]) % p + p) % p;
        r[k] = 0;
    }
    r.resize(D);
    return r;
}
std::vector<int64_t> GF::pow(std::vector<int64_t> a, unsigned __int128 e) const {
    std::vector<int64_t> r = one();
    while (e) {
        if (e & 1) r = mul(r, a);
        a = mul(a, a);
        e >>= 1;
    }
    return r;
}

// p^e exactly (p^D reaches 17^18 > 2^64 on the C5 shadow ring: 128-bit)
static unsigned __int128 ipow(uint64_t b, int e) { unsigned __int128 r = 1; while (e--) r *= b; return r; }

// solve V x = y over F_p (V: D x D, column-major list of columns)
static std::vector<int64_t> solve_fp(std::vector<std::vector<int64_t>> A, std::vector<int64_t> y, int64_t p) {
    int n = (int)y.size();
    for (int c = 0; c < n; ++c) {
        int piv = c;
        while (A[piv][c] % p == 0) ++piv;
        std::swap(A[piv], A[c]);
        std::swap(y[piv], y[c]);
        int64_t inv = (int64_t)powmod_h((uint64_t)((A[c][c] % p + p) % p), p - 2, p);
        for (int j = 0; j < n; ++j) A[c][j] = (A[c][j] * inv % p + p) % p;
        y[c] = (y[c] * inv % p + p) % p;
        for (int r = 0; r < n; ++r) {
            if (r == c || A[r][c] == 0) continue;
            int64_t f = A[r][c];
            for (int j = 0; j < n; ++j) A[r][j] = ((A[r][j] - f * A[c][j]) % p + p) % p;
            y[r] = ((y[r] - f * y[c]) % p + p) % p;
        }
    }
    return y;
}

bool SlotAlgebra::build(int64_t p_, uint32_t m_, const std::vector<int64_t> &phi, uint32_t dmax) {
    p = p_; m = m_; n = (uint32_t)phi.size() - 1;
    D = (uint32_t)mult_order((uint64_t)p, m);
    S = n / D;
    gf.p = p; gf.D = (int)D;
    // R5: G = X^D + sum c_i X^i with the smallest v = sum c_i p^i that is irreducible
    for (uint64_t v = 0;; ++v) {
        Poly G(D + 1, 0);
        uint64_t x = v;
        for (uint32_t i = 0; i < D; ++i) { G[i] = (int64_t)(x % p); x /= p; }
        G[D] = 1;
        if (D == 1 || irreducible(G, p)) { gf.G = G; break; }
    }
    // zeta = beta^((p^D-1)/m) for the first beta (v = 1, 2, ...) giving exact order m
    const unsigned __int128 pD = ipow((uint64_t)p, (int)D);
    std::vector<uint64_t> mf = prime_factors(m);
    for (uint64_t v = 1; (unsigned __int128)v < pD; ++v) {
        std::vector<int64_t> b(D, 0);
        uint64_t x = v;
        for (uint32_t i = 0; i < D; ++i) { b[i] = (int64_t)(x % p); x /= p; }
        std::vector<int64_t> z = gf.pow(b, (pD - 1) / m);
        bool ok = true;
        for (uint64_t r : mf) if (gf.is_one(gf.pow(z, m / r))) { ok = false; break; }
        if (ok) { zeta = z; break; }
    }
    if (zeta.empty()) { error = "no element of order m"; return false; }
    // R5 slot generators.  Quotient orders: the exponents k with t^k in <p> are the multiples of the
    // quotient order, so start from ord(t) (n divided by its primes while t^(o/r) = 1) and divide.
    std::set<uint32_t> H;
    for (uint32_t k = 0; k < D; ++k) H.insert((uint32_t)powmod_h((uint64_t)p, k, m));
    const std::vector<uint64_t> nf = prime_factors(n);
    auto qorder = [&](uint32_t tt) {
        uint64_t o = n;
        for (uint64_t r : nf) while (o % r == 0 && powmod_h(tt, o / r, m) == 1) o /= r;
        for (uint64_t r : nf) while (o % r == 0 && H.count((uint32_t)powmod_h(tt, o / r, m))) o /= r;
        return (uint32_t)o;
    };
    g = 0; g2 = 1; S1 = S; S2 = 1;
    uint32_t first_any = 0;
    if (S == 1) g = 1;
    // cyclic quotient: the smallest t of quotient order S with t^S = 1 (mod m), else the smallest of order S
    for (uint32_t tt = 2; tt < m && g == 0; ++tt) {
        if (gcd_u64(tt, m) != 1) continue;
        if (qorder(tt) != S) continue;
        if (!first_any) first_any = tt;
        if (powmod_h(tt, S, m) == 1) g = tt;
    }
    if (!g) g = first_any;
    if (!g) {
        // hypercube Z_S1 x Z_S2: S1 = the largest quotient order; g the smallest of that order, preferring
        // g^S1 = 1; g2 the smallest t outside <p, g> with t^S2 in <p, g> (and no smaller power), preferring t^S2 = 1
        std::vector<uint32_t> qo(m, 0);
        S1 = 0;
        for (uint32_t tt = 2; tt < m; ++tt)
            if (gcd_u64(tt, m) == 1) { qo[tt] = qorder(tt); S1 = std::max(S1, qo[tt]); }
        S2 = S / S1;
        uint32_t gf1 = 0;
        for (uint32_t tt = 2; tt < m && !g; ++tt) {
            if (qo[tt] != S1) continue;
            if (!gf1) gf1 = tt;
            if (powmod_h(tt, S1, m) == 1) g = tt;
        }
        if (!g) g = gf1;
        std::vector<char> inHg(m, 0);
        for (uint32_t k = 0; k < D; ++k)
            for (uint32_t i = 0; i < S1; ++i)
                inHg[powmod_h((uint64_t)p, k, m) * powmod_h(g, i, m) % m] = 1;
        uint32_t c2 = 0, good2 = 0;
        for (uint32_t tt = 2; tt < m && !good2; ++tt) {
            if (gcd_u64(tt, m) != 1 || inHg[tt]) continue;
            if (!inHg[powmod_h(tt, S2, m)]) continue;
            bool ok = true;
            for (uint32_t j = 1; j < S2 && ok; ++j) ok = !inHg[powmod_h(tt, j, m)];
            if (!ok) continue;
            if (!c2) c2 = tt;
            if (powmod_h(tt, S2, m) == 1) good2 = tt;
        }
        g2 = good2 ? good2 : c2;
        if (!g || !g2 || S1 * S2 != S) { error = "Z_m^*/<p> is not Z_S1 x Z_S2"; return false; }
        std::vector<char> cover(m, 0);
        uint64_t cnt = 0;
        for (uint32_t tt = 1; tt < m; ++tt)
            if (inHg[tt])
                for (uint32_t j = 0; j < S2; ++j) {
                    const uint64_t u = tt * powmod_h(g2, j, m) % m;
                    if (!cover[u]) { cover[u] = 1; ++cnt; }
                }
        if (cnt != n) { error = "Z_m^*/<p> is not generated by (p, g, g2)"; return false; }
    }
    t.resize(S);
    for (uint32_t s = 0; s < S; ++s) t[s] = (uint32_t)(powmod_h(g, s % S1, m) * powmod_h(g2, s / S1, m) % m);
    // zeta^e table
    zpow.assign((size_t)m * D, 0);
    std::vector<int64_t> x = gf.one();
    for (uint32_t e = 0; e < m; ++e) {
        for (uint32_t i = 0; i < D; ++i) zpow[(size_t)e * D + i] = x[i];
        x = gf.mul(x, zeta);
    }
    auto zp = [&](uint64_t e) { std::vector<int64_t> r(D); for (uint32_t i = 0; i < D; ++i) r[i] = zpow[(e % m) * D + i]; return r; };
    // slot-0 idempotent basis: F_0 = prod_k (x - zeta^{p^k}); H_0 = Phi_m / F_0 (mod p);
    // E0_i = H_0 * w_i with w_i(zeta) = X^i * H_0(zeta)^{-1}, deg w_i < D.
    std::vector<std::vector<int64_t>> F{gf.one()};
    for (uint32_t k = 0; k < D; ++k) {
        std::vector<int64_t> r = zp(powmod_h((uint64_t)p, k, m));
        std::vector<std::vector<int64_t>> nf(F.size() + 1, std::vector<int64_t>(D, 0));
        for (size_t i = 0; i < F.size(); ++i) {
            std::vector<int64_t> cr = gf.mul(F[i], r);
            for (uint32_t j = 0; j < D; ++j) {
                nf[i + 1][j] = (nf[i + 1][j] + F[i][j]) % p;
                nf[i][j] = ((nf[i][j] - cr[j]) % p + p) % p;
            }
        }
        F.swap(nf);
    }
    Poly F0(D + 1);
    for (uint32_t i = 0; i <= D; ++i) {
        for (uint32_t j = 1; j < D; ++j) if (F[i][j]) { error = "F_0 not over F_p"; return false; }
        F0[i] = F[i][0];
    }
    Poly phip(phi.size());
    for (size_t i = 0; i < phi.size(); ++i) phip[i] = ((phi[i] % p) + p) % p;
    Poly H0 = p_divexact(phip, F0, p);
    std::vector<int64_t> hval(D, 0);
    for (size_t e = 0; e < H0.size(); ++e) {
        if (!H0[e]) continue;
        std::vector<int64_t> ze = zp(e);
        for (uint32_t i = 0; i < D; ++i) hval[i] = (hval[i] + H0[e] * ze[i]) % p;
    }
    std::vector<int64_t> hinv = gf.pow(hval, pD - 2);
    std::vector<std::vector<int64_t>> V(D, std::vector<int64_t>(D));  // V[row i][col j] = coeff_i(zeta^j)
    for (uint32_t j = 0; j < D; ++j) { std::vector<int64_t> c = zp(j); for (uint32_t i = 0; i < D; ++i) V[i][j] = c[i]; }
    E0.assign(D, std::vector<int64_t>(n, 0));
    for (uint32_t i = 0; i < D; ++i) {
        std::vector<int64_t> Xi(D, 0);
        Xi[i] = 1;
        std::vector<int64_t> w = solve_fp(V, gf.mul(Xi, hinv), p);
        for (uint32_t a = 0; a < D; ++a) {
            if (!w[a]) continue;
            for (size_t e = 0; e < H0.size(); ++e) E0[i][a + e] = (E0[i][a + e] + w[a] * H0[e]) % p;
        }
    }
    // trace-dual basis of {X^i}: T[i][j] = Tr(X^{i+j}); mu_i solves T c = e_i (T symmetric)
    auto trace = [&](std::vector<int64_t> a) {
        std::vector<int64_t> s(D, 0);
        for (uint32_t k = 0; k < D; ++k) { for (uint32_t i = 0; i < D; ++i) s[i] = (s[i] + a[i]) % p; a = gf.pow(a, (uint64_t)p); }
        return s[0];
    };
    std::vector<std::vector<int64_t>> T(D, std::vector<int64_t>(D));
    for (uint32_t i = 0; i < D; ++i)
        for (uint32_t j = 0; j < D; ++j) {
            std::vector<int64_t> xi(D, 0), xj(D, 0);
            xi[i] = 1; xj[j] = 1;
            T[i][j] = trace(gf.mul(xi, xj));
        }
    kappa.clear();
    for (uint32_t i = 0; i < dmax; ++i) {
        std::vector<int64_t> e(D, 0);
        e[i] = 1;
        std::vector<int64_t> mu = solve_fp(T, e, p);
        for (uint32_t k = 0; k < D; ++k) kappa.push_back(gf.pow(mu, ipow((uint64_t)p, (int)k)));
    }
    return true;
}

}  // namespace bc
