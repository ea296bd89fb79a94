/*
 * oracle/ring_c.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct helpers for the CPU oracle of the BoostCom
 * BGV comparison path (arXiv 2407.07308).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load this library.  It shares no code
 * with the CUDA product path (paper_2407_07308_b200/).
 *
 * Everything here is a textbook definition written out:
 *   ring_mul   : schoolbook product, fold mod x^m - 1, division by Phi_m (§2.1)
 *   poly_mod_phi: long division by the monic integer polynomial Phi_m
 *   eval_naive : E[k] = f(omega^{z_k}) for z_k in Z_m^* ascending     (§2.2)
 *   vec_mulmod : element-wise (a*b) mod q
 * Products use unsigned __int128 and the '%' operator; q < 2^62, and a sum is reduced before
 * it could exceed 2^128 (at most 2^(128 - 2 bits(q)) - 1 products per reduction).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

static uint64_t submod(uint64_t a, uint64_t b, uint64_t q) { return a >= b ? a - b : a + q - b; }

/* reduce t[0..len) (residues mod q) modulo the monic Phi (degree n, coeffs phi[0..n],
 * phi[n] == 1, small signed integers) in place; result in t[0..n). */
void poly_mod_phi(uint64_t *t, int len, const int64_t *phi, int n, uint64_t q)
{
    for (int k = len - 1; k >= n; --k) {
        uint64_t c = t[k] % q;
        if (c == 0) continue;
        /* t -= c * x^(k-n) * Phi */
        #pragma omp parallel for schedule(static) if (n > 4096)
        for (int j = 0; j <= n; ++j) {
            int64_t f = phi[j];
            if (f == 0) continue;
            uint64_t af = (uint64_t)(f < 0 ? -f : f) % q;
            uint64_t prod = (uint64_t)(((u128)c * af) % q);
            uint64_t *dst = &t[k - n + j];
            if (f > 0) *dst = submod(*dst % q, prod, q);
            else       *dst = (*dst % q + prod) % q;
        }
    }
}

/* out = a*b mod (q, Phi_m); a, b, out length n; phi length n+1.
 * Definition: schoolbook product over Z_q, fold mod x^m - 1 (exact:
 * Phi_m divides x^m - 1), then long division by Phi_m (m - n steps).  The u128 accumulator is
 * reduced only when the next term could overflow it: with q < 2^b every product is < 2^(2b), so
 * 2^(128-2b) - 1 terms fit (C2-C5: b = 50, every output coefficient is reduced once). */
void ring_mul(const uint64_t *a, const uint64_t *b, uint64_t *out, int n,
              const int64_t *phi, uint64_t q, int m)
{
    int len = 2 * n - 1;
    int bits = 64 - __builtin_clzll(q);
    int lim = 2 * bits >= 127 ? 1 : (2 * bits > 96 ? (int)((((u128)1) << (128 - 2 * bits)) - 1) : 1 << 30);
    uint64_t *t = (uint64_t *)calloc((size_t)(len > m ? len : m), sizeof(uint64_t));
    #pragma omp parallel for schedule(dynamic, 64)
    for (int k = 0; k < len; ++k) {
        int lo = k - (n - 1) > 0 ? k - (n - 1) : 0;
        int hi = k < n - 1 ? k : n - 1;
        u128 acc = 0;
        int cnt = 0;
        for (int i = lo; i <= hi; ++i) {
            acc += (u128)a[i] * b[k - i];
            if (++cnt == lim) { acc %= q; cnt = 0; }
        }
        t[k] = (uint64_t)(acc % q);
    }
    /* fold mod x^m - 1: x^k = x^(k-m) for k >= m */
    for (int k = m; k < len; ++k) {
        uint64_t s = t[k - m] + t[k];
        t[k - m] = s >= q ? s - q : s;
        t[k] = 0;
    }
    poly_mod_phi(t, m, phi, n, q);
    memcpy(out, t, (size_t)n * sizeof(uint64_t));
    free(t);
}

/* E[k] = sum_j f[j] * w^(j*z[k] mod m) mod q; wpow[e] = w^e mod q for e < m. */
void eval_naive(const uint64_t *f, int n, const int32_t *z, int nz, int m,
                const uint64_t *wpow, uint64_t q, uint64_t *out)
{
    #pragma omp parallel for schedule(static)
    for (int k = 0; k < nz; ++k) {
        u128 acc = 0;
        int cnt = 0;
        int64_t zk = z[k];
        for (int j = 0; j < n; ++j) {
            acc += (u128)f[j] * wpow[(int64_t)j * zk % m];
            if (++cnt == 8) { acc %= q; cnt = 0; }
        }
        out[k] = (uint64_t)(acc % q);
    }
}

void vec_mulmod(const uint64_t *a, const uint64_t *b, uint64_t *out, int64_t len, uint64_t q)
{
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < len; ++i) out[i] = (uint64_t)(((u128)a[i] * b[i]) % q);
}

/* out[i] = (a[i] * c) mod q for a scalar c < q */
void vec_mulscalar(const uint64_t *a, uint64_t c, uint64_t *out, int64_t len, uint64_t q)
{
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < len; ++i) out[i] = (uint64_t)(((u128)a[i] * c) % q);
}
