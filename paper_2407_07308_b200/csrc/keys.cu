// keys.cu -- keygen / encrypt / decrypt at the boundary (R6-R10), all arithmetic on the GPU.
#include <algorithm>
#include <cstring>

#include "engine.h"

using namespace bc;

namespace bc {

enum { TAG_S = 1, TAG_PK_A = 2, TAG_PK_E = 3, TAG_KS_A = 4, TAG_KS_E = 5, TAG_ENC_U = 6, TAG_ENC_E0 = 7, TAG_ENC_E1 = 8 };

__global__ void k_enc_combine(const Mod *__restrict__ mods, const uint64_t *__restrict__ pk,
                              const uint64_t *__restrict__ u, const uint64_t *__restrict__ t0,
                              const uint64_t *__restrict__ t1, uint64_t *__restrict__ out, uint64_t total,
                              uint32_t L1, uint32_t n) {
    const uint64_t ln = (uint64_t)L1 * n;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t b = i / ln, r = i - b * ln;
        const uint32_t limb = (uint32_t)(r / n);
        const Mod M = mods[limb];
        const uint64_t uu = u[i];
        out[b * 2 * ln + r] = add_mod(mul_mod(pk[r], uu, M), t0[i], M.q);
        out[b * 2 * ln + ln + r] = add_mod(mul_mod(pk[ln + r], uu, M), t1[i], M.q);
    }
}

// b = e - a (.) s over limbs [0, nl)  (all single polys, eval)
__global__ void k_rlwe_b(const Mod *__restrict__ mods, const uint64_t *__restrict__ a, const uint64_t *__restrict__ s,
                         const uint64_t *__restrict__ e, uint64_t *__restrict__ b, uint64_t total, uint32_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        const Mod M = mods[i / n];
        b[i] = sub_mod(e[i], mul_mod(a[i], s[i], M), M.q);
    }
}

// b[i] += c_i * sp[i] on limbs [l0, l1)
__global__ void k_axpy_limbs(const Mod *__restrict__ mods, uint64_t *__restrict__ b, const uint64_t *__restrict__ sp,
                             const uint64_t *__restrict__ c, uint32_t l0, uint32_t l1, uint32_t n) {
    const uint64_t total = (uint64_t)(l1 - l0) * n;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t limb = l0 + (uint32_t)(i / n);
        const uint64_t idx = (uint64_t)l0 * n + i;
        const Mod M = mods[limb];
        b[idx] = add_mod(b[idx], mul_mod(sp[idx], c[limb - l0], M), M.q);
    }
}

static unsigned gsz(uint64_t total) { return (unsigned)std::min<uint64_t>((total + 255) / 256, 148 * 32); }

}  // namespace bc

extern "C" {

bc_status bc_keygen(bc_ctx *X, uint64_t seed, bc_sk **skout, bc_keys **kout) {
    try {
        if (!X || !skout || !kout) BC_THROW(BC_E_ARG, "null argument");
        CK(cudaSetDevice(X->device));
        cudaStream_t st = 0;
        const uint32_t n = X->n, L1 = X->L1, K = X->K, NP = L1 + K;
        const uint64_t pw = (uint64_t)NP * n;
        // temporary workspace
        size_t need = (pw * 6 + (uint64_t)NP * X->M) * 8 + (1 << 20);
        void *ws = nullptr;
        CK(cudaMalloc(&ws, need));
        Arena A;
        A.init(ws, need, false);
        Eng E{X, nullptr, &A, st};
        bc_sk *sk = new bc_sk();
        bc_keys *keys = new bc_keys();
        auto dalloc = [&](size_t words) {
            void *p = nullptr;
            CK(cudaMalloc(&p, words * 8));
            keys->owned.push_back(p);
            return (uint64_t *)p;
        };
        BufP s = E.alloc_words(pw), a = E.alloc_words(pw), e = E.alloc_words(pw), sp = E.alloc_words(pw);
        uint64_t *S_ = (uint64_t *)s->p, *A_ = (uint64_t *)a->p, *E_ = (uint64_t *)e->p, *SP = (uint64_t *)sp->p;
        // secret s (ternary, coefficient form on every QP limb) -> eval
        sample_small(X->d_mods, seed, TAG_S, 0, 0, 0, 1, nullptr, S_, 1, NP, 0, n, pw, st);
        {
            std::vector<uint64_t> h(n);
            CK(cudaMemcpy(h.data(), S_, n * 8, cudaMemcpyDeviceToHost));
            sk->s.resize(n);
            for (uint32_t i = 0; i < n; ++i) sk->s[i] = h[i] == 0 ? 0 : (h[i] == 1 ? 1 : -1);
        }
        E.ntt_fwd(S_, S_, 1, limbmap_plain(NP, 0), pw, pw);
        CK(cudaMalloc((void **)&sk->d_s, pw * 8));
        CK(cudaMemcpyAsync(sk->d_s, S_, pw * 8, cudaMemcpyDeviceToDevice, st));
        // public key over the cipher primes: (b, a), b = p e - a s
        keys->d_pk = dalloc((uint64_t)2 * L1 * n);
        sample_uniform(X->d_mods, seed, TAG_PK_A, 0, 0, A_, 1, limbmap_plain(L1, 0), n, pw, st);
        E.ntt_fwd(A_, A_, 1, limbmap_plain(L1, 0), pw, pw);
        sample_small(X->d_mods, seed, TAG_PK_E, 0, 0, 1, (int64_t)X->p, nullptr, E_, 1, L1, 0, n, pw, st);
        E.ntt_fwd(E_, E_, 1, limbmap_plain(L1, 0), pw, pw);
        k_rlwe_b<<<gsz((uint64_t)L1 * n), 256, 0, st>>>(X->d_mods, A_, S_, E_, keys->d_pk, (uint64_t)L1 * n, n);
        CK(cudaMemcpyAsync(keys->d_pk + (uint64_t)L1 * n, A_, (uint64_t)L1 * n * 8, cudaMemcpyDeviceToDevice, st));
        // switching keys (R8): swk_j = (-a_j s + p e_j + [i in G_j] (P mod q_i) s', a_j)
        std::vector<uint64_t> Pmod(L1);
        for (uint32_t i = 0; i < L1; ++i) {
            uint64_t q = X->moduli[i], P = 1;
            for (uint32_t k = 0; k < K; ++k) P = mulmod_h(P, X->moduli[L1 + k] % q, q);
            Pmod[i] = P;
        }
        uint64_t *d_Pmod = nullptr;
        CK(cudaMalloc((void **)&d_Pmod, L1 * 8));
        CK(cudaMemcpy(d_Pmod, Pmod.data(), L1 * 8, cudaMemcpyHostToDevice));
        std::vector<uint32_t> ids{0};
        ids.insert(ids.end(), X->galois.begin(), X->galois.end());
        for (uint32_t t : ids) {
            if (t == 0) ew_ptmul(X->d_mods, S_, S_, SP, 1, 1, NP, n, st);
            else ew_automorph(X->T, S_, SP, 1, 1, NP, t, st);
            uint64_t *key = dalloc((uint64_t)X->dnum * 2 * pw);
            for (uint32_t j = 0; j < X->dnum; ++j) {
                uint64_t *kb = key + (uint64_t)j * 2 * pw, *ka = kb + pw;
                const uint64_t stream = (uint64_t)t * 64 + j;
                sample_uniform(X->d_mods, seed, TAG_KS_A, stream, 0, ka, 1, limbmap_plain(NP, 0), n, pw, st);
                E.ntt_fwd(ka, ka, 1, limbmap_plain(NP, 0), pw, pw);
                sample_small(X->d_mods, seed, TAG_KS_E, stream, 0, 1, (int64_t)X->p, nullptr, E_, 1, NP, 0, n, pw, st);
                E.ntt_fwd(E_, E_, 1, limbmap_plain(NP, 0), pw, pw);
                k_rlwe_b<<<gsz(pw), 256, 0, st>>>(X->d_mods, ka, S_, E_, kb, pw, n);
                const uint32_t g0 = j * X->alpha, g1 = std::min(L1, (j + 1) * X->alpha);
                k_axpy_limbs<<<gsz((uint64_t)(g1 - g0) * n), 256, 0, st>>>(X->d_mods, kb, SP, d_Pmod + g0, g0, g1, n);
            }
            keys->ksk[t] = key;
        }
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(st));
        cudaFree(d_Pmod);
        s.reset(); a.reset(); e.reset(); sp.reset();
        cudaFree(ws);
        *skout = sk;
        *kout = keys;
    } catch (BcError &e) {
        last_error() = e.msg;
        return e.st;
    } catch (std::exception &e) {
        last_error() = e.what();
        return BC_E_INTERNAL;
    }
    return BC_OK;
}

void bc_sk_destroy(bc_sk *sk) {
    if (!sk) return;
    cudaFree(sk->d_s);
    delete sk;
}
void bc_keys_destroy(bc_keys *k) {
    if (!k) return;
    for (void *p : k->owned) cudaFree(p);
    delete k;
}

static bc_status encrypt_impl(bc_ctx *X, const bc_keys *keys, const int16_t *h_slots, uint32_t B, uint64_t seed,
                              uint64_t ct0, bc_ct out, void *ws, size_t wsb, void *stv) {
    try {
        if (!X || !keys || !h_slots || !out.data) BC_THROW(BC_E_ARG, "null argument");
        if (out.level != X->L1 || out.batch < B) BC_THROW(BC_E_LEVEL, "encrypt: output must be top level");
        cudaStream_t st = (cudaStream_t)stv;
        const uint32_t n = X->n, L1 = X->L1;
        const uint64_t cw = (uint64_t)L1 * n;
        // process in chunks that fit the workspace (per ct: slots, m~, u/t0/t1, NTT scratch)
        const size_t sd = (size_t)X->alg.S * X->alg.D;
        const size_t per = sd * 2 + (size_t)n * 2 + cw * 8 * 3 + (size_t)L1 * X->M * 8 + 4 * 256;
        const size_t fixed = (size_t)n * (1 + 4) * 1 + (1 << 20);
        if (wsb < per + fixed) BC_THROW(BC_E_OOM, "encrypt: workspace too small");
        const uint32_t chunk = (uint32_t)std::max<size_t>(1, std::min<size_t>(B, (wsb - fixed) / (per + (size_t)n * 5)));
        for (uint32_t b0 = 0; b0 < B; b0 += chunk) {
            const uint32_t nb = std::min(chunk, B - b0);
            Arena A;
            A.init(ws, wsb, false);
            Eng E{X, keys, &A, st};
            BufP sl(new Buf{&A, A.alloc((size_t)nb * sd * 2), (size_t)nb * sd * 2});
            BufP mt(new Buf{&A, A.alloc((size_t)nb * n * 2), (size_t)nb * n * 2});
            CK(cudaMemcpyAsync(sl->p, h_slots + (size_t)b0 * sd, (size_t)nb * sd * 2, cudaMemcpyHostToDevice, st));
            encode_slots_dev(X, (int16_t *)sl->p, nb, (int16_t *)mt->p, &A, st);
            BufP u = E.alloc_words((uint64_t)nb * cw), t0 = E.alloc_words((uint64_t)nb * cw), t1 = E.alloc_words((uint64_t)nb * cw);
            sample_small(X->d_mods, seed, TAG_ENC_U, ct0 + b0, 1, 0, 1, nullptr, (uint64_t *)u->p, nb, L1, 0, n, cw, st);
            sample_small(X->d_mods, seed, TAG_ENC_E0, ct0 + b0, 1, 1, (int64_t)X->p, (int16_t *)mt->p, (uint64_t *)t0->p, nb,
                         L1, 0, n, cw, st);
            sample_small(X->d_mods, seed, TAG_ENC_E1, ct0 + b0, 1, 1, (int64_t)X->p, nullptr, (uint64_t *)t1->p, nb, L1, 0, n,
                         cw, st);
            E.ntt_fwd((uint64_t *)u->p, (uint64_t *)u->p, nb, limbmap_plain(L1, 0), cw, cw);
            E.ntt_fwd((uint64_t *)t0->p, (uint64_t *)t0->p, nb, limbmap_plain(L1, 0), cw, cw);
            E.ntt_fwd((uint64_t *)t1->p, (uint64_t *)t1->p, nb, limbmap_plain(L1, 0), cw, cw);
            const uint64_t total = (uint64_t)nb * cw;
            k_enc_combine<<<gsz(total), 256, 0, st>>>(X->d_mods, keys->d_pk, (uint64_t *)u->p, (uint64_t *)t0->p,
                                                     (uint64_t *)t1->p, (uint64_t *)out.data + (uint64_t)b0 * 2 * cw, total, L1, n);
            launch_counter() += 1;
            CK(cudaGetLastError());
            CK(cudaStreamSynchronize(st));
        }
    } catch (BcError &e) {
        last_error() = e.msg;
        return e.st;
    } catch (std::exception &e) {
        last_error() = e.what();
        return BC_E_INTERNAL;
    }
    return BC_OK;
}

bc_status bc_encrypt_slots(bc_ctx *X, const bc_keys *keys, const int16_t *h_slots, uint32_t batch, uint64_t seed,
                           uint64_t ct_index0, bc_ct out, void *ws, size_t wsb, void *st) {
    return encrypt_impl(X, keys, h_slots, batch, seed, ct_index0, out, ws, wsb, st);
}

// R6: word j -> slots w0 .. w0+l-1, w0 = word_slot(j) (row-aligned; j*l when cyclic);
// slot w0+s coefficient i = digit s*d + i (little-endian)
bc_status bc_encrypt(bc_ctx *X, const bc_keys *keys, const uint64_t *h_words, uint32_t batch, uint64_t seed,
                     uint64_t ct_index0, bc_ct out, void *ws, size_t wsb, void *st) {
    if (!X || !h_words) { last_error() = "null argument"; return BC_E_ARG; }
    const uint32_t S = X->alg.S, D = X->alg.D, d = X->d, l = X->l, ints = X->ints;
    const uint64_t base = X->base;
    // capacity base^(d l) (saturating)
    unsigned __int128 cap = 1;
    bool inf = false;
    for (uint32_t i = 0; i < d * l; ++i) {
        cap *= base;
        if (cap > ((unsigned __int128)1 << 64)) { inf = true; break; }
    }
    std::vector<int16_t> slots((size_t)batch * S * D, 0);
    for (uint32_t b = 0; b < batch; ++b)
        for (uint32_t j = 0; j < ints; ++j) {
            uint64_t x = h_words[(size_t)b * ints + j];
            if (!inf && (unsigned __int128)x >= cap) { last_error() = "word out of range"; return BC_E_RANGE; }
            for (uint32_t s = 0; s < l; ++s)
                for (uint32_t i = 0; i < d; ++i) {
                    slots[((size_t)b * S + X->alg.word_slot(j, l) + s) * D + i] = (int16_t)(x % base);
                    x /= base;
                }
        }
    return encrypt_impl(X, keys, slots.data(), batch, seed, ct_index0, out, ws, wsb, st);
}

// decrypt to centered plaintext coefficients (int16 [B][n]) on the device
static void decrypt_coeffs(bc_ctx *X, const bc_sk *sk, const bc_ct &in, Arena &A, cudaStream_t st, int16_t *d_out) {
    const uint32_t n = X->n, lv = in.level, B = in.batch;
    Eng E{X, nullptr, &A, st};
    BufP x = E.alloc_words((uint64_t)B * lv * n);
    dec_dot(X->d_mods, (uint64_t *)in.data, sk->d_s, (uint64_t *)x->p, B, lv, n, st);
    E.ntt_inv((uint64_t *)x->p, (uint64_t *)x->p, B, limbmap_plain(lv, 0), (uint64_t)lv * n, (uint64_t)lv * n);
    lift(X->plan("dec:" + std::to_string(lv)), X->d_mods, X->p, (uint64_t *)x->p, (uint64_t)lv * n, nullptr, 0, d_out, B, n,
         0, 0, 2, st);
}

static bc_status decrypt_impl(bc_ctx *X, const bc_sk *sk, bc_ct in, void *ws, size_t wsb, void *stv, int16_t *h_coef,
                              int16_t *h_slots) {
    try {
        if (!X || !sk || !in.data) BC_THROW(BC_E_ARG, "null argument");
        if (in.level < 1 || in.level > X->L1) BC_THROW(BC_E_LEVEL, "bad level");
        cudaStream_t st = (cudaStream_t)stv;
        const uint32_t n = X->n;
        const size_t per = (size_t)in.level * n * 8 + (size_t)n * (2 + 1 + 4 + 2) + (size_t)in.level * X->M * 8 + 2048;
        if (wsb < per + (1 << 20)) BC_THROW(BC_E_OOM, "decrypt: workspace too small");
        const uint32_t chunk = (uint32_t)std::max<size_t>(1, std::min<size_t>(in.batch, (wsb - (1 << 20)) / per));
        for (uint32_t b0 = 0; b0 < in.batch; b0 += chunk) {
            const uint32_t nb = std::min(chunk, in.batch - b0);
            Arena A;
            A.init(ws, wsb, false);
            bc_ct v{(uint64_t *)in.data + (uint64_t)b0 * 2 * in.level * n, nb, in.level};
            BufP c16(new Buf{&A, A.alloc((size_t)nb * n * 2), (size_t)nb * n * 2});
            decrypt_coeffs(X, sk, v, A, st, (int16_t *)c16->p);
            if (h_coef) CK(cudaMemcpyAsync(h_coef + (size_t)b0 * n, c16->p, (size_t)nb * n * 2, cudaMemcpyDeviceToHost, st));
            if (h_slots) {
                BufP a8(new Buf{&A, A.alloc((size_t)nb * n), (size_t)nb * n});
                BufP c32(new Buf{&A, A.alloc((size_t)nb * n * 4), (size_t)nb * n * 4});
                BufP o16(new Buf{&A, A.alloc((size_t)nb * n * 2), (size_t)nb * n * 2});
                s16_to_s8((int16_t *)c16->p, (int8_t *)a8->p, (uint64_t)nb * n, (int32_t)X->p, st);
                gemm_s8((int8_t *)a8->p, X->d_Dm, (int32_t *)c32->p, nb, n, n, st);
                mod_p_center((int32_t *)c32->p, (int16_t *)o16->p, (uint64_t)nb * n, (int32_t)X->p, st);
                CK(cudaMemcpyAsync(h_slots + (size_t)b0 * n, o16->p, (size_t)nb * n * 2, cudaMemcpyDeviceToHost, st));
            }
            CK(cudaGetLastError());
            CK(cudaStreamSynchronize(st));
        }
        const int64_t p = X->p;
        auto canon = [p](int16_t *v, size_t cnt) { for (size_t i = 0; i < cnt; ++i) if (v[i] < 0) v[i] = (int16_t)(v[i] + p); };
        if (h_coef) canon(h_coef, (size_t)in.batch * n);
        if (h_slots) canon(h_slots, (size_t)in.batch * n);
    } catch (BcError &e) {
        last_error() = e.msg;
        return e.st;
    } catch (std::exception &e) {
        last_error() = e.what();
        return BC_E_INTERNAL;
    }
    return BC_OK;
}

bc_status bc_decrypt_slots(bc_ctx *X, const bc_sk *sk, bc_ct in, int16_t *h_slots, void *ws, size_t wsb, void *st) {
    return decrypt_impl(X, sk, in, ws, wsb, st, nullptr, h_slots);
}

bc_status bc_decrypt_poly(bc_ctx *X, const bc_sk *sk, bc_ct in, int64_t *h_out, void *ws, size_t wsb, void *st) {
    if (!X || !h_out) { last_error() = "null argument"; return BC_E_ARG; }
    std::vector<int16_t> c((size_t)in.batch * X->n);
    bc_status s = decrypt_impl(X, sk, in, ws, wsb, st, c.data(), nullptr);
    if (s != BC_OK) return s;
    for (size_t i = 0; i < c.size(); ++i) h_out[i] = c[i];
    return BC_OK;
}

bc_status bc_decrypt(bc_ctx *X, const bc_sk *sk, bc_ct in, uint64_t *h_out, int as_bits, void *ws, size_t wsb, void *st) {
    if (!X || !h_out) { last_error() = "null argument"; return BC_E_ARG; }
    const uint32_t S = X->alg.S, D = X->alg.D, d = X->d, l = X->l, ints = X->ints;
    std::vector<int16_t> sl((size_t)in.batch * X->n);
    bc_status s = decrypt_impl(X, sk, in, ws, wsb, st, nullptr, sl.data());
    if (s != BC_OK) return s;
    for (uint32_t b = 0; b < in.batch; ++b)
        for (uint32_t j = 0; j < ints; ++j) {
            const int16_t *blk = sl.data() + ((size_t)b * S + (size_t)X->alg.word_slot(j, l)) * D;
            if (as_bits) { h_out[(size_t)b * ints + j] = (uint64_t)blk[0]; continue; }
            unsigned __int128 x = 0, w = 1;
            for (uint32_t si = 0; si < l; ++si)
                for (uint32_t i = 0; i < d; ++i) {
                    x += w * (unsigned __int128)blk[(size_t)si * D + i];
                    w *= X->base;
                }
            h_out[(size_t)b * ints + j] = (uint64_t)x;
        }
    return BC_OK;
}

}  // extern "C"
