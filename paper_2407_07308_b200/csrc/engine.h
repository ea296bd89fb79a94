// engine.h -- host orchestration of the batched BGV comparison path (product side).
#pragma once
#include <cuda_runtime.h>

#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/boostcom.h"
#include "host_math.h"
#include "kernels.h"

namespace bc {

std::string &last_error();

struct BcError {
    bc_status st;
    std::string msg;
};
#define BC_THROW(code, m) throw ::bc::BcError{code, m}
#define CK(x)                                                                                 \
    do {                                                                                      \
        cudaError_t e_ = (x);                                                                 \
        if (e_ != cudaSuccess) BC_THROW(BC_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// ---------------------------------------------------------------- workspace arena
struct Arena {
    char *base = nullptr;
    size_t cap = 0;
    bool dry = false;
    size_t used = 0, peak = 0;
    size_t hwm = 0;                  // high-water address: the capacity this allocation sequence needs
                                     // (best fit places identically in any arena at least this large)
    std::map<size_t, size_t> freel;  // offset -> size
    void init(void *b, size_t c, bool dry_);
    char *alloc(size_t bytes);
    void release(char *p, size_t bytes);
};
struct Buf {
    Arena *a;
    char *p;
    size_t sz;
    ~Buf() { if (a && p) a->release(p, sz); }
};
typedef std::shared_ptr<Buf> BufP;

// a batch of ciphertexts: u64[B][parts][lvl][n] (possibly a view into a larger buffer)
struct CT {
    BufP keep;
    uint64_t *d = nullptr;
    uint32_t B = 0, lvl = 0, parts = 2;
    uint64_t bstride = 0;  // words between consecutive ciphertexts
};

}  // namespace bc

// ---------------------------------------------------------------- context
struct bc_ctx {
    bc_params prm;
    int device = 0;
    uint32_t p, m, n, M, R, C, logR, logC, L1, K, alpha, dnum, d, l, base, ints;
    uint32_t rad = 1, logN = 0;       // R25 mixed-radix rows: C = rad 2^logN (rad = 1: C = 2^logC)
    bool prime_m;
    std::vector<uint64_t> moduli, omega;
    std::vector<int64_t> phi;
    bc::SlotAlgebra alg;
    std::vector<uint32_t> galois;     // Galois elements with keys (besides relin)
    // device
    std::vector<void *> owned;
    bc::Mod *d_mods = nullptr;
    const double2 *d_fm = nullptr;    // (q, fl(1/q)) per prime when all primes are in [2^49, 2^50) (binary64 kernels)
    bc::NttTables T;
    bc::NttTables Tb;                   // composite m: size-Mb tables of the two Barrett convolutions (T.tb)
    uint64_t *d_plans = nullptr;
    std::map<std::string, size_t> plan_off;
    std::map<std::string, std::pair<uint32_t, uint32_t>> plan_dims;   // (sources, targets)
    bc::u64x2 *d_invP = nullptr;                // [L1] P^{-1} mod q_i
    bc::u64x2 *d_invq = nullptr;                // [L1+1][L1] q_{l-1}^{-1} mod q_i (row l)
    bc::u64x2 *d_Pm = nullptr;                  // [L1] P mod q_i
    bc::u64x2 *d_invD = nullptr;                // [L1+1][L1] (P q_{l-1})^{-1} mod q_i (row l)
    int8_t *d_Em = nullptr, *d_Dm = nullptr;    // encode / decode matrices (n x n)
    int16_t *d_E0 = nullptr, *d_zpow = nullptr;
    uint32_t *d_ts = nullptr;
    int8_t *d_red = nullptr;
    std::map<std::string, uint64_t *> pt;       // encoded plaintext constants, eval [L1][n]
    std::mutex pt_mu;                           // guards pt: the circuit constants are built in
                                                // ctx_precompute_pt, compaction masks on first use
    // circuit coefficients
    std::vector<int64_t> lt_u, eq_u;            // univariate LT / EQ coefficients
    std::vector<std::vector<int64_t>> lt_b;     // bivariate c[j][k] (Y^j Z^k)
    int r23_k = 0;                              // R23 baby-step size (params schedule 23), 0 = R16 circuits
    int r26_k = 0;                              // R26 bivariate block sizes k1 << 8 | k2 (schedule 26), 0 = off
    bool r27 = false;                           // R27 (schedule 27): R26 with one scale-down per sum of products
    const uint64_t *plan(const std::string &k) const;
};

struct bc_sk {
    std::vector<int64_t> s;    // ternary coefficients
    uint64_t *d_s = nullptr;   // eval form [L1+K][n]
};

struct bc_keys {
    std::map<uint32_t, uint64_t *> ksk;  // t -> [dnum][2][L1+K][n] eval (t = 0 relin)
    uint64_t *d_pk = nullptr;            // [2][L1][n] (b, a) eval
    std::vector<void *> owned;
};

namespace bc {

void ctx_build(bc_ctx *X);
void ctx_free(bc_ctx *X);
void lift_p(bc_ctx *X, const std::string &key, const Mod *mods, uint32_t p, const uint64_t *src, uint64_t src_pstride,
            uint64_t *out, uint64_t out_pstride, int16_t *out16, uint32_t npoly, uint32_t n, uint32_t skip0,
            uint32_t skipn, int mode, cudaStream_t st);

// modulus-switch memo (R12: switching is deterministic, so reusing an earlier switch of the same ciphertext
// never changes a bit): entries keyed by the source view, valid while the source buffer is the same live
// object; FIFO-bounded by entry count (so the dry-run sizing sees the same allocations as the real run)
struct MsMemo {
    struct Key {
        const uint64_t *d;
        uint32_t B, lvl;
        uint64_t bstride;
        bool operator<(const Key &o) const {
            if (d != o.d) return d < o.d;
            if (B != o.B) return B < o.B;
            if (lvl != o.lvl) return lvl < o.lvl;
            return bstride < o.bstride;
        }
    };
    struct Ent {
        std::weak_ptr<Buf> src;
        CT out;
        uint64_t seq;
    };
    static constexpr size_t N = 32;
    std::map<Key, Ent> m;
    std::deque<std::pair<Key, uint64_t>> order;
    uint64_t seq = 0;
    bool on = false;        // enabled inside the digit circuits only (their values are never modified in place)
    size_t hits = 0, misses = 0;
};

// engine: batched BGV ops on one stream over a workspace arena
struct Eng {
    bc_ctx *X;
    const bc_keys *keys;
    Arena *A;
    cudaStream_t st;
    std::shared_ptr<MsMemo> msm = std::make_shared<MsMemo>();
    bool dry() const { return A->dry; }

    BufP alloc_words(uint64_t words);
    CT ct_alloc(uint32_t B, uint32_t lvl, uint32_t parts = 2);
    CT view(uint64_t *d, uint32_t B, uint32_t lvl, uint32_t parts = 2);
    CT sub(const CT &a, uint32_t b0, uint32_t nb);  // sub-batch view

    // transforms / element-wise
    void ntt_fwd(const uint64_t *in, uint64_t *out, uint32_t npoly, LimbMap lm, uint64_t ips, uint64_t ops);
    void ntt_inv(const uint64_t *in, uint64_t *out, uint32_t npoly, LimbMap lm, uint64_t ips, uint64_t ops);
    // forward transform with the scale-sub / fused-ModDown epilogue in pass C (false: not available, nothing done)
    bool ntt_fwd_epi(const uint64_t *in, uint64_t *out, uint32_t npoly, LimbMap lm, uint64_t ips, uint64_t ops,
                     const NttEpi &e);

    CT modswitch(const CT &a);
    CT modswitch_to(const CT &a, uint32_t lvl);
    CT add(const CT &a, const CT &b);
    CT mul_sum(const std::vector<std::pair<CT, CT>> &prs);   // R27: sum of products, one scale-down
    CT axpy(const CT &acc, const CT &x, int64_t c);   // acc + c x (= add(acc, scalar(x, c)), one kernel)
    CT scalar(const CT &a, int64_t c);       // c in F_p (centered)
    CT add_const(const CT &a, int64_t c);
    CT ptmul(const CT &a, const uint64_t *pt);
    CT add_pt(const CT &a, const uint64_t *pt);
    CT ptmul_add_pt(const CT &a, const uint64_t *pm, const uint64_t *pa);   // add_pt(ptmul(a, pm), pa), one pass
    // key switch of polys d (ct b at d + b*dps, lvl limbs, eval) -> [B][2][lvl][n]
    CT keyswitch(const uint64_t *d, uint64_t dps, uint32_t B, uint32_t lvl, uint32_t key_id);
    BufP ks_up(const uint64_t *d, uint64_t dps, uint32_t B, uint32_t lvl, uint32_t key_id);  // ModUp + KIP
    BufP ks_modup(const uint64_t *d, uint64_t dps, uint32_t B, uint32_t lvl);
    BufP ks_kip(const uint64_t *d, uint64_t dps, const BufP &ext, uint32_t B, uint32_t lvl, uint32_t key_id,
                uint32_t perm_t);
    CT ks_moddown(const BufP &u, uint32_t B, uint32_t lvl);
    std::vector<CT> automorph_hoisted(const CT &a, const std::vector<uint32_t> &ts);   // R22
    CT mul(const CT &a, const CT &b);
    CT automorph(const CT &a, uint32_t t);
    CT rotate(const CT &a, int64_t k);
    CT frobenius(const CT &a, uint32_t k);
    void copy_into(const CT &src, uint64_t *dst);
};

// plaintext constants
uint64_t *ctx_pt(bc_ctx *X, const std::string &key, const std::vector<int16_t> &slots, cudaStream_t st);
// encodes every plaintext constant of the compare / select schedules (kappa, lexicographic and
// broadcast masks) once at context creation, so concurrent calls only read the cache
void ctx_precompute_pt(bc_ctx *X);
void encode_slots_dev(bc_ctx *X, const int16_t *d_slots, uint32_t B, int16_t *d_coef, Arena *A,
                      cudaStream_t st);

// comparison schedule (R16) and friends
void compare_batch(Eng &E, const CT &a, const CT &b, CT *lt, CT *eq);
CT select_batch(Eng &E, const CT &cond, const CT &x1, const CT &x2);
std::vector<CT> extract_batch(Eng &E, const CT &a);
CT broadcast_batch(Eng &E, const CT &cond);
CT power_batch(Eng &E, const CT &x, uint32_t e);                       // R24
CT private_query_batch(Eng &E, Eng *S, const CT &data, const CT &q, const CT &codes, const CT &op1, uint32_t e);
CT concat_batch(Eng &E, const std::vector<CT> &parts);
CT tournament_batch(Eng &E, std::vector<CT> elems, bool is_max);
std::vector<CT> sort_batch(Eng &E, const std::vector<CT> &x);

void circuit_plan(int64_t p, char circuit, int schedule, int *k, int *muls, int *depth);

void compact_plans_release(const bc_ctx *X);   // compact.cu: drop the context's cached plans

}  // namespace bc
