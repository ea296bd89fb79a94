// kernels.h -- launch wrappers for the sm_100a kernels of the BoostCom hot path.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "modarith.cuh"

namespace bc {

// Per-device kernel-attribute flags (cudaFuncSetAttribute acts on the current device): a call site
// sets its attributes while attr_pending() is true, then attr_done().  Thread-safe: the bit is set
// only after the attributes, and two racing threads both setting them is harmless (idempotent).
inline uint64_t cur_device_bit() {
    int dev = 0;
    cudaGetDevice(&dev);
    return 1ull << (dev & 63);
}
inline bool attr_pending(const std::atomic<uint64_t> &done) {
    return !(done.load(std::memory_order_acquire) & cur_device_bit());
}
inline void attr_done(std::atomic<uint64_t> &done) { done.fetch_or(cur_device_bit(), std::memory_order_acq_rel); }

struct __align__(16) u64x2 { uint64_t w, ws; };   // value + Shoup companion (16-byte aligned: one 128-bit load)

// Fused epilogue of a forward transform (binary64 pass C): the word x = NTT(in) at output position i of
// poly p, limb lb becomes
//   mode 1: (u - x) w_lb                  -- modulus switch (R13) / ModDown scale-sub (R14)
//   mode 2: (u + pm_lb d - x) w_lb        -- fused ModDown + modulus switch of a product (R15), p = 2 b + k
// with u = u[p ups + lb n + i], d = d[b dbs + k dks + lb n + i]; results identical to the separate kernels
// (ew_scale_sub / ew_fused_down_out) -- the delta words are never written to memory.
struct NttEpi {
    int mode = 0;
    const Mod *mods = nullptr;
    const uint64_t *u = nullptr;
    uint64_t ups = 0;
    const uint64_t *d = nullptr;
    uint64_t dbs = 0, dks = 0;
    const u64x2 *pm = nullptr, *w = nullptr;
};

// Device tables of the Bluestein transforms (§8(a) a1/a2), one slice per prime.
struct NttTables {
    const u64x2 *psi;     // [P][M]  psi^e (size-M root, free internal choice)
    const u64x2 *tf1;     // [P][m]  TF1_j = omega^(h j^2)            (forward input chirp)
    const u64x2 *tf1i;    // [P][m]  omega^(-h j^2)                    (inverse input chirp)
    const u64x2 *tfo;     // [P][m]  TF1_j * M^-1                      (forward output chirp)
    const u64x2 *tfoi;    // [P][m]  omega^(-h j^2) * M^-1 * m^-1      (inverse output chirp)
    const u64x2 *dhf;     // [P][M]  NTT_M(D_pad) in the pass layout   (forward)
    const u64x2 *dhi;     // [P][M]  NTT_M(D'_pad)                     (inverse)
    const int32_t *pos;   // [m]     position of t in Z_m^* (ascending) or -1 (Listing 2 prefix sum)
    const int32_t *z;     // [n]     Z_m^* ascending
    const int8_t *phi;    // [n+1]   Phi_m coefficients (for composite m)
    const Mod *mods;      // [P]
    const u64x2 *twR, *twRi, *twC, *twCi;   // [P][R/2], [P][C/2]: omega_R^{+-j}, omega_C^{+-j} (register passes)
    const u64x2 *xta;     // [P][M]  psi^(c brev(rp)) at rp*C + c   (pass A epilogue, contiguous)
    const u64x2 *xtb;     // [P][M]  psi^(-c brev(r)) at r*C + c    (pass B epilogue, contiguous)
    // binary64 variants (ntt3.cu): entry = (w centred in (-q/2, q/2], fl(w/q)); null when some q >= 2^50
    const double2 *fmods;                   // [P] (q, fl(1/q))
    const double2 *ftwRb, *ftwCb;           // [P][R/2], [P][C/2]: omega_L^{brev_{logL-1}(j)} (forward CT blocks)
    const double2 *ftwRi, *ftwCi;           // omega_L^{-j} (inverse)
    const double *ftf1, *ftf1i, *ftfo, *ftfoi, *fdhf, *fdhi, *fxta, *fxtb;   // as the u64x2 tables, w only (8 bytes)
    // composite m (binary64 path): Barrett reduction mod Phi_m by two size-M convolutions with constants, in
    // the D^ layout, M^{-1} folded: NTT(rev(Phi)^{-1} mod x^{m-n}) and NTT(Phi); null -> long division
    const double *fdhb1, *fdhb2;
    uint32_t Mslot;                // word stride of the per-job A slots read / written by modes 2 and 3
    const struct NttTables *tb;    // host pointer: the Barrett convolution tables (composite m), or null
    const int32_t *ir_off, *ir_val;   // Barrett set: Phi_m^{-1} mod x^(m-n) when it has <= 16 nonzero terms
    int ir_nnz;                       //   (the quotient is then a sum of shifted copies, no convolution)
    int q_in_s2;                      // mode 3 reads Q from the scr2 slot (sparse quotient) instead of A_{n..}
    uint32_t m, n, M, R, C, logR, logC;
    // R25 mixed-radix rows (f3): C = rad * 2^logN (rad in {3, 9}); ftwCb / ftwCi then hold the length-2^logN
    // sub-row twiddles.  rad = 1: power-of-two rows (C = 2^logC)
    uint32_t rad = 1, logN = 0;
    const double *frtw = nullptr, *frtwi = nullptr;     // [P][C]: omega_C^{+-i j} at i 2^logN + j
    const double *frcon = nullptr, *frconi = nullptr;   // [P][16]: omega_rad^{+-j}, j < rad
    int prime_m;
    NttEpi epi;           // forward transforms only (ntt_forward_epi); mode 0 elsewhere
    int dbg;              // ntt3.cu timing experiments only (bc_tune "ntt_dbg"): skip table reads; results invalid          // 1 if m is prime (reduction mod Phi_m is a single subtraction)
};

// Limb -> prime map of a batched job list: poly p in [0,npoly), jl in [0,njl):
//   limb = jl < skip0 ? jl : jl + skipn;  prime = limb < split ? limb + off_lo : limb - split + off_hi
struct LimbMap {
    uint32_t njl, skip0, skipn, split, off_lo, off_hi;
    uint32_t npoly = 0;   // set by the transform driver: jobs are ordered limb-major (job = jl * npoly + poly)
    __host__ __device__ uint32_t limb(uint32_t jl) const { return jl < skip0 ? jl : jl + skipn; }
    __host__ __device__ uint32_t prime(uint32_t lb) const { return lb < split ? lb + off_lo : lb - split + off_hi; }
};
inline LimbMap limbmap_plain(uint32_t nl, uint32_t prime0) { return LimbMap{nl, nl, 0, 0xffffffffu, prime0, 0}; }

// Batched Bluestein transforms.  in/out poly p limb lb at base + p*pstride + lb*n.
// scratch: npoly*njl*M words.
void ntt_forward(const NttTables &T, const uint64_t *in, uint64_t *out, uint32_t npoly, LimbMap lm,
                 uint64_t in_pstride, uint64_t out_pstride, uint64_t *scratch, cudaStream_t st);
void ntt_inverse(const NttTables &T, const uint64_t *in, uint64_t *out, uint32_t npoly, LimbMap lm,
                 uint64_t in_pstride, uint64_t out_pstride, uint64_t *scratch, cudaStream_t st);
// forward transform with a fused epilogue (NttEpi); only where ntt_epi_supported(T) (binary64 passes)
bool ntt_epi_supported(const NttTables &T);
void ntt_forward_epi(const NttTables &T, const NttEpi &e, const uint64_t *in, uint64_t *out, uint32_t npoly, LimbMap lm,
                     uint64_t in_pstride, uint64_t out_pstride, uint64_t *scratch, cudaStream_t st);

// ---- fused ModDown + modulus switch of a product (R15) ----
// step 1: u[b][k][level-1] += (P mod q) d_k[level-1]   (u: [B][2] polys of stride u_pstride)
void ew_fused_down(const Mod *mods, uint64_t *u, uint64_t u_pstride, const uint64_t *d, uint64_t d_bstride,
                   uint64_t d_kstride, const uint64_t *delta, const u64x2 *pm, const u64x2 *dinv, uint64_t *o,
                   uint32_t B, uint32_t level, uint32_t n, cudaStream_t st);
// step 2: o[b][k][i] = (u + Pm d_k - delta) Dinv for i < lvl_out  (o, delta: [B][2][lvl_out][n])
void ew_fused_down_out(const Mod *mods, const uint64_t *u, uint64_t u_pstride, const uint64_t *d, uint64_t d_bstride,
                       uint64_t d_kstride, const uint64_t *delta, const u64x2 *pm, const u64x2 *dinv, uint64_t *o,
                       uint32_t B, uint32_t lvl_out, uint32_t n, cudaStream_t st);

// ---- element-wise over [B][parts][level][n] (limb i uses prime i) ----
void ew_add(const Mod *mods, const uint64_t *a, const uint64_t *b, uint64_t *o, uint32_t B,
            uint32_t parts, uint32_t lvl, uint32_t n, int sub, cudaStream_t st);
// o = a (parts pa) + b (parts pb) where the extra parts are copied (3-part + 2-part etc.)
void ew_neg(const Mod *mods, const uint64_t *a, uint64_t *o, uint32_t B, uint32_t parts, uint32_t lvl,
            uint32_t n, cudaStream_t st);
void ew_ext_acc(const Mod *mods, uint64_t *W, const uint64_t *u, const uint64_t *d, uint64_t d_bstride,
                uint64_t d_kstride, const u64x2 *pm, uint32_t B, uint32_t lv, uint32_t K, uint32_t L1, uint32_t n,
                int first, cudaStream_t st);   // R27: W (+)= u + P d (extended basis)
struct PtSumArgs {       // up to 32 Frobenius images and their kappa plaintexts (contiguous [B][parts][lvl][n])
    const uint64_t *F[32];
    const uint64_t *pt[32];
    uint32_t D;
};
void ew_ptsum(const Mod *mods, const PtSumArgs &A, uint64_t *o, uint32_t B, uint32_t parts, uint32_t lvl, uint32_t n,
              cudaStream_t st, const double2 *fm);   // o = sum_k pt_k (.) F_k
void ew_ptmul_addpt(const double2 *fm, const uint64_t *a, const uint64_t *pm, const uint64_t *pa, uint64_t *o,
                    uint32_t B, uint32_t parts, uint32_t lvl, uint32_t n, cudaStream_t st);   // a (.) pm (+ pa on part 0)
void ew_axpy(const Mod *mods, const uint64_t *a, const uint64_t *x, int64_t c, uint64_t *o, uint32_t B, uint32_t parts,
             uint32_t lvl, uint32_t n, cudaStream_t st, const double2 *fm);   // o = a + c x
void ew_scalar(const Mod *mods, const uint64_t *a, int64_t c, uint64_t *o, uint32_t B, uint32_t parts,
               uint32_t lvl, uint32_t n, cudaStream_t st, const double2 *fm = nullptr);
// part 0 += c (constant polynomial: every evaluation point)
void ew_add_const(const Mod *mods, const uint64_t *a, int64_t c, uint64_t *o, uint32_t B, uint32_t parts,
                  uint32_t lvl, uint32_t n, cudaStream_t st);
// o = a (.) pt, pt u64[L][n] eval (first lvl limbs used), every part
void ew_ptmul(const Mod *mods, const uint64_t *a, const uint64_t *pt, uint64_t *o, uint32_t B,
              uint32_t parts, uint32_t lvl, uint32_t n, cudaStream_t st, const double2 *fm = nullptr);
void ew_add_pt(const Mod *mods, const uint64_t *a, const uint64_t *pt, uint64_t *o, uint32_t B,
               uint32_t parts, uint32_t lvl, uint32_t n, cudaStream_t st);
// fm: per-prime (q, fl(1/q)) when every prime is in [2^49, 2^50) -> binary64 kernels; nullptr -> integer kernels
void ew_tensor(const Mod *mods, const uint64_t *a, const uint64_t *b, uint64_t *o, uint32_t B,
               uint32_t lvl, uint32_t n, cudaStream_t st, const double2 *fm = nullptr);
void ew_automorph(const NttTables &T, const uint64_t *a, uint64_t *o, uint32_t B, uint32_t parts,
                  uint32_t lvl, uint32_t t, cudaStream_t st);
void ew_copy_parts(const uint64_t *a, uint64_t *o, uint32_t B, uint32_t parts_in, uint32_t part0,
                   uint32_t nparts, uint32_t lvl_in, uint32_t lvl_out, uint32_t n, uint32_t parts_out,
                   uint32_t opart0, cudaStream_t st);

// ---- key switching ----
// KIP: u[b][k][r][x] = sum_j ext[b][j][r][x] * key_j[k][klimb(r)][x], k in {0 (b-part),1 (a-part)};
// for r in G_j the digit is read from d (eval input) instead of ext.
// R22: KIP reading d and the extended digits through sigma_{perm_t}'s evaluation permutation
void ks_kip_perm(const Mod *mods, const NttTables &T, uint32_t perm_t, const uint64_t *d, uint64_t dps,
                 const uint64_t *ext, const uint64_t *key, uint64_t *u, uint32_t B, uint32_t lvl, uint32_t K, uint32_t L1,
                 uint32_t alpha, uint32_t ndig, uint32_t n, cudaStream_t st, const double2 *fm = nullptr);
void ew_automorph_part(const NttTables &T, const uint64_t *a, uint64_t abs, uint64_t *o, uint32_t B, uint32_t lvl,
                       uint32_t t, cudaStream_t st);
void ks_kip(const Mod *mods, const uint64_t *d, uint64_t dps, const uint64_t *ext, const uint64_t *key, uint64_t *u,
            uint32_t B, uint32_t lvl, uint32_t K, uint32_t L1, uint32_t alpha, uint32_t ndig,
            uint32_t n, cudaStream_t st, const double2 *fm = nullptr);
// o[b] = a[b] + b[b] (parts x lvl x n words per ciphertext), per-operand batch strides in words
void ew_add_bs(const Mod *mods, const uint64_t *a, uint64_t abs, const uint64_t *b, uint64_t bbs, uint64_t *o,
               uint64_t obs, uint32_t B, uint32_t parts, uint32_t lvl, uint32_t n, cudaStream_t st);
// out[b][k][i] = (u[b][k][i] - delta[b][k][i]) * inv_i  (Shoup constants per limb)
void ew_scale_sub(const Mod *mods, const uint64_t *u, uint64_t u_pstride, const uint64_t *delta,
                  const u64x2 *inv, uint64_t *o, uint32_t npoly, uint32_t lvl, uint32_t n,
                  cudaStream_t st);

// Exact centered CRT lift (Garner) -- plan blob layout in kernels.cu.
//  mode 0: residues mod each target prime -> out limbs (LimbMap-style skip over [skip0, skip0+skipn))
//  mode 1: delta = r + Q [-r]_p mod each target prime (modulus/ModDown correction, R13/R14)
//  mode 2: centered value mod p (as int16, centered in (-p/2, p/2]) -> out16[poly][n]
void lift(const uint64_t *plan, const Mod *mods, uint32_t p, const uint64_t *src, uint64_t src_pstride,
          uint64_t *out, uint64_t out_pstride, int16_t *out16, uint32_t npoly, uint32_t n,
          uint32_t skip0, uint32_t skipn, int mode, cudaStream_t st, uint32_t ns_hint = 0, uint32_t nt_hint = 0,
          const double2 *fm = nullptr);

// ---- sampling (R7) ----
// integer poly per (poly, coeff) -> residues on limbs prime0..prime0+nl-1
// kind 0 ternary, 1 cbd21; mult = multiplier applied to the integer (e.g. p for p*e);
// add16: optional int16[npoly][n] added after multiplication (message m~)
void sample_small(const Mod *mods, uint64_t seed, uint32_t tag, uint64_t stream0, uint64_t stream_step,
                  int kind, int64_t mult, const int16_t *add16, uint64_t *out, uint32_t npoly,
                  uint32_t nl, uint32_t prime0, uint32_t n, uint64_t pstride, cudaStream_t st);
// uniform residues: poly p limb lb (prime = lm.prime(lb)), counter limb index = klimb0 + lb
void sample_uniform(const Mod *mods, uint64_t seed, uint32_t tag, uint64_t stream0, uint64_t stream_step,
                    uint64_t *out, uint32_t npoly, LimbMap lm, uint32_t n, uint64_t pstride,
                    cudaStream_t st);

// ---- plaintext encode/decode (F_p linear maps as int8 GEMM) ----
// C[b][j] = sum_k A[b][k] * W[j][k]  (int8 x int8 -> int32), A [B][K], W [N][K]
void gemm_s8(const int8_t *A, const int8_t *W, int32_t *C, uint32_t B, uint32_t N, uint32_t K,
             cudaStream_t st);
// int32 -> centered mod p int16 (in (-p/2, p/2])
void mod_p_center(const int32_t *in, int16_t *out, uint64_t count, int32_t p, cudaStream_t st);
void s16_to_s8(const int16_t *in, int8_t *out, uint64_t count, int32_t p, cudaStream_t st);
// build encode matrix Em[j][s*D+i] (centered int8) from E0 (int16 [D][m]) and reduction rows
void build_encode_matrix(const int16_t *E0, const uint32_t *ts, const int8_t *red, int8_t *Em,
                         uint32_t n, uint32_t m, uint32_t D, uint32_t S, int32_t p, cudaStream_t st);
void build_decode_matrix(const int16_t *zpow, const uint32_t *ts, int8_t *Dm, uint32_t n, uint32_t m,
                         uint32_t D, uint32_t S, int32_t p, cudaStream_t st);
// int16 centered poly [npoly][n] -> residues on limbs 0..nl-1 (eval form needs an NTT after)
void s16_to_rns(const Mod *mods, const int16_t *in, uint64_t *out, uint32_t npoly, uint32_t nl,
                uint32_t n, cudaStream_t st);
// decrypt dot: x = c0 + c1 * s (eval), s eval [L][n]
void dec_dot(const Mod *mods, const uint64_t *ct, const uint64_t *s, uint64_t *o, uint32_t B,
             uint32_t lvl, uint32_t n, cudaStream_t st);

uint64_t &launch_counter();

// register-blocked passes (ntt2.cu) for the supported (R, C) shapes
bool ntt2_supported(const NttTables &T);
void ntt2_run(const NttTables &T, const uint64_t *in, uint64_t *out, LimbMap lm, uint64_t in_ps, uint64_t out_ps,
              uint64_t *scratch, uint64_t j0, uint32_t nj, int inv, cudaStream_t st);
// binary64-FMA passes (ntt3.cu)
bool nttf_supported(const NttTables &T);
int nttf_mr_loge(uint32_t rad, uint32_t logN);     // registers per thread (log2) of the mixed-radix sub-row transforms
int nttf_row_loge(uint32_t logR, uint32_t logC);   // D^ (fdhf/fdhi) layout: position r*C + tau*E + k at r*C + k*(C/E) + tau
// corner_buf (prime m, inverse): nj words; pass C then writes the reduction mod Phi_m directly (no k_reduce_prime)
void nttf_run(const NttTables &T, const uint64_t *in, uint64_t *out, LimbMap lm, uint64_t in_ps, uint64_t out_ps,
              uint64_t *scratch, uint64_t j0, uint32_t nj, int inv, cudaStream_t st, uint64_t *corner_buf = nullptr);
// fused thread-block-cluster transform (ntt4.cu): one kernel per batch, the size-M grid in distributed
// shared memory, no scratch; prime m only (the inverse writes the reduction mod Phi_m)
bool nttc_supported(const NttTables &T);
extern int g_nttc_clusters, g_nttc_active, g_nttc_variant;
void nttc_run(const NttTables &T, const uint64_t *in, uint64_t *out, LimbMap lm, uint64_t in_ps, uint64_t out_ps,
              uint64_t j0, uint32_t nj, int inv, cudaStream_t st);
// composite m: out (poly/limb layout) = A mod Phi_m for the A_t (t < m) the inverse left in the scr1 slots
// (stride B.Mslot), by the two Barrett convolutions of table set B (scr2: slots of B.M words)
void nttf_barrett(const NttTables &B, uint64_t *out, LimbMap lm, uint64_t out_ps, uint64_t *scr1, uint64_t *scr2,
                  uint64_t j0, uint32_t nj, cudaStream_t st);
extern uint64_t g_ntt_group_bytes;
uint64_t ntt_group_jobs(const NttTables &T, uint64_t jobs, bool barrett);
bool ntt_inverse_barrett(const NttTables &T);
extern int g_ntt_dbg;
extern int g_phi_conv;   // 1: always compute the Barrett quotient by convolution (testing)
extern int g_f64_elem;   // 1: binary64 element-wise / lift / KIP kernels when the context allows them   // scratch bytes per transform launch group (L2 residency)
extern uint64_t g_vec_chunk;
extern int g_kip_blocked;
extern int g_lift2;
extern int g_ntt_split;        // 1: transform calls split over two streams (see ntt_split_or_common)
extern int g_ntt_persist_occ;  // >0: cap of the persistent column passes' CTAs per SM
extern int g_ntt_epi;          // 1: scale-sub / fused-ModDown epilogues inside pass C of the forward transform
extern int g_ntt_lean;
extern int g_lift_blocks;      // binary64 lifts: row blocks capped at 148 x this / column blocks (0: one per poly)
extern int g_ptsum;            // 1: digit extraction as one kappa-weighted sum kernel per digit (default)
extern int g_axpy;             // 1: fused a + c x in the digit circuits' linear combinations (default)         // persistent column passes: table tiles in shared memory (0) or read through L2 (1-3)
extern int g_ntt_timing;
// comparison phases (bench "phases"; NVTX ranges of the same names)
enum { PH_EXTRACT = 0, PH_DIGIT, PH_LEX, PH_BCAST, PH_COMPACT, PH_PQMAIN, NPHASE };
extern int g_phase_timing;
struct PhaseScope {      // event pair (when g_phase_timing) + NVTX range around one leaf phase
    PhaseScope(int ph, cudaStream_t st, bool on = true);
    ~PhaseScope();
    int ph_;
    cudaStream_t st_;
    bool on_;
    void *a_ = nullptr;
};
int phase_timing_collect(double *ms, uint64_t *calls);   // ms[NPHASE], calls[NPHASE]; clears the records  // 1: record an event pair around every NTT call (bench roofline)
int ntt_timing_collect(double *ms, uint64_t *jobs, uint64_t *calls, uint64_t *inv_jobs = nullptr);
extern int g_ntt_impl;   // 0 = binary64 three-pass kernels (ntt3.cu) where supported; 1 = radix-2 passes;
                         // 2 = integer register passes; 10-19 = binary64 three-pass shapes; 20 = fused cluster kernel (ntt4.cu)

}  // namespace bc
