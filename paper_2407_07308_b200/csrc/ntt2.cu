// ntt2.cu -- register-blocked Bluestein NTT passes for sm_100a (a1/a2).
//
// Same four-step decomposition and data layout as the radix-2 passes in kernels.cu
// (M = R x C; pass A: chirp + column DIF + psi^(c k1); pass B: row DIF, x D^, row DIT,
// psi^(-c k1); pass C: column DIT + output chirp + Z_m^* gather), but every sub-transform of
// length L = 2^LOGL is done by L/E threads holding E = 2^LOGE elements in registers:
// LOGE butterfly stages per register pass, one shared-memory exchange between passes, lazy
// (Harvey) reduction in [0, 2q) with Shoup twiddles.  A thread in a pass with lowest stage
// 2^lo holds the E indices base + k 2^lo, base = (tau mod 2^lo) + (tau >> lo) 2^(lo+LOGE).
#include <cuda_runtime.h>

#include "kernels.h"

namespace bc {

template <int E>
struct Regs {
    uint64_t v[E];
};

// Shoup product with an approximate high word: hi ~ x1 p1 + hi32(x1 p0) + hi32(x0 p1) drops the
// low partial products (< 3 * 2^32), so hi_est in [hi - 2, hi] and r = x w - hi_est q in [0, 4q).
// r is formed as x w + hi_est (2^64 - q) mod 2^64 (IMAD accumulation, no separate subtract).
__device__ __forceinline__ uint64_t shoup4(uint64_t x, uint64_t w, uint64_t wp, uint64_t nq) {
    const uint32_t x0 = (uint32_t)x, x1 = (uint32_t)(x >> 32);
    const uint32_t p0 = (uint32_t)wp, p1 = (uint32_t)(wp >> 32);
    const uint64_t hi = (uint64_t)x1 * p1 + __umulhi(x1, p0) + __umulhi(x0, p1);
    return x * w + hi * nq;
}

// one register pass of NS <= LOGE stages: stage u = 0 .. NS-1 acts on half-size h = 2^(lo+u) between
// registers k and k + 2^u; DIF runs u downwards, DIT upwards.  tw = omega_L^{+j} (DIF) or
// omega_L^{-j} (DIT), j < L/2.  Lazy bounds (q < 2^51, shoup4 outputs < 4q):
//   DIF global stage g (g = LOGL-1-log h): inputs < B_g = 4q 2^g; x' = x + y < B_{g+1};
//       y' = shoup4(x + B_g - y) < 4q.        (B_9 = 2^11 q < 2^62)
//   DIT: y' = shoup4(y) < 4q; x' = x + y', y'' = x + 4q - y': bound grows by 4q per stage.
// In the pass with lowest stage 2^0 (LO = 0) the twiddle index is a compile-time constant and
// index 0 (omega^0 = 1) needs no product: DIF y' = x + B_g - y (< 2 B_g = B_{g+1}, the next
// stage's bound); DIT y' = x + B_s - y with stage input bound B_s = 4q 2^s (this pass is the first
// DIT pass, inputs < 4q; each of its stages at most doubles the bound: 2^NS * 4q <= 2^6 q).
// That skips 15 of the 32 products of a 16-register pass (23% of a 256-point transform).
template <int LOGE, int NS, bool DIF, int LO>
__device__ __forceinline__ void reg_pass(uint64_t (&v)[1 << LOGE], uint32_t base_mod, const u64x2 *__restrict__ tw,
                                         int logL, uint64_t q) {
    constexpr int E = 1 << LOGE;
    const uint64_t q4 = 4 * q, nq = 0 - q;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        const int u = DIF ? (NS - 1 - s) : s;
        const int lh = LO + u;                       // log2 h
        const int tsh = logL - 1 - lh;               // twiddle omega_{2h}^{i mod h} = omega_L^{(i mod h) L/2h}
        const uint64_t Bg = q4 << tsh;               // DIF input bound at this stage (g = tsh)
        const uint64_t Bs = q4 << s;                 // DIT input bound in the LO = 0 pass
#pragma unroll
        for (int k = 0; k < E; ++k) {
            if (k & (1 << u)) continue;
            const int k2 = k + (1 << u);
            const uint32_t kpart = (uint32_t)(k & ((1 << u) - 1));
            const bool trivial = LO == 0 && kpart == 0;
            if (DIF) {
                const uint64_t x = v[k], y = v[k2];
                v[k] = x + y;
                if (trivial) {
                    v[k2] = x + Bg - y;
                } else {
                    const u64x2 w = tw[(base_mod + (kpart << LO)) << tsh];
                    v[k2] = shoup4(x + Bg - y, w.w, w.ws, nq);
                }
            } else if (trivial) {
                const uint64_t x = v[k], y = v[k2];
                v[k] = x + y;
                v[k2] = x + Bs - y;
            } else {
                const u64x2 w = tw[(base_mod + (kpart << LO)) << tsh];
                const uint64_t x = v[k];
                const uint64_t y = shoup4(v[k2], w.w, w.ws, nq);
                v[k] = x + y;
                v[k2] = x + q4 - y;
            }
        }
    }
}

// pass schedule of a length-2^LOGL transform with 2^LOGE registers per thread.
// DIF: full passes from the top stage down, the short remainder pass (if any) last at lo = 0.
// DIT: the short remainder pass first at lo = 0, then full passes upwards.
template <int LOGL, int LOGE>
struct Passes {
    static constexpr int REM = LOGL % LOGE;
    static constexpr int NFULL = LOGL / LOGE;
    static constexpr int NP = NFULL + (REM ? 1 : 0);
    __device__ static constexpr int dif_lo(int p) { return p < NFULL ? LOGL - LOGE * (p + 1) : 0; }
    __device__ static constexpr int dif_ns(int p) { return p < NFULL ? LOGE : REM; }
    __device__ static constexpr int dit_lo(int p) { return REM ? (p == 0 ? 0 : REM + LOGE * (p - 1)) : LOGE * p; }
    __device__ static constexpr int dit_ns(int p) { return REM ? (p == 0 ? REM : LOGE) : LOGE; }
};

// index held by register k of thread tau in a pass with lowest stage 2^lo
template <int LOGE>
__device__ __forceinline__ uint32_t held_index(uint32_t tau, int lo, int k) {
    return (tau & ((1u << lo) - 1)) + ((tau >> lo) << (lo + LOGE)) + ((uint32_t)k << lo);
}

// ---------------------------------------------------------------------------------------------
// Row transform of length L = 2^LOGL by L/E threads (thread index tau in the row).
// Shared memory row: element i at srow[i + (i >> LOGE)] (padding breaks bank conflicts).
// DIF: natural -> bit-reversed; enters holding the first DIF pattern (lo = LOGL - LOGE), leaves
// holding lo = 0 (contiguous).  DIT: enters at lo = 0, leaves at lo = LOGL - LOGE.
template <int LOGL, int LOGE, bool DIF, int P>
__device__ __forceinline__ void rt_pass(uint64_t (&v)[1 << LOGE], uint32_t tau, uint64_t *srow, const u64x2 *__restrict__ tw,
                                        uint64_t q) {
    typedef Passes<LOGL, LOGE> PS;
    constexpr int E = 1 << LOGE;
    constexpr int lo = DIF ? PS::dif_lo(P) : PS::dit_lo(P);
    constexpr int ns = DIF ? PS::dif_ns(P) : PS::dit_ns(P);
    if (P > 0) {
        constexpr int plo = DIF ? PS::dif_lo(P > 0 ? P - 1 : 0) : PS::dit_lo(P > 0 ? P - 1 : 0);
#pragma unroll
        for (int k = 0; k < E; ++k) {
            const uint32_t i = held_index<LOGE>(tau, plo, k);
            srow[i + (i >> LOGE)] = v[k];
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < E; ++k) {
            const uint32_t i = held_index<LOGE>(tau, lo, k);
            v[k] = srow[i + (i >> LOGE)];
        }
        __syncthreads();
    }
    reg_pass<LOGE, ns, DIF, lo>(v, tau & ((1u << lo) - 1), tw, LOGL, q);
    if (P + 1 < PS::NP) rt_pass<LOGL, LOGE, DIF, (P + 1 < PS::NP ? P + 1 : P)>(v, tau, srow, tw, q);
}

template <int LOGL, int LOGE, bool DIF>
__device__ __forceinline__ void row_transform(uint64_t (&v)[1 << LOGE], uint32_t tau, uint64_t *srow,
                                              const u64x2 *__restrict__ tw, uint64_t q) {
    rt_pass<LOGL, LOGE, DIF, 0>(v, tau, srow, tw, q);
}

// column variant: element i of column `col` at scol[i * TC + col] (lanes = columns: no padding)
template <int LOGL, int LOGE, bool DIF, int TC, int P>
__device__ __forceinline__ void ct_pass(uint64_t (&v)[1 << LOGE], uint32_t tau, uint32_t col, uint64_t *scol,
                                        const u64x2 *__restrict__ tw, uint64_t q) {
    typedef Passes<LOGL, LOGE> PS;
    constexpr int E = 1 << LOGE;
    constexpr int lo = DIF ? PS::dif_lo(P) : PS::dit_lo(P);
    constexpr int ns = DIF ? PS::dif_ns(P) : PS::dit_ns(P);
    if (P > 0) {
        constexpr int plo = DIF ? PS::dif_lo(P > 0 ? P - 1 : 0) : PS::dit_lo(P > 0 ? P - 1 : 0);
#pragma unroll
        for (int k = 0; k < E; ++k) scol[held_index<LOGE>(tau, plo, k) * TC + col] = v[k];
        __syncthreads();
#pragma unroll
        for (int k = 0; k < E; ++k) v[k] = scol[held_index<LOGE>(tau, lo, k) * TC + col];
        __syncthreads();
    }
    reg_pass<LOGE, ns, DIF, lo>(v, tau & ((1u << lo) - 1), tw, LOGL, q);
    if (P + 1 < PS::NP) ct_pass<LOGL, LOGE, DIF, TC, (P + 1 < PS::NP ? P + 1 : P)>(v, tau, col, scol, tw, q);
}

template <int LOGL, int LOGE, bool DIF, int TC>
__device__ __forceinline__ void col_transform(uint64_t (&v)[1 << LOGE], uint32_t tau, uint32_t col, uint64_t *scol,
                                              const u64x2 *__restrict__ tw, uint64_t q) {
    ct_pass<LOGL, LOGE, DIF, TC, 0>(v, tau, col, scol, tw, q);
}

__device__ __forceinline__ uint32_t brev_n(uint32_t x, int bits) { return __brev(x) >> (32 - bits); }

// minimum resident blocks per SM requested from ptxas (caps registers at 65536 / (threads * minb))
#ifndef NTT_REG_TARGET
#define NTT_REG_TARGET 64
#endif
#define NTT_MINB(threads) ((65536 / NTT_REG_TARGET) / (threads) > 0 ? (65536 / NTT_REG_TARGET) / (threads) : 1)

struct JobInfoLite {
    uint32_t poly, lb, pr;
};

__device__ __forceinline__ JobInfoLite job_lite(const LimbMap &lm, uint32_t job) {
    JobInfoLite j;
    const uint32_t jl = job / lm.npoly;          // limb-major job order
    j.poly = job - jl * lm.npoly;
    j.lb = lm.limb(jl);
    j.pr = lm.prime(j.lb);
    return j;
}

// ---------------------------------------------------------------------------------------------
// pass A: chirp-multiply input, column DIF (length R), x psi^(c k1), store scratch[rp*C + c]
// block = TC columns (lanes) x R/E threads (warps); grid (C/TC, jobs)
template <int LOGR, int LOGE, int TC, int INV>
__global__ void __launch_bounds__(TC * (1 << (LOGR - LOGE)), NTT_MINB(TC * (1 << (LOGR - LOGE)))) k2_passA(NttTables T,
                                                                      const uint64_t *__restrict__ in, uint64_t in_pstride,
                                                                      LimbMap lm, uint64_t job0, uint64_t *__restrict__ scratch) {
    constexpr int E = 1 << LOGE, R = 1 << LOGR;
    extern __shared__ uint64_t sm2[];
    const uint32_t job = (uint32_t)(job0 + blockIdx.y);
    const JobInfoLite J = job_lite(lm, job);
    const uint64_t q = T.mods[J.pr].q;
    const uint32_t col = threadIdx.x % TC, tau = threadIdx.x / TC;
    const uint32_t c = blockIdx.x * TC + col;
    const u64x2 *tf = (INV ? T.tf1i : T.tf1) + (uint64_t)J.pr * T.m;
    const uint64_t *src = in + (uint64_t)J.poly * in_pstride + (uint64_t)J.lb * T.n;
    u64x2 *stw = (u64x2 *)(sm2 + (size_t)R * TC);          // omega_R^j, j < R/2
    for (int j = threadIdx.x; j < R / 2; j += blockDim.x) stw[j] = T.twR[(uint64_t)J.pr * (R / 2) + j];
    uint64_t v[E];
    // first DIF pass pattern: lo = LOGR - LOGE, base = tau (tau < 2^lo), indices tau + k 2^lo
#pragma unroll
    for (int k = 0; k < E; ++k) {
        const uint32_t r = held_index<LOGE>(tau, LOGR - LOGE, k);
        const uint32_t t = r * T.C + c;
        uint64_t x = 0;
        if (!INV) {
            if (t < T.n) { const u64x2 w = tf[t]; x = shoup4(__ldcs(src + t), w.w, w.ws, 0 - q); }
        } else if (t < T.m) {
            const int ps = T.pos[t];
            if (ps >= 0) { const u64x2 w = tf[t]; x = shoup4(__ldcs(src + ps), w.w, w.ws, 0 - q); }
        }
        v[k] = x;
    }
    __syncthreads();
    col_transform<LOGR, LOGE, true, TC>(v, tau, col, sm2, stw, q);
    const u64x2 *xt = T.xta + (uint64_t)J.pr * T.M;         // psi^(c k1) in pass layout
    uint64_t *dst = scratch + (uint64_t)blockIdx.y * T.M;
#pragma unroll
    for (int k = 0; k < E; ++k) {
        const uint32_t rp = held_index<LOGE>(tau, 0, k);
        const u64x2 w = xt[rp * T.C + c];
        __stcs(dst + rp * T.C + c, shoup4(v[k], w.w, w.ws, 0 - q));     // [0, 4q); streaming: keep tables in L2
    }
}

// pass B: row DIF (length C), x D^, row DIT, x psi^(-c k1); block = RB rows x C/E threads
template <int LOGC, int LOGE, int RB, int INV>
__global__ void __launch_bounds__(RB * (1 << (LOGC - LOGE)), NTT_MINB(RB * (1 << (LOGC - LOGE)))) k2_passB(NttTables T, LimbMap lm, uint64_t job0,
                                                                      uint64_t *__restrict__ scratch) {
    constexpr int E = 1 << LOGE, C = 1 << LOGC, TPR = C / E;
    constexpr int ROWW = C + C / E;        // padded row width in smem
    extern __shared__ uint64_t sm2[];
    const uint32_t job = (uint32_t)(job0 + blockIdx.y);
    const JobInfoLite J = job_lite(lm, job);
    const uint64_t q = T.mods[J.pr].q;
    const uint32_t rr = threadIdx.x / TPR, tau = threadIdx.x % TPR;
    const uint32_t row = blockIdx.x * RB + rr;
    uint64_t *srow = sm2 + rr * ROWW;
    uint64_t *grow = scratch + (uint64_t)blockIdx.y * T.M + (uint64_t)row * C;
    u64x2 *tw = (u64x2 *)(sm2 + (size_t)RB * ROWW), *twi = tw + C / 2;
    for (int j = threadIdx.x; j < C / 2; j += blockDim.x) {
        tw[j] = T.twC[(uint64_t)J.pr * (C / 2) + j];
        twi[j] = T.twCi[(uint64_t)J.pr * (C / 2) + j];
    }
    uint64_t v[E];
#pragma unroll
    for (int k = 0; k < E; ++k) v[k] = __ldcs(grow + held_index<LOGE>(tau, LOGC - LOGE, k));
    __syncthreads();
    row_transform<LOGC, LOGE, true>(v, tau, srow, tw, q);
    // contiguous positions tau*E + k: pointwise product with D^ (same pass layout)
    const u64x2 *dh = (INV ? T.dhi : T.dhf) + (uint64_t)J.pr * T.M + (uint64_t)row * C + tau * E;
#pragma unroll
    for (int k = 0; k < E; ++k) {
        const u64x2 w = dh[k];
        v[k] = shoup4(v[k], w.w, w.ws, 0 - q);
    }
    row_transform<LOGC, LOGE, false>(v, tau, srow, twi, q);
    const u64x2 *xt = T.xtb + (uint64_t)J.pr * T.M + (uint64_t)row * C;    // psi^(-c k1), row-contiguous
#pragma unroll
    for (int k = 0; k < E; ++k) {
        const uint32_t cc = held_index<LOGE>(tau, LOGC - LOGE, k);
        const u64x2 w = xt[cc];
        __stcs(grow + cc, shoup4(v[k], w.w, w.ws, 0 - q));
    }
}

// pass C: column DIT (length R) -> natural t, output chirp, Z_m^* gather (fwd) or A_t (inv)
template <int LOGR, int LOGE, int TC, int INV>
__global__ void __launch_bounds__(TC * (1 << (LOGR - LOGE)), NTT_MINB(TC * (1 << (LOGR - LOGE)))) k2_passC(NttTables T, uint64_t *__restrict__ out,
                                                                      uint64_t out_pstride, LimbMap lm, uint64_t job0,
                                                                      uint64_t *__restrict__ scratch) {
    constexpr int E = 1 << LOGE, R = 1 << LOGR;
    extern __shared__ uint64_t sm2[];
    const uint32_t job = (uint32_t)(job0 + blockIdx.y);
    const JobInfoLite J = job_lite(lm, job);
    const uint64_t q = T.mods[J.pr].q;
    const uint32_t col = threadIdx.x % TC, tau = threadIdx.x / TC;
    const uint32_t c = blockIdx.x * TC + col;
    uint64_t *scr = scratch + (uint64_t)blockIdx.y * T.M;
    u64x2 *stw = (u64x2 *)(sm2 + (size_t)R * TC);          // omega_R^-j, j < R/2
    for (int j = threadIdx.x; j < R / 2; j += blockDim.x) stw[j] = T.twRi[(uint64_t)J.pr * (R / 2) + j];
    uint64_t v[E];
#pragma unroll
    for (int k = 0; k < E; ++k) v[k] = __ldcs(scr + held_index<LOGE>(tau, 0, k) * T.C + c);
    __syncthreads();
    col_transform<LOGR, LOGE, false, TC>(v, tau, col, sm2, stw, q);
    const u64x2 *tfo = (INV ? T.tfoi : T.tfo) + (uint64_t)J.pr * T.m;
    uint64_t *dst = out + (uint64_t)J.poly * out_pstride + (uint64_t)J.lb * T.n;
    if (INV) __syncthreads();   // all columns of this block read before in-place writes of A_t
#pragma unroll
    for (int k = 0; k < E; ++k) {
        const uint32_t r = held_index<LOGE>(tau, LOGR - LOGE, k);
        const uint32_t t = r * T.C + c;
        if (t >= T.m) continue;
        const u64x2 w = tfo[t];
        const uint64_t x = mul_shoup(v[k], w.w, w.ws, q);      // canonical [0, q)
        if (!INV) {
            const int ps = T.pos[t];
            if (ps >= 0) __stcs(dst + ps, x);
        } else {
            scr[t] = x;
        }
    }
}

// ---------------------------------------------------------------------------------------------
template <int LOGR, int LOGER, int LOGC, int LOGEC, int TC_, int RB_>
struct Ntt2Shape {
    static constexpr int TC = TC_, RB = RB_ ? RB_ : ((LOGC - LOGEC) >= 6 ? 4 : ((LOGC - LOGEC) >= 4 ? 8 : 16));
    static constexpr int THA = TC << (LOGR - LOGER), THB = RB << (LOGC - LOGEC);
    static constexpr size_t SMA = (size_t)(1 << LOGR) * TC * 8 + (size_t)(1 << LOGR) / 2 * 16;
    static constexpr size_t SMB = (size_t)RB * ((1 << LOGC) + (1 << (LOGC - LOGEC))) * 8 + (size_t)(1 << LOGC) * 16;
};

template <int LOGR, int LOGER, int LOGC, int LOGEC, int TC_ = 16, int RB_ = 0>
static void run2(const NttTables &T, const uint64_t *in, uint64_t *out, LimbMap lm,
                 uint64_t in_ps, uint64_t out_ps, uint64_t *scratch, uint64_t j0, uint32_t nj, int inv, cudaStream_t st) {
    typedef Ntt2Shape<LOGR, LOGER, LOGC, LOGEC, TC_, RB_> S;
    static std::atomic<uint64_t> init_dev{0};
    if (attr_pending(init_dev)) {
        cudaFuncSetAttribute(k2_passA<LOGR, LOGER, S::TC, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMA);
        cudaFuncSetAttribute(k2_passA<LOGR, LOGER, S::TC, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMA);
        cudaFuncSetAttribute(k2_passC<LOGR, LOGER, S::TC, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMA);
        cudaFuncSetAttribute(k2_passC<LOGR, LOGER, S::TC, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMA);
        cudaFuncSetAttribute(k2_passB<LOGC, LOGEC, S::RB, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMB);
        cudaFuncSetAttribute(k2_passB<LOGC, LOGEC, S::RB, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMB);
        attr_done(init_dev);
    }
    dim3 gA((1 << LOGC) / S::TC, nj), gB((1 << LOGR) / S::RB, nj);
    if (!inv) {
        k2_passA<LOGR, LOGER, S::TC, 0><<<gA, S::THA, S::SMA, st>>>(T, in, in_ps, lm, j0, scratch);
        k2_passB<LOGC, LOGEC, S::RB, 0><<<gB, S::THB, S::SMB, st>>>(T, lm, j0, scratch);
        k2_passC<LOGR, LOGER, S::TC, 0><<<gA, S::THA, S::SMA, st>>>(T, out, out_ps, lm, j0, scratch);
    } else {
        k2_passA<LOGR, LOGER, S::TC, 1><<<gA, S::THA, S::SMA, st>>>(T, in, in_ps, lm, j0, scratch);
        k2_passB<LOGC, LOGEC, S::RB, 1><<<gB, S::THB, S::SMB, st>>>(T, lm, j0, scratch);
        k2_passC<LOGR, LOGER, S::TC, 1><<<gA, S::THA, S::SMA, st>>>(T, out, out_ps, lm, j0, scratch);
    }
    launch_counter() += 3;
}

bool ntt2_supported(const NttTables &T) {
    return T.logR >= 5 && T.logR <= 8 && T.logC >= 6 && T.logC <= 9 && T.logC >= T.logR && T.logC - T.logR <= 1;
}

// g_ntt_impl (256 x 256 shape): 0 -> E = 16, 8 columns per pass-A/C block, 8 rows per pass-B block
// (default, measured fastest); 2..6 -> tuning variants (E, TC, RB) = (8,16,*), (16,4,*), (16,8,4),
// (16,4,4), (16,8,16).  Other shapes use one variant.
void ntt2_run(const NttTables &T, const uint64_t *in, uint64_t *out, LimbMap lm, uint64_t in_ps,
              uint64_t out_ps, uint64_t *scratch, uint64_t j0, uint32_t nj, int inv, cudaStream_t st) {
#define RUN2(...) run2<__VA_ARGS__>(T, in, out, lm, in_ps, out_ps, scratch, j0, nj, inv, st)
    switch (T.logR * 16 + T.logC) {
        case 8 * 16 + 8:
            switch (g_ntt_impl) {
                case 2: RUN2(8, 3, 8, 3, 16); break;
                case 3: RUN2(8, 4, 8, 4, 4); break;
                case 4: RUN2(8, 4, 8, 4, 8, 4); break;
                case 5: RUN2(8, 4, 8, 4, 4, 4); break;
                case 6: RUN2(8, 4, 8, 4, 8, 16); break;
                default: RUN2(8, 4, 8, 4, 8); break;
            }
            break;
        case 8 * 16 + 9: RUN2(8, 4, 9, 3, 8); break;
        case 7 * 16 + 8: RUN2(7, 4, 8, 4, 16); break;
        case 7 * 16 + 7: RUN2(7, 4, 7, 4, 16); break;
        case 6 * 16 + 7: RUN2(6, 3, 7, 4, 16); break;
        case 6 * 16 + 6: RUN2(6, 3, 6, 3, 16); break;
        case 5 * 16 + 6: RUN2(5, 4, 6, 3, 16); break;
        default: break;
    }
#undef RUN2
}

}  // namespace bc
