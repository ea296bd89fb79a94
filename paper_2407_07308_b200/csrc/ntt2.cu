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

__device__ __forceinline__ uint64_t red2q(uint64_t x, uint64_t q2) { return x >= q2 ? x - q2 : x; }

// one register pass: stages u = 0 .. LOGE-1 act on half-size h = 2^(lo+u); DIF runs u downwards.
template <int LOGE, bool DIF>
__device__ __forceinline__ void reg_pass(uint64_t (&v)[1 << LOGE], int lo, uint32_t base_mod, const u64x2 *__restrict__ tw,
                                         int logL, uint64_t q) {
    constexpr int E = 1 << LOGE;
    const uint64_t q2 = 2 * q;
#pragma unroll
    for (int s = 0; s < LOGE; ++s) {
        const int u = DIF ? (LOGE - 1 - s) : s;
        const int lh = lo + u;                       // log2 h
        // twiddle omega_{2h}^{i mod h}; table tw holds omega_L^j (j < L/2): index (i mod h) * (L / 2h)
        const int tsh = logL - 1 - lh;
#pragma unroll
        for (int k = 0; k < E; ++k) {
            if (k & (1 << u)) continue;
            const int k2 = k + (1 << u);
            const uint32_t imod = base_mod + ((uint32_t)(k & ((1 << u) - 1)) << lo);
            if (DIF) {
                const u64x2 w = tw[imod << tsh];
                const uint64_t x = v[k], y = v[k2];
                v[k] = red2q(x + y, q2);
                v[k2] = mul_shoup_lazy(x + q2 - y, w.w, w.ws, q);
            } else {
                const u64x2 w = tw[imod << tsh];          // tw = omega_L^{-j} table for DIT
                const uint64_t x = v[k];
                const uint64_t y = mul_shoup_lazy(v[k2], w.w, w.ws, q);
                v[k] = red2q(x + y, q2);
                v[k2] = red2q(x + q2 - y, q2);
            }
        }
    }
}

// index held by register k of thread tau in a pass with lowest stage 2^lo
template <int LOGE>
__device__ __forceinline__ uint32_t held_index(uint32_t tau, int lo, int k) {
    return (tau & ((1u << lo) - 1)) + ((tau >> lo) << (lo + LOGE)) + ((uint32_t)k << lo);
}

// ---------------------------------------------------------------------------------------------
// Row transform of length L = 2^LOGL by L/E threads (thread index tau in the row).
// Shared memory row: element i at srow[i + (i >> LOGE)] (padding breaks bank conflicts).
// DIF: natural -> bit-reversed; enters with regs holding the first-pass pattern (lo = LOGL-LOGE)
// and leaves holding the last-pass pattern (lo = 0, contiguous).
// DIT: enters contiguous (lo = 0) and leaves with lo = LOGL - LOGE.
template <int LOGL, int LOGE, bool DIF>
__device__ __forceinline__ void row_transform(uint64_t (&v)[1 << LOGE], uint32_t tau, uint64_t *srow,
                                              const u64x2 *__restrict__ tw, uint64_t q) {
    constexpr int E = 1 << LOGE;
    constexpr int NP = LOGL / LOGE;
    static_assert(LOGL % LOGE == 0, "LOGL must be a multiple of LOGE");
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const int lo = DIF ? (LOGL - LOGE * (p + 1)) : (LOGE * p);
        if (p > 0) {
            // exchange: write with the previous pattern, read with this one
            const int plo = DIF ? (lo + LOGE) : (lo - LOGE);
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
        reg_pass<LOGE, DIF>(v, lo, tau & ((1u << lo) - 1), tw, LOGL, q);
    }
}

// column variant: element i of column `col` at scol[i * TC + col] (lanes = columns: no padding)
template <int LOGL, int LOGE, bool DIF, int TC>
__device__ __forceinline__ void col_transform(uint64_t (&v)[1 << LOGE], uint32_t tau, uint32_t col, uint64_t *scol,
                                              const u64x2 *__restrict__ tw, uint64_t q) {
    constexpr int E = 1 << LOGE;
    constexpr int NP = LOGL / LOGE;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const int lo = DIF ? (LOGL - LOGE * (p + 1)) : (LOGE * p);
        if (p > 0) {
            const int plo = DIF ? (lo + LOGE) : (lo - LOGE);
#pragma unroll
            for (int k = 0; k < E; ++k) scol[held_index<LOGE>(tau, plo, k) * TC + col] = v[k];
            __syncthreads();
#pragma unroll
            for (int k = 0; k < E; ++k) v[k] = scol[held_index<LOGE>(tau, lo, k) * TC + col];
            __syncthreads();
        }
        reg_pass<LOGE, DIF>(v, lo, tau & ((1u << lo) - 1), tw, LOGL, q);
    }
}

__device__ __forceinline__ uint32_t brev_n(uint32_t x, int bits) { return __brev(x) >> (32 - bits); }

struct JobInfoLite {
    uint32_t poly, lb, pr;
};

__device__ __forceinline__ JobInfoLite job_lite(const LimbMap &lm, uint32_t job) {
    JobInfoLite j;
    j.poly = job / lm.njl;
    const uint32_t jl = job - j.poly * lm.njl;
    j.lb = lm.limb(jl);
    j.pr = lm.prime(j.lb);
    return j;
}

// ---------------------------------------------------------------------------------------------
// pass A: chirp-multiply input, column DIF (length R), x psi^(c k1), store scratch[rp*C + c]
// block = TC columns (lanes) x R/E threads (warps); grid (C/TC, jobs)
template <int LOGR, int LOGE, int TC, int INV>
__global__ void __launch_bounds__(TC * (1 << (LOGR - LOGE))) k2_passA(NttTables T,
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
    uint64_t v[E];
    // first DIF pass pattern: lo = LOGR - LOGE, base = tau (tau < 2^lo), indices tau + k 2^lo
#pragma unroll
    for (int k = 0; k < E; ++k) {
        const uint32_t r = held_index<LOGE>(tau, LOGR - LOGE, k);
        const uint32_t t = r * T.C + c;
        uint64_t x = 0;
        if (!INV) {
            if (t < T.n) { const u64x2 w = tf[t]; x = mul_shoup_lazy(src[t], w.w, w.ws, q); }
        } else if (t < T.m) {
            const int ps = T.pos[t];
            if (ps >= 0) { const u64x2 w = tf[t]; x = mul_shoup_lazy(src[ps], w.w, w.ws, q); }
        }
        v[k] = x;
    }
    col_transform<LOGR, LOGE, true, TC>(v, tau, col, sm2, T.twR + (uint64_t)J.pr * (R / 2), q);
    const u64x2 *psi = T.psi + (uint64_t)J.pr * T.M;
    uint64_t *dst = scratch + (uint64_t)blockIdx.y * T.M;
#pragma unroll
    for (int k = 0; k < E; ++k) {
        const uint32_t rp = held_index<LOGE>(tau, 0, k);
        const uint32_t k1 = brev_n(rp, LOGR);
        const u64x2 w = psi[(c * k1) & (T.M - 1)];
        dst[rp * T.C + c] = mul_shoup_lazy(v[k], w.w, w.ws, q);     // [0, 2q)
    }
}

// pass B: row DIF (length C), x D^, row DIT, x psi^(-c k1); block = RB rows x C/E threads
template <int LOGC, int LOGE, int RB, int INV>
__global__ void __launch_bounds__(RB * (1 << (LOGC - LOGE))) k2_passB(NttTables T, LimbMap lm, uint64_t job0,
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
    const u64x2 *tw = T.twC + (uint64_t)J.pr * (C / 2), *twi = T.twCi + (uint64_t)J.pr * (C / 2);
    uint64_t v[E];
#pragma unroll
    for (int k = 0; k < E; ++k) v[k] = grow[held_index<LOGE>(tau, LOGC - LOGE, k)];
    row_transform<LOGC, LOGE, true>(v, tau, srow, tw, q);
    // contiguous positions tau*E + k: pointwise product with D^ (same pass layout)
    const u64x2 *dh = (INV ? T.dhi : T.dhf) + (uint64_t)J.pr * T.M + (uint64_t)row * C + tau * E;
#pragma unroll
    for (int k = 0; k < E; ++k) {
        const u64x2 w = dh[k];
        v[k] = mul_shoup_lazy(v[k], w.w, w.ws, q);
    }
    row_transform<LOGC, LOGE, false>(v, tau, srow, twi, q);
    const u64x2 *psi = T.psi + (uint64_t)J.pr * T.M;
    const uint32_t k1 = brev_n(row, T.logR);
#pragma unroll
    for (int k = 0; k < E; ++k) {
        const uint32_t cc = held_index<LOGE>(tau, LOGC - LOGE, k);
        const u64x2 w = psi[(T.M - cc * k1) & (T.M - 1)];
        grow[cc] = mul_shoup_lazy(v[k], w.w, w.ws, q);
    }
}

// pass C: column DIT (length R) -> natural t, output chirp, Z_m^* gather (fwd) or A_t (inv)
template <int LOGR, int LOGE, int TC, int INV>
__global__ void __launch_bounds__(TC * (1 << (LOGR - LOGE))) k2_passC(NttTables T, uint64_t *__restrict__ out,
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
    uint64_t v[E];
#pragma unroll
    for (int k = 0; k < E; ++k) v[k] = scr[held_index<LOGE>(tau, 0, k) * T.C + c];
    col_transform<LOGR, LOGE, false, TC>(v, tau, col, sm2, T.twRi + (uint64_t)J.pr * (R / 2), q);
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
            if (ps >= 0) dst[ps] = x;
        } else {
            scr[t] = x;
        }
    }
}

// ---------------------------------------------------------------------------------------------
template <int LOGR, int LOGER, int LOGC, int LOGEC>
struct Ntt2Shape {
    static constexpr int TC = 32, RB = (LOGC - LOGEC) >= 6 ? 4 : 8;
    static constexpr int THA = TC << (LOGR - LOGER), THB = RB << (LOGC - LOGEC);
    static constexpr size_t SMA = (size_t)(1 << LOGR) * TC * 8;
    static constexpr size_t SMB = (size_t)RB * ((1 << LOGC) + (1 << (LOGC - LOGEC))) * 8;
};

template <int LOGR, int LOGER, int LOGC, int LOGEC>
static void run2(const NttTables &T, const uint64_t *in, uint64_t *out, LimbMap lm,
                 uint64_t in_ps, uint64_t out_ps, uint64_t *scratch, uint64_t j0, uint32_t nj, int inv, cudaStream_t st) {
    typedef Ntt2Shape<LOGR, LOGER, LOGC, LOGEC> S;
    static bool init = false;
    if (!init) {
        cudaFuncSetAttribute(k2_passA<LOGR, LOGER, S::TC, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMA);
        cudaFuncSetAttribute(k2_passA<LOGR, LOGER, S::TC, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMA);
        cudaFuncSetAttribute(k2_passC<LOGR, LOGER, S::TC, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMA);
        cudaFuncSetAttribute(k2_passC<LOGR, LOGER, S::TC, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMA);
        cudaFuncSetAttribute(k2_passB<LOGC, LOGEC, S::RB, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMB);
        cudaFuncSetAttribute(k2_passB<LOGC, LOGEC, S::RB, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMB);
        init = true;
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
    return (T.logR == 8 && T.logC == 8) || (T.logR == 8 && T.logC == 9);
}

void ntt2_run(const NttTables &T, const uint64_t *in, uint64_t *out, LimbMap lm, uint64_t in_ps,
              uint64_t out_ps, uint64_t *scratch, uint64_t j0, uint32_t nj, int inv, cudaStream_t st) {
    if (T.logR == 8 && T.logC == 8) run2<8, 4, 8, 4>(T, in, out, lm, in_ps, out_ps, scratch, j0, nj, inv, st);
    else run2<8, 4, 9, 3>(T, in, out, lm, in_ps, out_ps, scratch, j0, nj, inv, st);
}

}  // namespace bc
