// nttf_core.cuh -- register / shared-memory building blocks of the binary64 Bluestein transforms (a1/a2,
// P:315-316): bound-tracked modular butterflies (f64arith.cuh), register passes of up to 2^LOGE points,
// row / column sub-transforms with one shared-memory exchange per register pass, per-thread twiddle tables.
// Used by the three-pass kernels (ntt3.cu) and the fused thread-block-cluster kernel (ntt4.cu).
#pragma once
#include <cuda_runtime.h>

#include "kernels.h"
#include "f64arith.cuh"

namespace bc {
namespace f64 {

constexpr int UQ = 16;        // canonical residue, [0, q)
constexpr int UMUL = 10;      // fmm output, |r| <= 0.625 q
constexpr int URED = 9;       // fred output, |r| <= q/2 + 2
constexpr int LIM_MUL = 64;   // fmm input, |a| <= 4q (q < 2^50: |a wq| <= 2q < 2^51, |a| < 2^52)
constexpr int LIM_VAL = 128;  // any value, |v| <= 8q < 2^53

// product with an 8-byte table entry w (wq = fl(w fl(1/q)) formed here: |wq - w/q| <= 2^-53, so
// |a wq - a w/q| <= 1/2 for |a| <= 4q and |r| <= q).  Halves the table bytes of the pointwise products.
constexpr int UMUL8 = 16;
__device__ __forceinline__ double fmm8(double a, double w, double q, double qi) {
    const double h = __dmul_rn(a, w);
    const double l = __fma_rn(a, w, -h);
    const double t = __dsub_rn(__fma_rn(a, __dmul_rn(w, qi), RND), RND);
    const double r = __fma_rn(-t, q, h);
    return __dadd_rn(r, l);
}
// make v[k] a valid fmm input / keep the exact range
template <int E>
__device__ __forceinline__ void need(double (&v)[E], int (&bd)[E], int k, int lim, double q, double qi) {
    if (bd[k] > lim) { v[k] = fred(v[k], q, qi); bd[k] = URED; }
}
// at a register-pass boundary: every register takes the largest bound (the exchange permutes them);
// if the NS stages ahead would push fmm inputs past LIM_MUL, reduce all now (each value once per pass
// instead of the y operands of every later stage and the epilogue operands)
template <int E>
__device__ __forceinline__ void flatten(double (&v)[E], int (&bd)[E], int ns, double q, double qi) {
    int mx = 0;
#pragma unroll
    for (int k = 0; k < E; ++k) mx = bd[k] > mx ? bd[k] : mx;
    const bool red = mx + UMUL * ns > LIM_MUL;
#pragma unroll
    for (int k = 0; k < E; ++k) {
        if (red) v[k] = fred(v[k], q, qi);
        bd[k] = red ? URED : mx;
    }
}

// One register pass of NS <= LOGE stages on registers k, k + 2^u (u = stage within the pass).
// FWD (natural -> bit-reversed, DIF order u = NS-1 .. 0): block b = i >> (lh+1) of the held index i,
//   s = tb[b] = omega_L^{brev_{logL-1}(b)};  b = ((tau >> LO) << (LOGE-u-1)) + (k >> (u+1)).
// INV (bit-reversed -> natural, u = 0 .. NS-1): s = omega_L^{-(i mod h) L/2h} (as ntt2.cu).
// Both: y' = s y, (x, y) <- (x + y', x - y').  s = 1 is skipped where it is known at compile time.
// Passes after the first take their twiddles from a per-thread table pt[e * TPR] (smem, entry-major,
// thread-minor: conflict-free), e = the entry of (stage u, block or kpart) below; the first pass
// (FWD: TOP, INV: LO = 0) has compile-time indices into tw (broadcast reads).
__host__ __device__ constexpr int pt_entry_f(int LOGE, int u, int bk) { return (1 << LOGE) - (1 << (LOGE - u)) + bk; }
__host__ __device__ constexpr int pt_entry_i(int u, int kp) { return (1 << u) - 1 + kp; }

template <int LOGE, int NS, bool FWD, int LO, bool TOP>
__device__ __forceinline__ void freg_pass(double (&v)[1 << LOGE], int (&bd)[1 << LOGE], uint32_t tau, const double2 *__restrict__ tw,
                                          const double2 *__restrict__ pt, int TPR, int logL, double q, double qi) {
    constexpr int E = 1 << LOGE;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        const int u = FWD ? (NS - 1 - s) : s;
        const int lh = LO + u;
#pragma unroll
        for (int k = 0; k < E; ++k) {
            if (k & (1 << u)) continue;
            const int k2 = k + (1 << u);
            if (bd[k2] == 0) {          // y known to be exactly 0 (bound 0): (x + 0, x - 0) = (x, x)
                v[k2] = v[k];
                bd[k2] = bd[k];
                continue;
            }
            bool trivial;
            uint32_t ti;
            if (FWD) {
                const uint32_t bk = (uint32_t)(k >> (u + 1));
                trivial = TOP && bk == 0;                       // TOP: tau >> LO == 0
                ti = TOP ? bk : (((tau >> LO) << (LOGE - u - 1)) + bk);
            } else {
                const uint32_t kpart = (uint32_t)(k & ((1 << u) - 1));
                trivial = LO == 0 && kpart == 0;
                ti = ((tau & ((1u << LO) - 1)) + (kpart << LO)) << (logL - 1 - lh);
            }
            double y;
            int by;
            if (trivial) {
                y = v[k2];
                by = bd[k2];
                if (bd[k] + by > LIM_VAL) { need(v, bd, k2, 0, q, qi); y = v[k2]; by = URED; }
            } else {
                need(v, bd, k2, LIM_MUL, q, qi);
                const bool first = FWD ? TOP : (LO == 0);
                const int e = FWD ? pt_entry_f(LOGE, u, k >> (u + 1)) : pt_entry_i(u, k & ((1 << u) - 1));
                y = fmm(v[k2], first ? tw[ti] : pt[e * TPR], q);
                by = UMUL;
            }
            need(v, bd, k, LIM_VAL - by, q, qi);
            const double x = v[k];
            v[k] = __dadd_rn(x, y);
            v[k2] = __dsub_rn(x, y);
            bd[k] = bd[k2] = bd[k] + by;
        }
    }
}

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

template <int LOGE>
__device__ __forceinline__ uint32_t held_index(uint32_t tau, int lo, int k) {
    return (tau & ((1u << lo) - 1)) + ((tau >> lo) << (lo + LOGE)) + ((uint32_t)k << lo);
}

// per-thread twiddle tables of passes 1 .. NP-1 of one transform direction: pt[((P-1) NE + e) TPR + tau]
template <int LOGL, int LOGE, bool FWD>
struct PtTab {
    static constexpr int NE = (1 << LOGE) - 1;
    static constexpr int TPR = 1 << (LOGL - LOGE);
    static constexpr int NPT = Passes<LOGL, LOGE>::NP - 1;
    static constexpr int WORDS = NPT > 0 ? NPT * NE * TPR : 1;   // double2 entries
    __device__ static void fill(double2 *pt, uint32_t tau, const double2 *__restrict__ tw) {
        typedef Passes<LOGL, LOGE> PS;
#pragma unroll
        for (int P = 1; P < PS::NP; ++P) {
            const int lo = FWD ? PS::dif_lo(P) : PS::dit_lo(P);
            const int ns = FWD ? PS::dif_ns(P) : PS::dit_ns(P);
            double2 *d = pt + (size_t)(P - 1) * NE * TPR + tau;
            for (int u = 0; u < ns; ++u) {
                if (FWD) {
                    for (int j = 0; j < (1 << (LOGE - 1 - u)); ++j)
                        d[pt_entry_f(LOGE, u, j) * TPR] = tw[((tau >> lo) << (LOGE - u - 1)) + j];
                } else {
                    for (int j = 0; j < (1 << u); ++j)
                        d[pt_entry_i(u, j) * TPR] = tw[((tau & ((1u << lo) - 1)) + ((uint32_t)j << lo)) << (LOGL - 1 - lo - u)];
                }
            }
        }
    }
};

// second half of a split cluster barrier (ntt4.cu: the arrive is issued after the tile reads, the wait
// only before the first shared-memory exchange overwrites the tile buffer)
__device__ __forceinline__ void cluster_wait_acq() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

// row transform (element i at srow[i + (i >> LOGE)]); CW: cluster wait before the first exchange
template <int LOGL, int LOGE, bool FWD, int P, bool CW = false>
__device__ __forceinline__ void frt_pass(double (&v)[1 << LOGE], int (&bd)[1 << LOGE], uint32_t tau, double *srow,
                                         const double2 *__restrict__ tw, const double2 *__restrict__ pt, double q, double qi) {
    typedef Passes<LOGL, LOGE> PS;
    constexpr int E = 1 << LOGE;
    constexpr int lo = FWD ? PS::dif_lo(P) : PS::dit_lo(P);
    constexpr int ns = FWD ? PS::dif_ns(P) : PS::dit_ns(P);
    if (P > 0) {
        constexpr int plo = FWD ? PS::dif_lo(P > 0 ? P - 1 : 0) : PS::dit_lo(P > 0 ? P - 1 : 0);
        if (CW && P == 1) cluster_wait_acq();
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
        flatten(v, bd, ns, q, qi);
    }
    constexpr int TPR = 1 << (LOGL - LOGE);
    freg_pass<LOGE, ns, FWD, lo, (FWD && P == 0)>(v, bd, tau, tw, pt + (size_t)(P > 0 ? P - 1 : 0) * (E - 1) * TPR + tau,
                                                  TPR, LOGL, q, qi);
    if (P + 1 < PS::NP) frt_pass<LOGL, LOGE, FWD, (P + 1 < PS::NP ? P + 1 : P), CW>(v, bd, tau, srow, tw, pt, q, qi);
}

// column transform (element i of column col at scol[i * TC + col]); CW as frt_pass
template <int LOGL, int LOGE, bool FWD, int TC, int P, bool CW = false>
__device__ __forceinline__ void fct_pass(double (&v)[1 << LOGE], int (&bd)[1 << LOGE], uint32_t tau, uint32_t col,
                                         double *scol, const double2 *__restrict__ tw, const double2 *__restrict__ pt, double q, double qi) {
    typedef Passes<LOGL, LOGE> PS;
    constexpr int E = 1 << LOGE;
    constexpr int lo = FWD ? PS::dif_lo(P) : PS::dit_lo(P);
    constexpr int ns = FWD ? PS::dif_ns(P) : PS::dit_ns(P);
    if (P > 0) {
        constexpr int plo = FWD ? PS::dif_lo(P > 0 ? P - 1 : 0) : PS::dit_lo(P > 0 ? P - 1 : 0);
        if (CW && P == 1) cluster_wait_acq();
#pragma unroll
        for (int k = 0; k < E; ++k) scol[held_index<LOGE>(tau, plo, k) * TC + col] = v[k];
        __syncthreads();
#pragma unroll
        for (int k = 0; k < E; ++k) v[k] = scol[held_index<LOGE>(tau, lo, k) * TC + col];
        __syncthreads();
        flatten(v, bd, ns, q, qi);
    }
    constexpr int TPR = 1 << (LOGL - LOGE);
    freg_pass<LOGE, ns, FWD, lo, (FWD && P == 0)>(v, bd, tau, tw, pt + (size_t)(P > 0 ? P - 1 : 0) * (E - 1) * TPR + tau,
                                                  TPR, LOGL, q, qi);
    if (P + 1 < PS::NP) fct_pass<LOGL, LOGE, FWD, TC, (P + 1 < PS::NP ? P + 1 : P), CW>(v, bd, tau, col, scol, tw, pt, q, qi);
}

#ifndef NTTF_LOGE_89
#define NTTF_LOGE_89 3     // registers per thread 2^LOGE of the 512-point row transforms (M = 131072)
#endif
#ifndef NTT_REG_TARGET
#define NTT_REG_TARGET 64
#endif
#define FNTT_MINB(threads) ((65536 / NTT_REG_TARGET) / (threads) > 0 ? (65536 / NTT_REG_TARGET) / (threads) : 1)

struct JobF {
    uint32_t poly, lb, pr;
};
__device__ __forceinline__ JobF job_f(const LimbMap &lm, uint32_t job) {
    JobF j;
    const uint32_t jl = job / lm.npoly;
    j.poly = job - jl * lm.npoly;
    j.lb = lm.limb(jl);
    j.pr = lm.prime(j.lb);
    return j;
}
}  // namespace f64
}  // namespace bc
