// ntt3.cu -- Bluestein NTT passes in binary64 FMA arithmetic for sm_100a (a1/a2).
//
// Why binary64: every prime of the paper's sets must be = 1 (mod lcm(p, m, M)) (R1), which is
// > 2^32 for all of them, so residues need 64-bit words.  On B200 the FP64 pipe issues 64 DFMA per
// clock per SM -- the same rate as the 32-bit IMAD pipe -- and one exact modular product of
// residues below 2^50 costs 6 binary64 operations (DMUL, 3 DFMA, 2 DADD) against ~10 IMAD-class
// plus 4-6 ALU instructions for the 64-bit Shoup product (ntt2.cu).  Measured on B200 in a register
// microbenchmark (tools/micro/bfly_micro.cu): 1.53e12 FP64 butterflies/s vs 0.89e12 Shoup ones.
//
// Representation: a residue class mod q (q < 2^50) is held as a signed integer-valued double v,
// |v| <= 8q < 2^53 (exact).  The modular product with a table entry (w, wq), w in (-q/2, q/2]
// centred and wq = fl(w/q), is
//     h = fl(a w); l = a w - h (exact, one FMA); t = rint(a wq) (FMA with 1.5*2^52, DADD);
//     r = (h - t q) + l   (both steps exact: the results are integers below 2^53),
// exact for |a| <= 4q, with |r| <= (1/2 + 1/8) q.  A reduction x - rint(x/q) q gives |x| <= q/2 + 2.
// Bounds are tracked per register at compile time (units of q/16) and a value is reduced only when
// the next operation would leave the exact range, so the lazy growth of the Cooley-Tukey
// butterflies (+0.625 q per stage) costs about one reduction per value per six stages.
//
// Structure, layouts and tables are those of ntt2.cu (four-step M = R x C; pass A: chirp + column
// forward transform + cross twiddle; pass B: row forward, x D^, row inverse, cross twiddle; pass C:
// column inverse + output chirp + Z_m^* gather or reduction input), except that the forward
// (natural -> bit-reversed) sub-transforms use Cooley-Tukey butterflies (x + s y, x - s y) with one
// twiddle s = omega_L^{brev(b)} per block b (the CRT splitting X^{2h} - c = (X^h - s)(X^h + s)),
// whose bounds grow linearly, instead of Gentleman-Sande butterflies whose sums double per stage.
// The output order (bit-reversed) and therefore every table and the results are unchanged.
//
// Further structure used here (all exact, results identical to the integer passes):
//  - pointwise tables (chirps, D^, cross twiddles) are 8-byte centred residues, fl(w/q) formed in a
//    register (fmm8, |r| <= q); D^ is stored in pass B's thread-minor order (coalesced);
//  - passes after the first read their twiddles from per-thread shared-memory tables (conflict-free);
//  - the upper half of every pass-A input is zero (M/2 >= m > n) and is a compile-time zero (bound 0),
//    and the rows >= R/2 of pass C are never output (their last-stage differences are dead code);
//  - prime m, inverse: kf_corner computes A_{m-1} per job after pass B, so pass C writes the reduction
//    A_t - A_{m-1} mod Phi_m directly (no separate reduction pass);
//  - composite m, inverse: modes 2 / 3 of the same passes (no chirps, index maps, the constant's
//    transform in place of D^) run the Barrett division by Phi_m at the smallest sufficient size Mb,
//    the quotient as a sparse sum of shifted copies (k_ir_sparse) when Phi_m^{-1} mod x^(m-n) is short.
#include <cuda_runtime.h>

#include <algorithm>

#include "nttf_core.cuh"

namespace bc {

namespace f64 {

// pass A: chirp, column forward transform (length R), x psi^(c brev(rp)); scratch[rp*C + c] (doubles, |v| <= 0.625q)
template <int LOGR, int LOGE, int TC, int INV, int LOGC>
__global__ void __launch_bounds__(TC * (1 << (LOGR - LOGE)), FNTT_MINB(TC * (1 << (LOGR - LOGE))))
    kf_passA(NttTables T, const uint64_t *__restrict__ in, uint64_t in_pstride, LimbMap lm, uint64_t job0,
             double *__restrict__ scratch) {
    constexpr int E = 1 << LOGE, R = 1 << LOGR;
    constexpr uint32_t CC = 1u << LOGC;
    extern __shared__ double smf[];
    const uint32_t job = (uint32_t)(job0 + blockIdx.y);
    const JobF J = job_f(lm, job);
    const double q = T.fmods[J.pr].x, qi = T.fmods[J.pr].y;
    const uint32_t col = threadIdx.x % TC, tau = threadIdx.x / TC;
    const uint32_t c = blockIdx.x * TC + col;
    // INV: 0 Bluestein forward, 1 Bluestein inverse, 2/3 the Barrett reduction mod Phi_m of a composite m
    // (2: quotient convolution, input rev(A)_t = A_{m-1-t}, t < m - n; 3: Phi_m * Q, input Q_t = A'_{n+t})
    const double *tf = (INV == 1 ? T.ftf1i : T.ftf1) + (uint64_t)J.pr * T.m;
    const uint64_t *src = INV >= 2 ? in + (uint64_t)blockIdx.y * (INV == 3 && T.q_in_s2 ? T.M : T.Mslot) : in + (uint64_t)J.poly * in_pstride + (uint64_t)J.lb * T.n;
    typedef PtTab<LOGR, LOGE, true> PTT;
    double2 *stw = (double2 *)(smf + (size_t)R * TC), *spt = stw + R / 2;
    const double2 *gtw = T.ftwRb + (uint64_t)J.pr * (R / 2);
    for (int j = threadIdx.x; j < R / 2; j += blockDim.x) stw[j] = gtw[j];
    if (col == 0) PTT::fill(spt, tau, gtw);
    double v[E];
    int bd[E];
#pragma unroll
    for (int k = 0; k < E; ++k) {
        const uint32_t r = held_index<LOGE>(tau, LOGR - LOGE, k);
        const uint32_t t = r * CC + c;
        double x = 0.0;
        if (k >= E / 2) {
            // rows >= R/2: t >= M/2, the zero half of the input (Bluestein: M/2 >= m > n; Barrett modes:
            // Mb >= 2k - 1 so k <= Mb/2; bound 0 = exactly 0: the first forward stage copies)
            v[k] = 0.0;
            bd[k] = 0;
            continue;
        }
        if (INV == 0) {
            if (t < T.n) {
                const double xin = (T.dbg & 64) ? (double)t : from_u64(__ldcs(src + t));
                x = (T.dbg & 1) ? xin : fmm8(xin, tf[t], q, qi);
            }
        } else if (INV == 1) {
            if (t < T.m) {
                const int ps = T.pos[t];
                if (ps >= 0) x = fmm8(from_u64(__ldcs(src + ps)), tf[t], q, qi);
            }
        } else if (t < T.m - T.n) {
            x = from_u64(src[INV == 2 ? T.m - 1 - t : (T.q_in_s2 ? t : T.n + t)]);   // canonical, bound q (UMUL8)
        }
        v[k] = x;
        bd[k] = UMUL8;
    }
    __syncthreads();
    fct_pass<LOGR, LOGE, true, TC, 0>(v, bd, tau, col, smf, stw, spt, q, qi);
    const double *xt = T.fxta + (uint64_t)J.pr * T.M;
    double *dst = scratch + (uint64_t)blockIdx.y * T.M;
#pragma unroll
    for (int k = 0; k < E; ++k) {
        const uint32_t rp = held_index<LOGE>(tau, 0, k);
        need(v, bd, k, LIM_MUL, q, qi);
        __stcs(dst + rp * CC + c, (T.dbg & 2) ? fred(v[k], q, qi) : fmm8(v[k], xt[rp * CC + c], q, qi));
    }
}

// pass A, persistent (forward Bluestein): CTA (column group, g) runs jobs g, g + G, ... of its column group.
// The group's chirp and cross-twiddle tiles (per prime) stay in shared memory across those jobs, and each
// thread prefetches the next job's inputs into a shared staging tile with cp.async (LDGSTS) while the
// current job is transformed; every thread reads back exactly the words it copied, so cp.async.wait_group
// suffices (no barrier).  Results are identical to kf_passA (same arithmetic, same order).
// fused forward epilogue (NttEpi, kernels.h): x = the transform's canonical output word at position i of poly
// `poly`, limb lb -> (u - x) w_lb or (u + pm_lb d - x) w_lb, the values ew_scale_sub / ew_fused_down_out compute
__device__ __forceinline__ uint64_t epi_apply(const NttEpi &e, uint32_t poly, uint32_t lb, uint32_t n, uint32_t i,
                                              uint64_t x) {
    const uint64_t q = e.mods[lb].q;
    const uint64_t off = (uint64_t)lb * n + i;
    uint64_t u = __ldcs(e.u + (uint64_t)poly * e.ups + off);
    if (e.mode == 2) {
        const u64x2 pm = e.pm[lb];
        const uint64_t d = __ldcs(e.d + (uint64_t)(poly >> 1) * e.dbs + (uint64_t)(poly & 1) * e.dks + off);
        u = add_mod(u, mul_shoup(d, pm.w, pm.ws, q), q);
    }
    const u64x2 w = e.w[lb];
    return mul_shoup(sub_mod(u, x, q), w.w, w.ws, q);
}

__device__ __forceinline__ void cp_async8(void *sdst, const void *gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(sdst)), "l"(gsrc)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <int LOGR, int LOGE, int TC, int CCV, int LEAN = 0>
struct PersistA {
    static constexpr int R = 1 << LOGR, E = 1 << LOGE;
    typedef PtTab<LOGR, LOGE, true> PTT;
    // LEAN 0 -- doubles: exchange R*TC, chirp tile (R/2)*TC, cross-twiddle tile R*TC, staging (R/2)*TC; int32
    // position tile (R/2)*TC (inverse gather); double2: twiddles.  LEAN >= 1 (tables read through L1 / L2, positions
    // computed or read from T.pos): exchange + staging + twiddles only, 4 CTAs of 256 threads per SM.
    static constexpr size_t SMEM = LEAN ? ((size_t)R * TC + (size_t)(R / 2) * TC) * 8 + ((size_t)R / 2 + PTT::WORDS) * 16
                                        : ((size_t)R * TC * 2 + (size_t)R * TC) * 8 + (size_t)(R / 2) * TC * 4 +
                                              ((size_t)R / 2 + PTT::WORDS) * 16;
};

// INV 0: forward (input t < n), 1: inverse (input gathered through pos[t], t < m).  LEAN 0: the group's
// chirp / cross-twiddle / position tiles resident in shared memory (2 CTAs per SM); LEAN >= 1: the same values
// read from the global tables (L2-resident) at their point of use, at MINB CTAs per SM.
template <int LOGR, int LOGE, int TC, int CCV, int INV, int LEAN = 0, int MINB = 2>
__global__ void __launch_bounds__(TC * (1 << (LOGR - LOGE)), MINB)
    kf_passA_p(NttTables T, const uint64_t *__restrict__ in, uint64_t in_pstride, LimbMap lm, uint64_t job0, uint32_t nj,
               double *__restrict__ scratch) {
    typedef PersistA<LOGR, LOGE, TC, CCV, LEAN> PA;
    constexpr int E = 1 << LOGE, R = 1 << LOGR;
    constexpr uint32_t CC = CCV;          // columns (a power of two, or 256 r N' for the mixed-radix lengths)
    extern __shared__ double smf[];
    double *scol = smf, *ttf = scol + R * TC, *txt = ttf + (LEAN ? 0 : (R / 2) * TC);
    uint64_t *stage = (uint64_t *)(LEAN ? ttf : txt + R * TC);
    double2 *stw = (double2 *)(stage + (R / 2) * TC), *spt = stw + R / 2;
    int32_t *tpos = (int32_t *)(spt + PA::PTT::WORDS);
    const uint32_t col = threadIdx.x % TC, tau = threadIdx.x / TC;
    const uint32_t c = blockIdx.x * TC + col;
    const uint32_t G = gridDim.y;
    const uint32_t tlim = INV ? T.m : T.n;
    // input position of row r of this thread's column (-1: zero)
    auto posf = [&](uint32_t r) -> int {
        const uint32_t t = r * CC + c;
        if (!INV) return t < T.n ? (int)t : -1;
        if (!LEAN) return tpos[r * TC + col];
        return t < T.m ? T.pos[t] : -1;
    };
    if (!LEAN && INV) {    // the position tile does not depend on the prime: filled once
        for (int i = threadIdx.x; i < (R / 2) * TC; i += blockDim.x) {
            const uint32_t t = (uint32_t)(i / TC) * CC + blockIdx.x * TC + (uint32_t)(i % TC);
            tpos[i] = t < T.m ? T.pos[t] : -1;
        }
        __syncthreads();
    }
    // staging words that no job copies (position -1) hold 0 for the whole kernel: the input products below
    // are then branch-free (fmm8(0, w) = 0)
#pragma unroll
    for (int k = 0; k < E / 2; ++k) {
        const uint32_t r = held_index<LOGE>(tau, LOGR - LOGE, k);
        if (posf(r) < 0) stage[r * TC + col] = 0;
    }
    uint32_t cur_pr = 0xffffffffu;
    auto prefetch = [&](uint32_t jj) {
        const JobF Jn = job_f(lm, (uint32_t)(job0 + jj));
        const uint64_t *sn = in + (uint64_t)Jn.poly * in_pstride + (uint64_t)Jn.lb * T.n;
#pragma unroll
        for (int k = 0; k < E / 2; ++k) {
            const uint32_t r = held_index<LOGE>(tau, LOGR - LOGE, k);
            const int ps = posf(r);
            if (ps >= 0) cp_async8(stage + r * TC + col, sn + ps);
        }
        cp_async_commit();
    };
    if (blockIdx.y < nj) prefetch(blockIdx.y);
    for (uint32_t jj = blockIdx.y; jj < nj; jj += G) {
        const JobF J = job_f(lm, (uint32_t)(job0 + jj));
        const double q = T.fmods[J.pr].x, qi = T.fmods[J.pr].y;
        const double *tf = (INV ? T.ftf1i : T.ftf1) + (uint64_t)J.pr * T.m, *xt = T.fxta + (uint64_t)J.pr * T.M;
        if (J.pr != cur_pr) {           // uniform over the CTA: the tiles of this prime
            __syncthreads();
            const double2 *gtw = T.ftwRb + (uint64_t)J.pr * (R / 2);
            for (int j = threadIdx.x; j < R / 2; j += blockDim.x) stw[j] = gtw[j];
            if (col == 0) PA::PTT::fill(spt, tau, gtw);
            if (!LEAN) {
                for (int i = threadIdx.x; i < (R / 2) * TC; i += blockDim.x) {
                    const uint32_t t = (uint32_t)(i / TC) * CC + blockIdx.x * TC + (uint32_t)(i % TC);
                    ttf[i] = t < tlim ? tf[t] : 0.0;
                }
                for (int i = threadIdx.x; i < R * TC; i += blockDim.x)
                    txt[i] = xt[(uint32_t)(i / TC) * CC + blockIdx.x * TC + (uint32_t)(i % TC)];
            }
            cur_pr = J.pr;
            __syncthreads();
        }
        cp_async_wait_all();            // this thread's staged inputs of job jj
        double v[E];
        int bd[E];
#pragma unroll
        for (int k = 0; k < E; ++k) {
            if (k >= E / 2) {           // rows >= R/2: the zero half of the Bluestein input
                v[k] = 0.0;
                bd[k] = 0;
                continue;
            }
            const uint32_t r = held_index<LOGE>(tau, LOGR - LOGE, k);
            const uint32_t t = r * CC + c;
            v[k] = fmm8(from_u64(stage[r * TC + col]), LEAN ? __ldg(tf + (t < tlim ? t : tlim - 1)) : ttf[r * TC + col], q, qi);
            bd[k] = UMUL8;
        }
        if (jj + G < nj) prefetch(jj + G);   // the next job's inputs while this one is transformed
        fct_pass<LOGR, LOGE, true, TC, 0>(v, bd, tau, col, scol, stw, spt, q, qi);
        double *dst = scratch + (uint64_t)jj * T.M;
#pragma unroll
        for (int k = 0; k < E; ++k) {
            const uint32_t rp = held_index<LOGE>(tau, 0, k);
            need(v, bd, k, LIM_MUL, q, qi);
            __stcs(dst + rp * CC + c, fmm8(v[k], LEAN ? __ldg(xt + rp * CC + c) : txt[rp * TC + col], q, qi));
        }
    }
    cp_async_wait_all();
}

// pass C, persistent: column inverse + output chirp + Z_m^* gather (INV 0) or A_t - A_{m-1} (INV 1, prime m,
// corner[] from kf_corner).  As kf_passA_p: per-prime output-chirp tile and the position tile in shared
// memory (LEAN 0), the next job's pass-B output prefetched with cp.async while this one is transformed.
// LEAN 1: chirp and positions read from the global tables; LEAN 2: in addition the staging tile is the
// exchange buffer (the next job's prefetch is issued after the exchange, overlapping the second register
// pass and the epilogue), so 4 CTAs of 256 threads fit an SM; LEAN 4: tiles in shared memory, staging tile
// as exchange buffer (3 CTAs per SM).
template <int LOGR, int LOGE, int TC, int CCV, int LEAN = 0>
struct PersistC {
    static constexpr int R = 1 << LOGR;
    typedef PtTab<LOGR, LOGE, false> PTT;
    // doubles: exchange R*TC, staging R*TC, chirp tile (R/2)*TC; int32 positions (R/2)*TC; double2 twiddles
    static constexpr bool GT = LEAN == 1 || LEAN == 2;     // chirp / positions from the global tables
    static constexpr bool XCH = LEAN == 2 || LEAN == 4;    // the staging tile is the exchange buffer
    static constexpr size_t SMEM = (size_t)R * TC * 8 * (XCH ? 1 : 2) + (GT ? 0 : (size_t)(R / 2) * TC * 12) +
                                   ((size_t)R / 2 + PTT::WORDS) * 16;
};

template <int LOGR, int LOGE, int TC, int CCV, int INV, int LEAN = 0, int MINB = 2>
__global__ void __launch_bounds__(TC * (1 << (LOGR - LOGE)), MINB)
    kf_passC_p(NttTables T, uint64_t *__restrict__ out, uint64_t out_pstride, LimbMap lm, uint64_t job0, uint32_t nj,
               const double *__restrict__ scratch, const uint64_t *__restrict__ corner) {
    typedef PersistC<LOGR, LOGE, TC, CCV, LEAN> PC;
    typedef Passes<LOGR, LOGE> PS;
    constexpr bool GT = PC::GT, XCH = PC::XCH;
    static_assert(!XCH || PS::NP == 2, "staging tile as exchange buffer: two register passes");
    constexpr int E = 1 << LOGE, R = 1 << LOGR;
    constexpr uint32_t CC = CCV;
    extern __shared__ double smf[];
    double *scol = smf, *stage = XCH ? scol : scol + R * TC, *tfo = stage + R * TC;
    int32_t *tpos = (int32_t *)(tfo + (R / 2) * TC);
    double2 *stw = (double2 *)(GT ? tfo : (double *)(tpos + (R / 2) * TC)), *spt = stw + R / 2;
    const uint32_t col = threadIdx.x % TC, tau = threadIdx.x / TC;
    const uint32_t c = blockIdx.x * TC + col;
    const uint32_t G = gridDim.y;
    auto posf = [&](uint32_t r) -> int {
        if (!GT) return tpos[r * TC + col];
        const uint32_t t = r * CC + c;
        return INV ? (t < T.n ? (int)t : -1) : (t < T.m ? T.pos[t] : -1);
    };
    if (!GT) {
        for (int i = threadIdx.x; i < (R / 2) * TC; i += blockDim.x) {
            const uint32_t t = (uint32_t)(i / TC) * CC + blockIdx.x * TC + (uint32_t)(i % TC);
            tpos[i] = INV ? (t < T.n ? (int32_t)t : -1) : (t < T.m ? T.pos[t] : -1);
        }
        __syncthreads();
    }
    uint32_t cur_pr = 0xffffffffu;
    auto prefetch = [&](uint32_t jj) {
        const double *src = scratch + (uint64_t)jj * T.M;
#pragma unroll
        for (int k = 0; k < E; ++k) {
            const uint32_t rp = held_index<LOGE>(tau, 0, k);
            cp_async8(stage + rp * TC + col, src + rp * CC + c);
        }
        cp_async_commit();
    };
    if (blockIdx.y < nj) prefetch(blockIdx.y);
    for (uint32_t jj = blockIdx.y; jj < nj; jj += G) {
        const JobF J = job_f(lm, (uint32_t)(job0 + jj));
        const double q = T.fmods[J.pr].x, qi = T.fmods[J.pr].y;
        const double *tf = (INV ? T.ftfoi : T.ftfo) + (uint64_t)J.pr * T.m;
        if (J.pr != cur_pr) {
            __syncthreads();
            const double2 *gtw = T.ftwRi + (uint64_t)J.pr * (R / 2);
            for (int j = threadIdx.x; j < R / 2; j += blockDim.x) stw[j] = gtw[j];
            if (col == 0) PC::PTT::fill(spt, tau, gtw);
            if (!GT) {
                for (int i = threadIdx.x; i < (R / 2) * TC; i += blockDim.x) {
                    const uint32_t t = (uint32_t)(i / TC) * CC + blockIdx.x * TC + (uint32_t)(i % TC);
                    tfo[i] = t < T.m ? tf[t] : 0.0;
                }
            }
            cur_pr = J.pr;
            __syncthreads();
        }
        cp_async_wait_all();
        double v[E];
        int bd[E];
#pragma unroll
        for (int k = 0; k < E; ++k) {
            v[k] = stage[held_index<LOGE>(tau, 0, k) * TC + col];
            bd[k] = UMUL8;
        }
        if (!XCH) {
            if (jj + G < nj) prefetch(jj + G);
            fct_pass<LOGR, LOGE, false, TC, 0>(v, bd, tau, col, scol, stw, spt, q, qi);
        } else {
            // fct_pass<.., 0> written out: register pass 0, exchange through the staging tile (each thread
            // writes back exactly the words it read), prefetch of the next job once every thread has read its
            // exchanged values, register pass 1
            constexpr int TPR = 1 << (LOGR - LOGE);
            freg_pass<LOGE, PS::dit_ns(0), false, PS::dit_lo(0), false>(v, bd, tau, stw, spt + tau, TPR, LOGR, q, qi);
#pragma unroll
            for (int k = 0; k < E; ++k) scol[held_index<LOGE>(tau, PS::dit_lo(0), k) * TC + col] = v[k];
            __syncthreads();
#pragma unroll
            for (int k = 0; k < E; ++k) v[k] = scol[held_index<LOGE>(tau, PS::dit_lo(1), k) * TC + col];
            __syncthreads();
            if (jj + G < nj) prefetch(jj + G);
            flatten(v, bd, PS::dit_ns(1), q, qi);
            freg_pass<LOGE, PS::dit_ns(1), false, PS::dit_lo(1), false>(v, bd, tau, stw, spt + tau, TPR, LOGR, q, qi);
        }
        uint64_t *dst = out + (uint64_t)J.poly * out_pstride + (uint64_t)J.lb * T.n;
        const uint64_t cn = INV ? corner[jj] : 0;
#pragma unroll
        for (int k = 0; k < E / 2; ++k) {   // rows >= R/2: t >= M/2 >= m, never output
            const uint32_t r = held_index<LOGE>(tau, LOGR - LOGE, k);
            const int ps = posf(r);
            if (ps < 0) continue;
            need(v, bd, k, LIM_MUL, q, qi);
            const uint64_t x = to_u64(fmm8(v[k], GT ? __ldg(tf + r * CC + c) : tfo[r * TC + col], q, qi), q);
            __stcs(dst + ps, INV ? (x >= cn ? x - cn : x + (uint64_t)q - cn)
                                 : (T.epi.mode ? epi_apply(T.epi, J.poly, J.lb, T.n, (uint32_t)ps, x) : x));
        }
    }
    cp_async_wait_all();
}

// pass B: row forward (length C), x D^, row inverse, x psi^(-c brev(r)); block = RB rows x C/E threads
template <int LOGC, int LOGE, int RB, int INV>
__global__ void __launch_bounds__(RB * (1 << (LOGC - LOGE)), FNTT_MINB(RB * (1 << (LOGC - LOGE))))
    kf_passB(NttTables T, LimbMap lm, uint64_t job0, double *__restrict__ scratch) {
    constexpr int E = 1 << LOGE, C = 1 << LOGC, TPR = C / E;
    constexpr int ROWW = C + C / E;
    extern __shared__ double smf[];
    const uint32_t job = (uint32_t)(job0 + blockIdx.y);
    const JobF J = job_f(lm, job);
    const double q = T.fmods[J.pr].x, qi = T.fmods[J.pr].y;
    const uint32_t rr = threadIdx.x / TPR, tau = threadIdx.x % TPR;
    const uint32_t row = blockIdx.x * RB + rr;
    double *srow = smf + rr * ROWW;
    double *grow = scratch + (uint64_t)blockIdx.y * T.M + (uint64_t)row * C;
    typedef PtTab<LOGC, LOGE, true> PTF;
    typedef PtTab<LOGC, LOGE, false> PTI;
    double2 *tw = (double2 *)(smf + (size_t)RB * ROWW), *twi = tw + C / 2, *ptf = twi + C / 2, *pti = ptf + PTF::WORDS;
    const double2 *gtw = T.ftwCb + (uint64_t)J.pr * (C / 2), *gtwi = T.ftwCi + (uint64_t)J.pr * (C / 2);
    for (int j = threadIdx.x; j < C / 2; j += blockDim.x) {
        tw[j] = gtw[j];
        twi[j] = gtwi[j];
    }
    if (rr == 0) PTF::fill(ptf, tau, gtw);
    if (rr == 1 % RB) PTI::fill(pti, tau, gtwi);
    double v[E];
    int bd[E];
#pragma unroll
    for (int k = 0; k < E; ++k) {
        v[k] = __ldcs(grow + held_index<LOGE>(tau, LOGC - LOGE, k));
        bd[k] = UMUL8;
    }
    __syncthreads();
    frt_pass<LOGC, LOGE, true, 0>(v, bd, tau, srow, tw, ptf, q, qi);
    // D^ in the thread-minor layout of this pass (entry of position tau*E + k at k*TPR + tau: coalesced)
    const double *dh = (INV == 0 ? T.fdhf : INV == 1 ? T.fdhi : INV == 2 ? T.fdhb1 : T.fdhb2) + (uint64_t)J.pr * T.M + (uint64_t)row * C + tau;
#pragma unroll
    for (int k = 0; k < E; ++k) {
        need(v, bd, k, LIM_MUL, q, qi);
        v[k] = (T.dbg & 4) ? fred(v[k], q, qi) : fmm8(v[k], dh[k * TPR], q, qi);
        bd[k] = UMUL8;
    }
    frt_pass<LOGC, LOGE, false, 0>(v, bd, tau, srow, twi, pti, q, qi);
    const double *xt = T.fxtb + (uint64_t)J.pr * T.M + (uint64_t)row * C;
#pragma unroll
    for (int k = 0; k < E; ++k) {
        const uint32_t cc = held_index<LOGE>(tau, LOGC - LOGE, k);
        need(v, bd, k, LIM_MUL, q, qi);
        __stcs(grow + cc, (T.dbg & 8) ? fred(v[k], q, qi) : fmm8(v[k], xt[cc], q, qi));
    }
}

// ---- R25 mixed-radix rows (f3): C = RAD * 2^LOGN.  Forward row DFT by decimation in frequency:
//   u_i[j] = omega_C^{i j} * DFT_RAD(x_j, x_{j+N'}, ..., x_{j+(RAD-1)N'})_i   (j < N' = 2^LOGN, i < RAD),
//   X[i + RAD k'] = NTT_N'(u_i)[k'] (the power-of-two sub-row transforms of the register passes, output
//   bit-reversed: sub-row i, position p holds k' = brev(p)); the inverse runs the steps backwards with the
//   inverse roots (unnormalised, as every inverse here).  Any exact DFT algorithm gives the same residues.
// small DFTs (fmm8 products; inputs |x| <= q, outputs |y| <= 3q)
__device__ __forceinline__ void dft3(double &a, double &b, double &c, double w, double q, double qi) {
    // y0 = a + b + c, y1 = (a - c) + w (b - c), y2 = (a - b) - w (b - c)   (1 + w + w^2 = 0)
    const double t = fmm8(__dsub_rn(b, c), w, q, qi);
    const double y0 = __dadd_rn(__dadd_rn(a, b), c);
    const double y1 = __dadd_rn(__dsub_rn(a, c), t);
    const double y2 = __dsub_rn(__dsub_rn(a, b), t);
    a = y0; b = y1; c = y2;
}
template <int RAD>
__device__ __forceinline__ void dft_small(double (&x)[RAD], const double *__restrict__ w, double q, double qi) {
    static_assert(RAD == 3 || RAD == 9, "radix");
    if (RAD == 3) {
        dft3(x[0], x[1], x[2], w[1], q, qi);
    } else {
        // 9 = 3 x 3: A[n2][k1] = DFT3_n1(x[3 n1 + n2]); B = A * w9^{n2 k1}; X[k1 + 3 k2] = DFT3_n2(B[n2][k1])
        const double w3 = w[3];
        double a[3][3];
#pragma unroll
        for (int n2 = 0; n2 < 3; ++n2) {
            a[n2][0] = x[n2]; a[n2][1] = x[3 + n2]; a[n2][2] = x[6 + n2];
            dft3(a[n2][0], a[n2][1], a[n2][2], w3, q, qi);
        }
#pragma unroll
        for (int n2 = 0; n2 < 3; ++n2)
#pragma unroll
            for (int k1 = 0; k1 < 3; ++k1)
                a[n2][k1] = (n2 && k1) ? fmm8(a[n2][k1], w[n2 * k1], q, qi) : fred(a[n2][k1], q, qi);
#pragma unroll
        for (int k1 = 0; k1 < 3; ++k1) {
            double b0 = a[0][k1], b1 = a[1][k1], b2 = a[2][k1];
            dft3(b0, b1, b2, w3, q, qi);
            x[k1] = b0; x[k1 + 3] = b1; x[k1 + 6] = b2;
        }
    }
}

// pass B, mixed-radix rows: RB rows per block, each split into RAD sub-rows of N' = 2^LOGN (TPS = N'/E threads
// each).  Radix stage and the sub-row transforms exchange through one shared buffer of RB*RAD padded sub-rows.
template <int LOGN, int LOGE, int RB, int INV, int RAD>
__global__ void __launch_bounds__(RB * RAD * (1 << (LOGN - LOGE)))
    kf_passB_mr(NttTables T, LimbMap lm, uint64_t job0, double *__restrict__ scratch) {
    constexpr int E = 1 << LOGE, NN = 1 << LOGN, TPS = NN / E, C = RAD * NN;
    constexpr int ROWW = NN + NN / E;
    extern __shared__ double smf[];
    const uint32_t job = (uint32_t)(job0 + blockIdx.y);
    const JobF J = job_f(lm, job);
    const double q = T.fmods[J.pr].x, qi = T.fmods[J.pr].y;
    const uint32_t sr = threadIdx.x / TPS, tau = threadIdx.x % TPS;   // sub-row sr = rr RAD + i of this block
    const uint32_t rr = sr / RAD, i = sr % RAD, row = blockIdx.x * RB + rr;
    double *buf = smf;
    double *rtw = buf + RB * RAD * ROWW, *rtwi = rtw + C, *rc = rtwi + C, *rci = rc + 16;
    typedef PtTab<LOGN, LOGE, true> PTF;
    typedef PtTab<LOGN, LOGE, false> PTI;
    double2 *tw = (double2 *)(rci + 16), *twi = tw + NN / 2, *ptf = twi + NN / 2, *pti = ptf + PTF::WORDS;
    const double2 *gtw = T.ftwCb + (uint64_t)J.pr * (NN / 2), *gtwi = T.ftwCi + (uint64_t)J.pr * (NN / 2);
    for (int j = threadIdx.x; j < NN / 2; j += blockDim.x) {
        tw[j] = gtw[j];
        twi[j] = gtwi[j];
    }
    for (int j = threadIdx.x; j < C; j += blockDim.x) {
        rtw[j] = T.frtw[(uint64_t)J.pr * C + j];
        rtwi[j] = T.frtwi[(uint64_t)J.pr * C + j];
    }
    if (threadIdx.x < 16) {
        rc[threadIdx.x] = T.frcon[(uint64_t)J.pr * 16 + threadIdx.x];
        rci[threadIdx.x] = T.frconi[(uint64_t)J.pr * 16 + threadIdx.x];
    }
    if (sr == 0) PTF::fill(ptf, tau, gtw);
    if (sr == 1 % (RB * RAD)) PTI::fill(pti, tau, gtwi);
    __syncthreads();
    double *grow0 = scratch + (uint64_t)blockIdx.y * T.M + (uint64_t)blockIdx.x * RB * C;
    // forward radix stage: (row, j) -> u_i[j] into sub-row buffers (natural order, padded)
    for (int idx = threadIdx.x; idx < RB * NN; idx += blockDim.x) {
        const int r2 = idx / NN, j = idx % NN;
        const double *g = grow0 + (uint64_t)r2 * C;
        double x[RAD];
#pragma unroll
        for (int l = 0; l < RAD; ++l) x[l] = __ldcs(g + j + l * NN);   // |x| <= q (pass A output)
        dft_small<RAD>(x, rc, q, qi);
#pragma unroll
        for (int l = 0; l < RAD; ++l) buf[(r2 * RAD + l) * ROWW + j + (j >> LOGE)] = fmm8(x[l], rtw[l * NN + j], q, qi);
    }
    __syncthreads();
    double *srow = buf + sr * ROWW;
    double v[E];
    int bd[E];
#pragma unroll
    for (int k = 0; k < E; ++k) {
        const uint32_t e = held_index<LOGE>(tau, LOGN - LOGE, k);
        v[k] = srow[e + (e >> LOGE)];
        bd[k] = UMUL8;
    }
    __syncthreads();
    frt_pass<LOGN, LOGE, true, 0>(v, bd, tau, srow, tw, ptf, q, qi);
    // D^ in the sub-row thread-minor layout: position tau E + k of sub-row i at row C + i N' + k TPS + tau
    const double *dh = (INV == 0 ? T.fdhf : T.fdhi) + (uint64_t)J.pr * T.M + (uint64_t)row * C + i * NN + tau;
#pragma unroll
    for (int k = 0; k < E; ++k) {
        need(v, bd, k, LIM_MUL, q, qi);
        v[k] = fmm8(v[k], dh[k * TPS], q, qi);
        bd[k] = UMUL8;
    }
    frt_pass<LOGN, LOGE, false, 0>(v, bd, tau, srow, twi, pti, q, qi);
#pragma unroll
    for (int k = 0; k < E; ++k) {               // natural positions j; undo the radix twiddle
        const uint32_t j = held_index<LOGE>(tau, LOGN - LOGE, k);
        need(v, bd, k, LIM_MUL, q, qi);
        srow[j + (j >> LOGE)] = fmm8(v[k], rtwi[i * NN + j], q, qi);
    }
    __syncthreads();
    // inverse radix stage, cross twiddle psi^(-c brev(r)), back to the scratch row
    for (int idx = threadIdx.x; idx < RB * NN; idx += blockDim.x) {
        const int r2 = idx / NN, j = idx % NN;
        double x[RAD];
#pragma unroll
        for (int l = 0; l < RAD; ++l) x[l] = buf[(r2 * RAD + l) * ROWW + j + (j >> LOGE)];
        dft_small<RAD>(x, rci, q, qi);
        double *g = grow0 + (uint64_t)r2 * C;
        const double *xt = T.fxtb + (uint64_t)J.pr * T.M + (uint64_t)(blockIdx.x * RB + r2) * C;
#pragma unroll
        for (int l = 0; l < RAD; ++l) __stcs(g + j + l * NN, fmm8(x[l], xt[j + l * NN], q, qi));
    }
}

template <int LOGN, int LOGE, int RB, int RAD>
struct ShapeMR {
    static constexpr int NN = 1 << LOGN, C = RAD * NN, THREADS = RB * RAD * (NN >> LOGE);
    static constexpr size_t SMEM = (size_t)RB * RAD * (NN + NN / (1 << LOGE)) * 8 + (size_t)(2 * C + 32) * 8 +
                                   (size_t)(NN + PtTab<LOGN, LOGE, true>::WORDS + PtTab<LOGN, LOGE, false>::WORDS) * 16;
};

// pass C: column inverse (length R) -> natural t, output chirp, canonical u64: Z_m^* gather (fwd) or A_t (inv)
template <int LOGR, int LOGE, int TC, int INV, int LOGC>
__global__ void __launch_bounds__(TC * (1 << (LOGR - LOGE)), FNTT_MINB(TC * (1 << (LOGR - LOGE))))
    kf_passC(NttTables T, uint64_t *__restrict__ out, uint64_t out_pstride, LimbMap lm, uint64_t job0,
             double *__restrict__ scratch, uint64_t *__restrict__ aux) {
    constexpr int E = 1 << LOGE, R = 1 << LOGR;
    constexpr uint32_t CC = 1u << LOGC;
    extern __shared__ double smf[];
    const uint32_t job = (uint32_t)(job0 + blockIdx.y);
    const JobF J = job_f(lm, job);
    const double q = T.fmods[J.pr].x, qi = T.fmods[J.pr].y;
    const uint32_t col = threadIdx.x % TC, tau = threadIdx.x / TC;
    const uint32_t c = blockIdx.x * TC + col;
    double *scr = scratch + (uint64_t)blockIdx.y * T.M;
    typedef PtTab<LOGR, LOGE, false> PTT;
    double2 *stw = (double2 *)(smf + (size_t)R * TC), *spt = stw + R / 2;
    const double2 *gtw = T.ftwRi + (uint64_t)J.pr * (R / 2);
    for (int j = threadIdx.x; j < R / 2; j += blockDim.x) stw[j] = gtw[j];
    if (col == 0) PTT::fill(spt, tau, gtw);
    double v[E];
    int bd[E];
#pragma unroll
    for (int k = 0; k < E; ++k) {
        v[k] = __ldcs(scr + held_index<LOGE>(tau, 0, k) * CC + c);
        bd[k] = UMUL8;
    }
    __syncthreads();
    fct_pass<LOGR, LOGE, false, TC, 0>(v, bd, tau, col, smf, stw, spt, q, qi);
    const double *tfo = (INV == 1 ? T.ftfoi : T.ftfo) + (uint64_t)J.pr * T.m;
    uint64_t *dst = out + (uint64_t)J.poly * out_pstride + (uint64_t)J.lb * T.n;
    uint64_t *scru = (uint64_t *)scr;
    uint64_t *A1 = INV >= 2 ? aux + (uint64_t)blockIdx.y * T.Mslot : nullptr;    // the A_t of this job (Barrett)
    const uint32_t kq = T.m - T.n;
    // prime m (aux = per-job A_{m-1} from kf_corner): out_t = A_t - A_{m-1} written directly (t < n);
    // composite m: A_t into the scratch slot in place (read by the Barrett passes)
    const bool direct = INV == 1 && T.prime_m && aux != nullptr;
    const uint64_t corner = direct ? aux[blockIdx.y] : 0;
    if (INV == 1 && !direct) __syncthreads();   // all columns of this block read before in-place writes of A_t
#pragma unroll
    for (int k = 0; k < E; ++k) {
        if (INV <= 2 && k >= E / 2) continue;   // rows >= R/2: t >= M/2 >= m (mode 2: >= k), never output (the last
                                                // stage's differences feeding them are dead code)
        const uint32_t r = held_index<LOGE>(tau, LOGR - LOGE, k);
        const uint32_t t = r * CC + c;
        if (t >= T.m) continue;
        need(v, bd, k, LIM_MUL, q, qi);
        if (INV == 2) {               // Qr_t (t < m - n) -> Q_{m-n-1-t}, stored over A_{n..m-1}
            if (t < kq) A1[T.n + (kq - 1 - t)] = to_u64(fred(v[k], q, qi), q);
            continue;
        }
        if (INV == 3) {               // a_t = A_t - (Phi_m Q)_t, t < n
            if (t < T.n) {
                const double a = from_u64(A1[t]);
                __stcs(dst + t, to_u64(fred(__dsub_rn(a, fred(v[k], q, qi)), q, qi), q));
            }
            continue;
        }
        const uint64_t x = to_u64((T.dbg & 16) ? fred(v[k], q, qi) : fmm8(v[k], tfo[t], q, qi), q);
        if (!INV) {
            const int ps = (T.dbg & 32) ? (t < T.n ? (int)t : -1) : T.pos[t];
            if (ps >= 0) __stcs(dst + ps, T.epi.mode ? epi_apply(T.epi, J.poly, J.lb, T.n, (uint32_t)ps, x) : x);
        } else if (direct) {
            if (t < T.n) __stcs(dst + t, x >= corner ? x - corner : x + (uint64_t)q - corner);
        } else {
            scru[t] = x;
        }
    }
}

// prime m, inverse: A_{m-1} of every job of the group, from the pass-B output column c* = (m-1) mod C:
// A_{m-1} = tfoi[m-1] * sum_rp x[rp C + c*] omega_R^{-r* brev(rp)}, r* = (m-1) / C (the value pass C computes
// at t = m-1), so that pass C can write the reduction A_t - A_{m-1} (mod Phi_m, m prime) directly
template <int LOGR>
__global__ void __launch_bounds__(32) kf_corner(NttTables T, LimbMap lm, uint64_t job0, const double *__restrict__ scratch,
                                                 uint64_t *__restrict__ corner) {
    constexpr int R = 1 << LOGR;
    const JobF J = job_f(lm, (uint32_t)(job0 + blockIdx.x));
    const double q = T.fmods[J.pr].x, qi = T.fmods[J.pr].y;
    const double *scr = scratch + (uint64_t)blockIdx.x * T.M;
    const uint32_t cs = (T.m - 1) % T.C, rs = (T.m - 1) / T.C;
    const double2 *tw = T.ftwRi + (uint64_t)J.pr * (R / 2);
    double acc = 0.0;                                   // <= (R/32) 0.625 q per lane
    for (uint32_t rp = threadIdx.x; rp < (uint32_t)R; rp += 32) {
        const uint32_t e = (rs * (__brev(rp) >> (32 - LOGR))) & (R - 1);
        double2 w = tw[e & (R / 2 - 1)];
        if (e >= (uint32_t)(R / 2)) { w.x = -w.x; w.y = -w.y; }      // omega_R^{-R/2} = -1
        acc = __dadd_rn(acc, fmm(scr[(uint64_t)rp * T.C + cs], w, q));
    }
    acc = fred(acc, q, qi);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = fred(__dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o)), q, qi);
    if (threadIdx.x == 0) {
        const double *tfo = T.ftfoi + (uint64_t)J.pr * T.m;
        corner[blockIdx.x] = to_u64(fmm8(acc, tfo[T.m - 1], q, qi), q);
    }
}

// persistent column passes: attributes and occupancy per device (once), CTAs per column group = resident CTAs
// per SM x 148 / column groups (capped by bc_tune "ntt_persist_occ")
template <int LOGR, int LOGER, int TC, int CCV, int LEAN, int MINB>
static void launch_pA(int inv, const NttTables &T, const uint64_t *in, uint64_t in_ps, LimbMap lm, uint64_t j0, uint32_t nj,
                      double *scr, cudaStream_t st) {
    typedef PersistA<LOGR, LOGER, TC, CCV, LEAN> PA;
    constexpr int TH = TC << (LOGR - LOGER);
    static std::atomic<uint64_t> init_dev{0};
    static int nb[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (attr_pending(init_dev)) {
        cudaFuncSetAttribute(kf_passA_p<LOGR, LOGER, TC, CCV, 0, LEAN, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PA::SMEM);
        cudaFuncSetAttribute(kf_passA_p<LOGR, LOGER, TC, CCV, 1, LEAN, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PA::SMEM);
        int b = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kf_passA_p<LOGR, LOGER, TC, CCV, 0, LEAN, MINB>, TH, PA::SMEM);
        nb[dev & 63] = b > 0 ? b : 1;
        attr_done(init_dev);
    }
    const uint32_t ncg = CCV / TC;
    const int occ = g_ntt_persist_occ > 0 ? std::min(g_ntt_persist_occ, nb[dev & 63]) : nb[dev & 63];
    const uint32_t G = std::max<uint32_t>(1, std::min<uint32_t>(nj, (uint32_t)(occ * 148) / ncg));
    if (inv) kf_passA_p<LOGR, LOGER, TC, CCV, 1, LEAN, MINB><<<dim3(ncg, G), TH, PA::SMEM, st>>>(T, in, in_ps, lm, j0, nj, scr);
    else kf_passA_p<LOGR, LOGER, TC, CCV, 0, LEAN, MINB><<<dim3(ncg, G), TH, PA::SMEM, st>>>(T, in, in_ps, lm, j0, nj, scr);
}
template <int LOGR, int LOGER, int TC, int CCV, int LEAN, int MINB>
static void launch_pC(int inv, const NttTables &T, uint64_t *out, uint64_t out_ps, LimbMap lm, uint64_t j0, uint32_t nj,
                      const double *scr, const uint64_t *corner, cudaStream_t st) {
    typedef PersistC<LOGR, LOGER, TC, CCV, LEAN> PC;
    constexpr int TH = TC << (LOGR - LOGER);
    static std::atomic<uint64_t> init_dev{0};
    static int nb[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (attr_pending(init_dev)) {
        cudaFuncSetAttribute(kf_passC_p<LOGR, LOGER, TC, CCV, 0, LEAN, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PC::SMEM);
        cudaFuncSetAttribute(kf_passC_p<LOGR, LOGER, TC, CCV, 1, LEAN, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PC::SMEM);
        int b = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kf_passC_p<LOGR, LOGER, TC, CCV, 0, LEAN, MINB>, TH, PC::SMEM);
        nb[dev & 63] = b > 0 ? b : 1;
        attr_done(init_dev);
    }
    const uint32_t ncg = CCV / TC;
    const int occ = g_ntt_persist_occ > 0 ? std::min(g_ntt_persist_occ, nb[dev & 63]) : nb[dev & 63];
    const uint32_t G = std::max<uint32_t>(1, std::min<uint32_t>(nj, (uint32_t)(occ * 148) / ncg));
    if (inv) kf_passC_p<LOGR, LOGER, TC, CCV, 1, LEAN, MINB><<<dim3(ncg, G), TH, PC::SMEM, st>>>(T, out, out_ps, lm, j0, nj, scr, corner);
    else kf_passC_p<LOGR, LOGER, TC, CCV, 0, LEAN, MINB><<<dim3(ncg, G), TH, PC::SMEM, st>>>(T, out, out_ps, lm, j0, nj, scr, nullptr);
}
// g_ntt_lean (measured, C2 / C4 / C5 limb-transforms): 4 (default, 1-2% faster than 0) -> round-2 A + C with
// shared-memory tiles and the staging tile as exchange buffer (3 per SM); 0 -> shared-memory table tiles
// (2 CTAs per SM); 1 -> lean A (4 per SM) + lean C (3 per SM);
// 2 -> lean A + C with the staging tile as exchange buffer (4 per SM); 3 -> round-2 A + that C
template <int LOGR, int LOGER, int TC, int CCV>
static void persist_A(int inv, const NttTables &T, const uint64_t *in, uint64_t in_ps, LimbMap lm, uint64_t j0, uint32_t nj,
                      double *scr, cudaStream_t st) {
    if (g_ntt_lean == 0 || g_ntt_lean >= 3) launch_pA<LOGR, LOGER, TC, CCV, 0, 2>(inv, T, in, in_ps, lm, j0, nj, scr, st);
    else launch_pA<LOGR, LOGER, TC, CCV, 1, 4>(inv, T, in, in_ps, lm, j0, nj, scr, st);
}
template <int LOGR, int LOGER, int TC, int CCV>
static void persist_C(int inv, const NttTables &T, uint64_t *out, uint64_t out_ps, LimbMap lm, uint64_t j0, uint32_t nj,
                      const double *scr, const uint64_t *corner, cudaStream_t st) {
    if (g_ntt_lean == 1) launch_pC<LOGR, LOGER, TC, CCV, 1, 3>(inv, T, out, out_ps, lm, j0, nj, scr, corner, st);
    else if (g_ntt_lean == 2 || g_ntt_lean == 3) launch_pC<LOGR, LOGER, TC, CCV, 2, 4>(inv, T, out, out_ps, lm, j0, nj, scr, corner, st);
    else if (g_ntt_lean == 4) launch_pC<LOGR, LOGER, TC, CCV, 4, 3>(inv, T, out, out_ps, lm, j0, nj, scr, corner, st);
    else launch_pC<LOGR, LOGER, TC, CCV, 0, 2>(inv, T, out, out_ps, lm, j0, nj, scr, corner, st);
}

// mixed-radix transform (prime m): persistent passes A / C with C = RAD 2^LOGN columns, mixed row pass B
template <int RAD, int LOGN, int LOGEB, int RB>
static void runf_mr(const NttTables &T0, const uint64_t *in, uint64_t *out, LimbMap lm, uint64_t in_ps, uint64_t out_ps,
                    uint64_t *scratch, uint64_t j0, uint32_t nj, int inv, cudaStream_t st, uint64_t *corner_buf) {
    constexpr int LOGR = 8, LOGER = 4, TC = 16, CCV = RAD << LOGN;
    typedef ShapeMR<LOGN, LOGEB, RB, RAD> SB;
    static std::atomic<uint64_t> init_dev{0};
    if (attr_pending(init_dev)) {
        cudaFuncSetAttribute(kf_passB_mr<LOGN, LOGEB, RB, 0, RAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SB::SMEM);
        cudaFuncSetAttribute(kf_passB_mr<LOGN, LOGEB, RB, 1, RAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SB::SMEM);
        attr_done(init_dev);
    }
    NttTables T = T0;
    T.dbg = 0;
    double *scr = (double *)scratch;
    dim3 gB((1 << LOGR) / RB, nj);
    persist_A<LOGR, LOGER, TC, CCV>(inv, T, in, in_ps, lm, j0, nj, scr, st);
    if (!inv) {
        kf_passB_mr<LOGN, LOGEB, RB, 0, RAD><<<gB, SB::THREADS, SB::SMEM, st>>>(T, lm, j0, scr);
    } else {
        kf_passB_mr<LOGN, LOGEB, RB, 1, RAD><<<gB, SB::THREADS, SB::SMEM, st>>>(T, lm, j0, scr);
        kf_corner<LOGR><<<nj, 32, 0, st>>>(T, lm, j0, scr, corner_buf);
        launch_counter() += 1;
    }
    persist_C<LOGR, LOGER, TC, CCV>(inv, T, out, out_ps, lm, j0, nj, scr, inv ? corner_buf : nullptr, st);
    launch_counter() += 3;
}

template <int LOGR, int LOGER, int LOGC, int LOGEC, int TC_, int RB_>
struct Shape {
    static constexpr int TC = TC_, RB = RB_ ? RB_ : ((LOGC - LOGEC) >= 6 ? 4 : ((LOGC - LOGEC) >= 4 ? 8 : 16));
    static constexpr int THA = TC << (LOGR - LOGER), THB = RB << (LOGC - LOGEC);
    static constexpr size_t SMA = (size_t)(1 << LOGR) * TC * 8 + (size_t)(1 << LOGR) / 2 * 16 +
                                  (size_t)(PtTab<LOGR, LOGER, true>::WORDS > PtTab<LOGR, LOGER, false>::WORDS
                                               ? PtTab<LOGR, LOGER, true>::WORDS : PtTab<LOGR, LOGER, false>::WORDS) * 16;
    static constexpr size_t SMB = (size_t)RB * ((1 << LOGC) + (1 << (LOGC - LOGEC))) * 8 + (size_t)(1 << LOGC) * 16 +
                                  (size_t)(PtTab<LOGC, LOGEC, true>::WORDS + PtTab<LOGC, LOGEC, false>::WORDS) * 16;
};

template <int LOGR, int LOGER, int LOGC, int LOGEC, int TC_ = 8, int RB_ = 0>
static void runf(const NttTables &T0, const uint64_t *in, uint64_t *out, LimbMap lm, uint64_t in_ps, uint64_t out_ps,
                 uint64_t *scratch, uint64_t j0, uint32_t nj, int inv, cudaStream_t st, uint64_t *corner_buf,
                 bool persist = false) {
    typedef Shape<LOGR, LOGER, LOGC, LOGEC, TC_, RB_> S;
    static std::atomic<uint64_t> init_dev{0};
    if (attr_pending(init_dev)) {
        cudaFuncSetAttribute(kf_passA<LOGR, LOGER, S::TC, 0, LOGC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMA);
        cudaFuncSetAttribute(kf_passA<LOGR, LOGER, S::TC, 1, LOGC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMA);
        cudaFuncSetAttribute(kf_passC<LOGR, LOGER, S::TC, 0, LOGC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMA);
        cudaFuncSetAttribute(kf_passC<LOGR, LOGER, S::TC, 1, LOGC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMA);
        cudaFuncSetAttribute(kf_passB<LOGC, LOGEC, S::RB, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMB);
        cudaFuncSetAttribute(kf_passB<LOGC, LOGEC, S::RB, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMB);
        attr_done(init_dev);
    }
    double *scr = (double *)scratch;
    NttTables T = T0;
    T.dbg = g_ntt_dbg;
    dim3 gA((1 << LOGC) / S::TC, nj), gB((1 << LOGR) / S::RB, nj);
    // persistent passes A and C (tiles of the prime resident in shared memory, cp.async prefetch of the next job)
    if constexpr (LOGR == 8) {
        if (persist && !T.dbg && (!inv || (T.prime_m && corner_buf))) {
            constexpr int CCV = 1 << LOGC;
        persist_A<LOGR, LOGER, S::TC, CCV>(inv, T, in, in_ps, lm, j0, nj, scr, st);
        if (!inv) {
            kf_passB<LOGC, LOGEC, S::RB, 0><<<gB, S::THB, S::SMB, st>>>(T, lm, j0, scr);
        } else {
            kf_passB<LOGC, LOGEC, S::RB, 1><<<gB, S::THB, S::SMB, st>>>(T, lm, j0, scr);
            kf_corner<LOGR><<<nj, 32, 0, st>>>(T, lm, j0, scr, corner_buf);
            launch_counter() += 1;
        }
        persist_C<LOGR, LOGER, S::TC, CCV>(inv, T, out, out_ps, lm, j0, nj, scr, inv ? corner_buf : nullptr, st);
            launch_counter() += 3;
            return;
        }
    }
    if (!inv) {
        kf_passA<LOGR, LOGER, S::TC, 0, LOGC><<<gA, S::THA, S::SMA, st>>>(T, in, in_ps, lm, j0, scr);
        kf_passB<LOGC, LOGEC, S::RB, 0><<<gB, S::THB, S::SMB, st>>>(T, lm, j0, scr);
        kf_passC<LOGR, LOGER, S::TC, 0, LOGC><<<gA, S::THA, S::SMA, st>>>(T, out, out_ps, lm, j0, scr, nullptr);
    } else {
        bool pa = false;
        if constexpr (LOGR == 8) {      // composite m: the persistent pass A (identical scratch), pass C below
            if (persist && !T.dbg && g_ntt_lean != 0) {   // (ntt_lean 0: the round-2 passes)
                persist_A<LOGR, LOGER, S::TC, (1 << LOGC)>(1, T, in, in_ps, lm, j0, nj, scr, st);
                pa = true;
            }
        }
        if (!pa) kf_passA<LOGR, LOGER, S::TC, 1, LOGC><<<gA, S::THA, S::SMA, st>>>(T, in, in_ps, lm, j0, scr);
        kf_passB<LOGC, LOGEC, S::RB, 1><<<gB, S::THB, S::SMB, st>>>(T, lm, j0, scr);
        uint64_t *corner = nullptr;
        if (T.prime_m && corner_buf) {
            corner = corner_buf;
            kf_corner<LOGR><<<nj, 32, 0, st>>>(T, lm, j0, scr, corner);
            launch_counter() += 1;
        }
        kf_passC<LOGR, LOGER, S::TC, 1, LOGC><<<gA, S::THA, S::SMA, st>>>(T, out, out_ps, lm, j0, scr, corner);
    }
    launch_counter() += 3;
}

// sparse quotient: Qr_i = sum_j ir_val_j Fr_{i - ir_off_j}, Fr_i = A_{m-1-i}; Q_{k-1-i} = Qr_i -> scr2 slot (stride B.M)
__global__ void k_ir_sparse(NttTables T, LimbMap lm, uint64_t job0, const uint64_t *__restrict__ scr1,
                            uint64_t *__restrict__ scr2) {
    const uint32_t k = T.m - T.n, i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= k) return;
    const JobF J = job_f(lm, (uint32_t)(job0 + blockIdx.y));
    const Mod Md = T.mods[J.pr];
    const uint64_t q = Md.q;
    const uint64_t *A = scr1 + (uint64_t)blockIdx.y * T.Mslot;
    uint64_t acc = 0;
    for (int j = 0; j < T.ir_nnz; ++j) {
        const int32_t o = T.ir_off[j], v = T.ir_val[j];
        if ((int32_t)i < o) continue;
        const uint64_t f = A[T.m - 1 - (i - o)];
        if (v == 1) acc = add_mod(acc, f, q);
        else if (v == -1) acc = sub_mod(acc, f, q);
        else acc = add_mod(acc, mul_mod(f, from_signed(v, q), Md), q);
    }
    scr2[(uint64_t)blockIdx.y * T.M + (k - 1 - i)] = acc;
}

// composite m: Barrett division mod Phi_m of the A_t in the scr1 slots (two convolutions with table set B)
template <int LOGR, int LOGER, int LOGC, int LOGEC, int TC_ = 8, int RB_ = 0>
static void runb(const NttTables &B, uint64_t *out, LimbMap lm, uint64_t out_ps, uint64_t *scr1, uint64_t *scr2,
                 uint64_t j0, uint32_t nj, cudaStream_t st) {
    typedef Shape<LOGR, LOGER, LOGC, LOGEC, TC_, RB_> S;
    static std::atomic<uint64_t> init_dev{0};
    if (attr_pending(init_dev)) {
        cudaFuncSetAttribute(kf_passA<LOGR, LOGER, S::TC, 2, LOGC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMA);
        cudaFuncSetAttribute(kf_passA<LOGR, LOGER, S::TC, 3, LOGC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMA);
        cudaFuncSetAttribute(kf_passC<LOGR, LOGER, S::TC, 2, LOGC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMA);
        cudaFuncSetAttribute(kf_passC<LOGR, LOGER, S::TC, 3, LOGC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMA);
        cudaFuncSetAttribute(kf_passB<LOGC, LOGEC, S::RB, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMB);
        cudaFuncSetAttribute(kf_passB<LOGC, LOGEC, S::RB, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMB);
        attr_done(init_dev);
    }
    NttTables T = B;
    T.dbg = 0;
    double *s2 = (double *)scr2;
    dim3 gA((1 << LOGC) / S::TC, nj), gB((1 << LOGR) / S::RB, nj);
    if (T.ir_nnz > 0 && !g_phi_conv) {
        // Phi_m^{-1} mod x^k is sparse (m = r1 r2 with a small factor: (1 + ... + x^{r1-1})(1 - x^{r2})):
        // the quotient is a short sum of shifted copies, written as Q into the scr2 slots
        const uint32_t k = T.m - T.n;
        k_ir_sparse<<<dim3((k + 255) / 256, nj), 256, 0, st>>>(T, lm, j0, scr1, scr2);
        T.q_in_s2 = 1;
        kf_passA<LOGR, LOGER, S::TC, 3, LOGC><<<gA, S::THA, S::SMA, st>>>(T, scr2, 0, lm, j0, s2);
        kf_passB<LOGC, LOGEC, S::RB, 3><<<gB, S::THB, S::SMB, st>>>(T, lm, j0, s2);
        kf_passC<LOGR, LOGER, S::TC, 3, LOGC><<<gA, S::THA, S::SMA, st>>>(T, out, out_ps, lm, j0, s2, scr1);
        launch_counter() += 4;
        return;
    }
    T.q_in_s2 = 0;
    kf_passA<LOGR, LOGER, S::TC, 2, LOGC><<<gA, S::THA, S::SMA, st>>>(T, scr1, 0, lm, j0, s2);
    kf_passB<LOGC, LOGEC, S::RB, 2><<<gB, S::THB, S::SMB, st>>>(T, lm, j0, s2);
    kf_passC<LOGR, LOGER, S::TC, 2, LOGC><<<gA, S::THA, S::SMA, st>>>(T, out, out_ps, lm, j0, s2, scr1);
    kf_passA<LOGR, LOGER, S::TC, 3, LOGC><<<gA, S::THA, S::SMA, st>>>(T, scr1, 0, lm, j0, s2);
    kf_passB<LOGC, LOGEC, S::RB, 3><<<gB, S::THB, S::SMB, st>>>(T, lm, j0, s2);
    kf_passC<LOGR, LOGER, S::TC, 3, LOGC><<<gA, S::THA, S::SMA, st>>>(T, out, out_ps, lm, j0, s2, scr1);
    launch_counter() += 6;
}

}  // namespace f64

// register count E = 2^LOGE of the pass-B row transform of each shape (the D^ table layout depends on it)
int nttf_row_loge(uint32_t logR, uint32_t logC) {
    switch (logR * 16 + logC) {
        case 8 * 16 + 9: return NTTF_LOGE_89;
        case 6 * 16 + 6: case 5 * 16 + 6: return 3;
        default: return 4;
    }
}

int nttf_mr_loge(uint32_t rad, uint32_t logN) { return (rad == 9 && logN == 5) ? 3 : 4; }   // runf_mr shapes

bool nttf_supported(const NttTables &T) {
    if (T.rad > 1) return T.fmods != nullptr && T.prime_m && T.logR == 8 &&
                          ((T.rad == 9 && T.logN == 5) || (T.rad == 3 && T.logN == 7));
    return T.fmods != nullptr && ntt2_supported(T);
}

void nttf_run(const NttTables &T, const uint64_t *in, uint64_t *out, LimbMap lm, uint64_t in_ps, uint64_t out_ps,
              uint64_t *scratch, uint64_t j0, uint32_t nj, int inv, cudaStream_t st, uint64_t *corner_buf) {
    if (T.rad > 1) {        // R25 mixed-radix lengths (prime m): C4 9 x 32, C5 3 x 128 row shapes
        if (T.rad == 9 && T.logN == 5) f64::runf_mr<9, 5, 3, 4>(T, in, out, lm, in_ps, out_ps, scratch, j0, nj, inv, st, corner_buf);
        else if (T.rad == 3 && T.logN == 7) f64::runf_mr<3, 7, 4, 4>(T, in, out, lm, in_ps, out_ps, scratch, j0, nj, inv, st, corner_buf);
        return;
    }
#define RUNF(...) f64::runf<__VA_ARGS__>(T, in, out, lm, in_ps, out_ps, scratch, j0, nj, inv, st, corner_buf)
#define RUNP(...) f64::runf<__VA_ARGS__>(T, in, out, lm, in_ps, out_ps, scratch, j0, nj, inv, st, corner_buf, true)
    switch (T.logR * 16 + T.logC) {
        case 8 * 16 + 8:
            switch (g_ntt_impl) {
                case 11: RUNF(8, 4, 8, 4, 4); break;
                case 12: RUNF(8, 4, 8, 4, 8); break;
                case 14: RUNF(8, 4, 8, 4, 16, 4); break;
                case 15: RUNF(8, 4, 8, 4, 32); break;
                case 16: RUNF(8, 4, 8, 4, 16); break;
                case 17: RUNF(8, 4, 8, 4, 16, 16); break;     // non-persistent A / C (round-1 default)
                default: RUNP(8, 4, 8, 4, 16, 16); break;      // persistent A / C: 0.865 us per C2 limb-transform
                                                               // (0.923 with the non-persistent passes)
            }
            break;
        case 8 * 16 + 9:
            if (g_ntt_impl == 12) RUNF(8, 4, 9, NTTF_LOGE_89, 8);
            else if (g_ntt_impl == 13) RUNF(8, 4, 9, NTTF_LOGE_89, 16, 8);
            else if (g_ntt_impl == 17) RUNF(8, 4, 9, NTTF_LOGE_89, 16);
            else RUNP(8, 4, 9, NTTF_LOGE_89, 16);
            break;
        case 7 * 16 + 8: RUNF(7, 4, 8, 4, 16); break;
        case 7 * 16 + 7: RUNF(7, 4, 7, 4, 16); break;
        case 6 * 16 + 7: RUNF(6, 3, 7, 4, 16); break;
        case 6 * 16 + 6: RUNF(6, 3, 6, 3, 16); break;
        case 5 * 16 + 6: RUNF(5, 4, 6, 3, 16); break;
        default: break;
    }
#undef RUNF
#undef RUNP
}

}  // namespace bc

namespace bc {
void nttf_barrett(const NttTables &B, uint64_t *out, LimbMap lm, uint64_t out_ps, uint64_t *scr1, uint64_t *scr2,
                  uint64_t j0, uint32_t nj, cudaStream_t st) {
#define RUNB(...) f64::runb<__VA_ARGS__>(B, out, lm, out_ps, scr1, scr2, j0, nj, st)
    switch (B.logR * 16 + B.logC) {
        case 8 * 16 + 8: RUNB(8, 4, 8, 4, 16, 16); break;
        case 8 * 16 + 9: RUNB(8, 4, 9, NTTF_LOGE_89, 16); break;
        case 7 * 16 + 8: RUNB(7, 4, 8, 4, 16); break;
        case 7 * 16 + 7: RUNB(7, 4, 7, 4, 16); break;
        case 6 * 16 + 7: RUNB(6, 3, 7, 4, 16); break;
        case 6 * 16 + 6: RUNB(6, 3, 6, 3, 16); break;
        case 5 * 16 + 6: RUNB(5, 4, 6, 3, 16); break;
        default: break;
    }
#undef RUNB
}
}  // namespace bc
