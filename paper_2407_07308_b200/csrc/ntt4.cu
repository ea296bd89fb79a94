// ntt4.cu -- the Bluestein transform of one limb in ONE kernel: a thread-block cluster holds the whole
// size-M convolution in its distributed shared memory (a1/a2, Listings 1-2 at P:445-464).
//
// The three-pass form (ntt3.cu) moves every limb-transform through HBM/L2 twice between its passes
// (pass A -> scratch -> pass B -> scratch -> pass C: 4 x 8M bytes of scratch traffic against 16n bytes of
// input and output).  Here the CL CTAs of a cluster split the M = R x C grid instead:
//   phase A  CTA k: columns [k TC, (k+1) TC) -- input chirp, column forward transform (length R), cross
//            twiddle psi^(c brev(rp)); the tile stays in its own shared memory, [rp][c - k TC];
//   phase B  CTA k: rows [k RB, (k+1) RB) read from the CL tiles over DSMEM (ld.shared::cluster) -- row
//            forward transform, x D^, row inverse transform, cross twiddle psi^(-c brev(r)); tile [r][c];
//   phase C  CTA k: columns again, read over DSMEM -- column inverse transform, output chirp, Z_m^* gather
//            (forward) or the reduction mod Phi_m (inverse, prime m: A_t - A_{m-1}, with A_{m-1} broadcast
//            over DSMEM by the CTA that computes it).
// The arithmetic (binary64 bound-tracked butterflies, tables, orders) is exactly that of ntt3.cu, so the
// results are bit-identical (every kernel boundary is canonical u64).  HBM traffic per limb-transform is
// the 16n bytes of input and output plus the per-prime tables (L2-resident: jobs are limb-major and a
// persistent cluster keeps its prime's twiddles in shared memory).  Clusters are persistent (one per
// co-resident slot, jobs strided), and each CTA prefetches the next job's input into L2 while it works.
// Synchronisation: a cluster barrier after each tile is written (data visible) and after each tile is
// read (the single tile buffer may be reused); the inverse adds one for the A_{m-1} broadcast.
#include <cuda_runtime.h>

#include <algorithm>

#include "nttf_core.cuh"

namespace bc {

int g_nttc_clusters = 0;   // persistent clusters per launch (0: the occupancy query's maximum)
int g_nttc_active = 0;     // the occupancy query's maximum (last launch's device)
int g_nttc_variant = 0;    // cluster shape: 0 = 8 CTAs x 512 threads, 1 = 16 x 256, 2 = 4 x 1024

namespace f64 {

__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t dsmem_map(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ double dsmem_ld(uint32_t a) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void dsmem_st(uint32_t a, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive_rel() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void prefetch_l2(const void *p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

template <int LOGR, int LOGC, int CL>
struct FusedShape {
    static constexpr int LOGE = 4, E = 1 << LOGE, R = 1 << LOGR, C = 1 << LOGC;
    static constexpr int TC = C / CL;                    // columns per CTA (phases A, C)
    static constexpr int RB = R / CL;                    // rows per CTA (phase B)
    static constexpr int THREADS = TC * (R / E);
    static_assert(THREADS == RB * (C / E), "phase shapes");
    static constexpr int ROWW = C + C / E;               // padded row of the row-transform exchange
    static constexpr int BUF = (R * TC > RB * ROWW ? R * TC : RB * ROWW);   // doubles
    typedef PtTab<LOGR, LOGE, true> PCF;
    typedef PtTab<LOGC, LOGE, true> PRF;
    typedef PtTab<LOGC, LOGE, false> PRI;
    typedef PtTab<LOGR, LOGE, false> PCI;
    // double2 words after the tile buffer: column fwd, column inv, then (R != C) row fwd, row inv -- twiddles and
    // per-thread tables; for R == C the row sets are the column sets (omega_R = omega_C, same table layouts)
    static constexpr bool SHARE = LOGR == LOGC;
    static constexpr int TWW = (R / 2 + PCF::WORDS) + (R / 2 + PCI::WORDS) + (SHARE ? 0 : (C / 2 + PRF::WORDS) + (C / 2 + PRI::WORDS));
    static constexpr size_t SMEM = (size_t)BUF * 8 + (size_t)TWW * 16 + 16;
};

// INV: 0 forward Bluestein, 1 inverse Bluestein (prime m: output reduced mod Phi_m)
template <int LOGR, int LOGC, int CL, int INV, int MINB>
__global__ void __launch_bounds__(FusedShape<LOGR, LOGC, CL>::THREADS, MINB)
    kc_bluestein(NttTables T, const uint64_t *__restrict__ in, uint64_t in_ps, uint64_t *__restrict__ out,
                 uint64_t out_ps, LimbMap lm, uint64_t job0, uint32_t nj) {
    typedef FusedShape<LOGR, LOGC, CL> S;
    constexpr int E = S::E, LOGE = S::LOGE, R = S::R, C = S::C, TC = S::TC, RB = S::RB;
    extern __shared__ __align__(16) double smc[];
    double *buf = smc;
    double2 *twA = (double2 *)(smc + S::BUF), *ptA = twA + R / 2;
    double2 *twC = ptA + S::PCF::WORDS, *ptC = twC + R / 2;
    double2 *twBf = S::SHARE ? twA : ptC + S::PCI::WORDS, *ptBf = S::SHARE ? ptA : twBf + C / 2;
    double2 *twBi = S::SHARE ? twC : ptBf + S::PRF::WORDS, *ptBi = S::SHARE ? ptC : twBi + C / 2;
    uint64_t *corner_slot = (uint64_t *)(twA + S::TWW);
    const uint32_t tid = threadIdx.x;
    const uint32_t rank = cluster_rank();
    const uint32_t ncl = gridDim.x / CL, cid = blockIdx.x / CL;
    const uint32_t buf_s = smem_addr(buf);
    // phase A / C thread roles: column col of this CTA's TC, register block tau of the length-R column
    const uint32_t col = tid % TC, tauc = tid / TC, c = rank * TC + col;
    // phase B: row rr of this CTA's RB, register block taur of the length-C row
    const uint32_t rr = tid / (C / E), taur = tid % (C / E), row = rank * RB + rr;
    uint32_t cur_pr = 0xffffffffu;
    for (uint32_t jj = cid; jj < nj; jj += ncl) {
        const JobF J = job_f(lm, (uint32_t)(job0 + jj));
        const double q = T.fmods[J.pr].x, qi = T.fmods[J.pr].y;
        if (J.pr != cur_pr) {           // uniform over the cluster (same job sequence)
            __syncthreads();
            const double2 *gA = T.ftwRb + (uint64_t)J.pr * (R / 2), *gBf = T.ftwCb + (uint64_t)J.pr * (C / 2);
            const double2 *gBi = T.ftwCi + (uint64_t)J.pr * (C / 2), *gC = T.ftwRi + (uint64_t)J.pr * (R / 2);
            for (uint32_t j = tid; j < (uint32_t)(R / 2); j += blockDim.x) {
                twA[j] = gA[j];
                twC[j] = gC[j];
            }
            if (!S::SHARE)
                for (uint32_t j = tid; j < (uint32_t)(C / 2); j += blockDim.x) {
                    twBf[j] = gBf[j];
                    twBi[j] = gBi[j];
                }
            if (tid < (uint32_t)(R / E)) {
                S::PCF::fill(ptA, tid, gA);
                S::PCI::fill(ptC, tid, gC);
            } else if (!S::SHARE && tid >= 32 && tid < 32 + (uint32_t)(C / E)) {
                S::PRF::fill(ptBf, tid - 32, gBf);
                S::PRI::fill(ptBi, tid - 32, gBi);
            }
            cur_pr = J.pr;
            __syncthreads();
        }
        double v[E];
        int bd[E];
        // ---------------- phase A: chirp + column forward transform + cross twiddle ----------------
        {
            const uint64_t *src = in + (uint64_t)J.poly * in_ps + (uint64_t)J.lb * T.n;
            const double *tf = (INV ? T.ftf1i : T.ftf1) + (uint64_t)J.pr * T.m;
#ifndef NOPF
            if (jj + ncl < nj) {        // next job of this cluster: its input into L2 while this one runs
                const JobF Jn = job_f(lm, (uint32_t)(job0 + jj + ncl));
                const uint64_t *sn = in + (uint64_t)Jn.poly * in_ps + (uint64_t)Jn.lb * T.n;
#pragma unroll
                for (int k = 0; k < E / 2; ++k) {
                    const uint32_t t = (tauc + ((uint32_t)k << (LOGR - LOGE))) * C + c;
                    if ((col & 3) == 0 && t < T.n) prefetch_l2(sn + t);
                }
            }
#endif
#pragma unroll
            for (int k = 0; k < E; ++k) {
                const uint32_t r = held_index<LOGE>(tauc, LOGR - LOGE, k);
                const uint32_t t = r * C + c;
                if (k >= E / 2) {       // rows >= R/2: the zero half of the Bluestein input (M/2 >= m > n)
                    v[k] = 0.0;
                    bd[k] = 0;
                    continue;
                }
                double x = 0.0;
                if (!INV) {
                    if (t < T.n) x = fmm8(from_u64(__ldcs(src + t)), tf[t], q, qi);
                } else if (t < T.m) {
                    const int ps = T.pos[t];
                    if (ps >= 0) x = fmm8(from_u64(__ldcs(src + ps)), tf[t], q, qi);
                }
                v[k] = x;
                bd[k] = UMUL8;
            }
            fct_pass<LOGR, LOGE, true, TC, 0>(v, bd, tauc, col, buf, twA, ptA, q, qi);
            const double *xt = T.fxta + (uint64_t)J.pr * T.M;
#pragma unroll
            for (int k = 0; k < E; ++k) {
                const uint32_t rp = held_index<LOGE>(tauc, 0, k);
                need(v, bd, k, LIM_MUL, q, qi);
                buf[rp * TC + col] = fmm8(v[k], xt[rp * C + c], q, qi);
            }
        }
        cluster_sync_all();             // every column tile written
        // ---------------- phase B: row forward, x D^, row inverse, cross twiddle ----------------
        {
#pragma unroll
            for (int k = 0; k < E; ++k) {
                const uint32_t cc = held_index<LOGE>(taur, LOGC - LOGE, k);
                v[k] = dsmem_ld(dsmem_map(buf_s + (row * TC + (cc % TC)) * 8, cc / TC));
                bd[k] = UMUL8;
            }
            cluster_arrive_rel();       // this CTA's tile reads are done; the first register pass runs before the
            double *srow = buf + rr * S::ROWW;  // wait (in frt_pass) that frees the tile buffer for the exchange
            frt_pass<LOGC, LOGE, true, 0, true>(v, bd, taur, srow, twBf, ptBf, q, qi);
            const double *dh = (INV ? T.fdhi : T.fdhf) + (uint64_t)J.pr * T.M + (uint64_t)row * C + taur;
#pragma unroll
            for (int k = 0; k < E; ++k) {
                need(v, bd, k, LIM_MUL, q, qi);
                v[k] = fmm8(v[k], dh[k * (C / E)], q, qi);
                bd[k] = UMUL8;
            }
            frt_pass<LOGC, LOGE, false, 0>(v, bd, taur, srow, twBi, ptBi, q, qi);
            const double *xt = T.fxtb + (uint64_t)J.pr * T.M + (uint64_t)row * C;
            __syncthreads();            // row exchanges done before the tile is rewritten
#pragma unroll
            for (int k = 0; k < E; ++k) {
                const uint32_t cc = held_index<LOGE>(taur, LOGC - LOGE, k);
                need(v, bd, k, LIM_MUL, q, qi);
                buf[rr * C + cc] = fmm8(v[k], xt[cc], q, qi);
            }
        }
        cluster_sync_all();             // every row tile written
        // ---------------- phase C: column inverse, output chirp, gather / reduction ----------------
        {
#pragma unroll
            for (int k = 0; k < E; ++k) {
                const uint32_t r = held_index<LOGE>(tauc, 0, k);
                v[k] = dsmem_ld(dsmem_map(buf_s + ((r % RB) * C + c) * 8, r / RB));
                bd[k] = UMUL8;
            }
            cluster_arrive_rel();       // tile reads done; wait before the first exchange (fct_pass)
            fct_pass<LOGR, LOGE, false, TC, 0, true>(v, bd, tauc, col, buf, twC, ptC, q, qi);
            const double *tfo = (INV ? T.ftfoi : T.ftfo) + (uint64_t)J.pr * T.m;
            uint64_t *dst = out + (uint64_t)J.poly * out_ps + (uint64_t)J.lb * T.n;
            if (!INV) {
#pragma unroll
                for (int k = 0; k < E / 2; ++k) {   // rows >= R/2: t >= M/2 >= m, never output
                    const uint32_t t = held_index<LOGE>(tauc, LOGR - LOGE, k) * C + c;
                    if (t >= T.m) continue;
                    need(v, bd, k, LIM_MUL, q, qi);
                    const int ps = T.pos[t];
                    if (ps >= 0) __stcs(dst + ps, to_u64(fmm8(v[k], tfo[t], q, qi), q));
                }
            } else {
                // prime m: a_t = A_t - A_{m-1} (t < n); the owner of t = m - 1 broadcasts A_{m-1}
                uint64_t x[E / 2];
#pragma unroll
                for (int k = 0; k < E / 2; ++k) {
                    const uint32_t t = held_index<LOGE>(tauc, LOGR - LOGE, k) * C + c;
                    x[k] = 0;
                    if (t >= T.m) continue;
                    need(v, bd, k, LIM_MUL, q, qi);
                    x[k] = to_u64(fmm8(v[k], tfo[t], q, qi), q);
                    if (t == T.m - 1) {
                        const uint32_t a = smem_addr(corner_slot);
                        for (uint32_t j = 0; j < (uint32_t)CL; ++j)
                            asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(dsmem_map(a, j)), "l"(x[k]) : "memory");
                    }
                }
                cluster_sync_all();     // A_{m-1} visible in every CTA
                const uint64_t corner = *(volatile uint64_t *)corner_slot, qq = (uint64_t)q;
#pragma unroll
                for (int k = 0; k < E / 2; ++k) {
                    const uint32_t t = held_index<LOGE>(tauc, LOGR - LOGE, k) * C + c;
                    if (t < T.n) __stcs(dst + t, x[k] >= corner ? x[k] - corner : x[k] + qq - corner);
                }
            }
        }
    }
}

template <int LOGR, int LOGC, int CL, int MINB>
static void runc(const NttTables &T, const uint64_t *in, uint64_t *out, LimbMap lm, uint64_t in_ps, uint64_t out_ps,
                 uint64_t j0, uint32_t nj, int inv, cudaStream_t st) {
    typedef FusedShape<LOGR, LOGC, CL> S;
    static std::atomic<uint64_t> init_dev{0};
    static int max_clusters[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    void (*kf)(NttTables, const uint64_t *, uint64_t, uint64_t *, uint64_t, LimbMap, uint64_t, uint32_t) =
        inv ? kc_bluestein<LOGR, LOGC, CL, 1, MINB> : kc_bluestein<LOGR, LOGC, CL, 0, MINB>;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(S::THREADS, 1, 1);
    cfg.dynamicSmemBytes = S::SMEM;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (attr_pending(init_dev)) {
        for (int d = 0; d < 2; ++d) {
            auto k = d ? kc_bluestein<LOGR, LOGC, CL, 1, MINB> : kc_bluestein<LOGR, LOGC, CL, 0, MINB>;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMEM);
            if (CL > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        }
        cfg.gridDim = dim3(CL * 148, 1, 1);
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, (void *)kc_bluestein<LOGR, LOGC, CL, 0, MINB>, &cfg) != cudaSuccess || ncl <= 0)
            ncl = 148 / CL;
        (void)cudaGetLastError();
        max_clusters[dev & 63] = ncl;
        attr_done(init_dev);
    }
    g_nttc_active = max_clusters[dev & 63];
    const uint32_t cap = g_nttc_clusters > 0 ? (uint32_t)g_nttc_clusters : (uint32_t)max_clusters[dev & 63];
    const uint32_t ncl = std::max<uint32_t>(1, std::min<uint32_t>(nj, cap));
    cfg.gridDim = dim3(ncl * CL, 1, 1);
    cudaLaunchKernelEx(&cfg, kf, T, in, in_ps, out, out_ps, lm, j0, nj);
    launch_counter() += 1;
}

}  // namespace f64

// the fused cluster kernel covers this table set: binary64 tables, the 256 x 256 grid (M = 65536), prime m
bool nttc_supported(const NttTables &T) {
    return T.fmods != nullptr && T.prime_m && T.logR == 8 && T.logC == 8 && nttf_row_loge(8, 8) == 4;
}

void nttc_run(const NttTables &T, const uint64_t *in, uint64_t *out, LimbMap lm, uint64_t in_ps, uint64_t out_ps,
              uint64_t j0, uint32_t nj, int inv, cudaStream_t st) {
    switch (g_nttc_variant) {
        case 1: f64::runc<8, 8, 16, 4>(T, in, out, lm, in_ps, out_ps, j0, nj, inv, st); break;
        case 2: f64::runc<8, 8, 4, 1>(T, in, out, lm, in_ps, out_ps, j0, nj, inv, st); break;
        default: f64::runc<8, 8, 8, 2>(T, in, out, lm, in_ps, out_ps, j0, nj, inv, st); break;
    }
}

}  // namespace bc
