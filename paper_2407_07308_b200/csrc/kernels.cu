// kernels.cu -- sm_100a kernels of the BoostCom BGV comparison hot path.
//
// a1/a2  Bluestein NTT (§2.2): chirp (TF1), size-M cyclic convolution with D_pad by a
//        four-step NTT (M = R x C: column pass, row pass with the pointwise D^ product fused
//        between the forward and inverse row transforms, inverse column pass), output chirp
//        and the Z_m^* filter of Listing 2 as a branch-free gather via pos[].
// a3     element-wise ring ops (§5.2): tensor, add, plaintext / scalar products.
// a4     automorphisms as an evaluation-index permutation.
// a5/a6  exact centered CRT lifts (Garner) for ModUp / ModDown / modulus switching.
// R7     counter-based sampler.  Encode/decode as exact int8 GEMMs over F_p.
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <stdexcept>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "kernels.h"
#include "f64arith.cuh"

namespace bc {

int g_ntt_impl = 0;
int g_ntt_dbg = 0;
int g_phi_conv = 0;
int g_f64_elem = 1;
uint64_t g_ntt_group_bytes = 1ull << 40;   // one launch group (measured best on B200)

uint64_t &launch_counter() {
    static thread_local uint64_t c = 0;
    return c;
}
#define LAUNCHED() (++launch_counter())

// live timing of the NTT family (bench roofline): an event pair around every ntt_forward /
// ntt_inverse call on the caller's stream, with the number of limb-transforms it ran
int g_ntt_timing = 0;
uint64_t g_vec_chunk = 0;   // max ciphertext pairs per batched compare in tournament / sort (0 = all)
int g_lift2 = 1;            // 1: binary64 lift with two coefficients per thread (k_lift_f2), 0: one (k_lift_f)
int g_kip_blocked = 1;      // 1: batch-blocked KIP (key words reused over 4 ciphertexts; two coefficients per
                            // thread with 128-bit accesses when no automorphism permutes the digits), 2: blocked
                            // with one coefficient per thread, 0: one ciphertext per thread
struct NttRec {
    cudaEvent_t a, b;
    uint64_t jobs;
    int inv;
};
static std::vector<NttRec> &ntt_recs() {
    static std::vector<NttRec> r;
    return r;
}
static std::vector<cudaEvent_t> &ev_pool() {
    static std::vector<cudaEvent_t> p;
    return p;
}
static cudaEvent_t ev_get() {
    auto &p = ev_pool();
    if (!p.empty()) {
        cudaEvent_t e = p.back();
        p.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}
int ntt_timing_collect(double *ms, uint64_t *jobs, uint64_t *calls, uint64_t *inv_jobs) {
    double t = 0;
    uint64_t j = 0, c = 0, ji = 0;
    for (auto &r : ntt_recs()) {
        float x = 0;
        if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&x, r.a, r.b) != cudaSuccess) return -1;
        t += x;
        j += r.jobs;
        if (r.inv) ji += r.jobs;
        ++c;
        ev_pool().push_back(r.a);
        ev_pool().push_back(r.b);
    }
    ntt_recs().clear();
    if (ms) *ms = t;
    if (jobs) *jobs = j;
    if (calls) *calls = c;
    if (inv_jobs) *inv_jobs = ji;
    return 0;
}

// per-phase timing of the comparison schedule (bench "phases": the Fig. 3 time breakdown):
// an event pair on the launching stream around each leaf phase, plus an NVTX range of the same name
int g_phase_timing = 0;
static const char *const k_phase_names[NPHASE] = {"extract", "digit_circuit", "lexicographic", "broadcast_select",
                                                 "compaction", "private_query_main"};
struct PhaseRec {
    int ph;
    cudaEvent_t a, b;
};
static std::vector<PhaseRec> &phase_recs() {
    static std::vector<PhaseRec> r;
    return r;
}
PhaseScope::PhaseScope(int ph, cudaStream_t st, bool on) : ph_(ph), st_(st), on_(on && ph >= 0 && ph < NPHASE) {
    if (!on_) return;
    nvtxRangePushA(k_phase_names[ph_]);
    if (g_phase_timing) {
        a_ = ev_get();
        cudaEventRecord((cudaEvent_t)a_, st_);
    }
}
PhaseScope::~PhaseScope() {
    if (!on_) return;
    if (g_phase_timing) {
        cudaEvent_t b = ev_get();
        cudaEventRecord(b, st_);
        phase_recs().push_back(PhaseRec{ph_, (cudaEvent_t)a_, b});
    }
    nvtxRangePop();
}
int phase_timing_collect(double *ms, uint64_t *calls) {
    for (int i = 0; i < NPHASE; ++i) {
        if (ms) ms[i] = 0;
        if (calls) calls[i] = 0;
    }
    for (auto &r : phase_recs()) {
        float x = 0;
        if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&x, r.a, r.b) != cudaSuccess) return -1;
        if (ms) ms[r.ph] += x;
        if (calls) calls[r.ph] += 1;
        ev_pool().push_back(r.a);
        ev_pool().push_back(r.b);
    }
    phase_recs().clear();
    return 0;
}

static inline unsigned grid_for(uint64_t total, unsigned threads, unsigned cap = 148u * 32u) {
    uint64_t g = (total + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (unsigned)g;
}

// Row-wise 2D launches (no per-element 64-bit division): blockIdx.x/threadIdx.x over the n coefficients
// of one row (a (ciphertext, part, limb) polynomial limb), blockIdx.y over rows.
#define ROW_LOOP(RV_, XV_, NROWS_, N_)                                  \
    const uint32_t XV_ = blockIdx.x * blockDim.x + threadIdx.x;         \
    if (XV_ >= (N_)) return;                                            \
    for (uint32_t RV_ = blockIdx.y; RV_ < (NROWS_); RV_ += gridDim.y)
// two coefficients per thread (n = phi(m) is even and every row starts 16-byte aligned): one 128-bit
// access per operand, x even
#define ROW_LOOP2(RV_, XV_, NROWS_, N_)                                 \
    const uint32_t XV_ = 2 * (blockIdx.x * blockDim.x + threadIdx.x);   \
    if (XV_ >= (N_)) return;                                            \
    for (uint32_t RV_ = blockIdx.y; RV_ < (NROWS_); RV_ += gridDim.y)
#define LD2(P_) (*(const ulonglong2 *)(P_))
#define ST2(P_, A_, B_) (*(ulonglong2 *)(P_) = make_ulonglong2((A_), (B_)))
static inline dim3 grid_rows(uint32_t n, uint64_t rows, unsigned threads = 256) {
    return dim3((n + threads - 1) / threads, (unsigned)(rows < 65535 ? (rows ? rows : 1) : 65535));
}

// =====================================================================================
// NTT building blocks (shared memory, radix-2)
// =====================================================================================
// cnt transforms of length len; element (a, i) at s[a*sa + i*si].
// COLT: consecutive threads take consecutive transforms a (column tiles, sa == 1);
// otherwise consecutive threads take consecutive butterflies (row tiles, si == 1).
template <bool COLT>
__device__ __forceinline__ void smem_dif(uint64_t *s, int lcnt, int llen, int sa, int si,
                                         const u64x2 *__restrict__ psi, uint32_t M, uint64_t q) {
    const int cnt = 1 << lcnt, halfn = 1 << (llen - 1);
    const int nb = cnt * halfn;
    for (int lh = llen - 1; lh >= 0; --lh) {
        const int h = 1 << lh;
        const uint32_t tstep = M >> (lh + 1);
        for (int t = threadIdx.x; t < nb; t += blockDim.x) {
            int a, b;
            if (COLT) { a = t & (cnt - 1); b = t >> lcnt; }
            else { a = t >> (llen - 1); b = t & (halfn - 1); }
            const int blk = b >> lh, jj = b & (h - 1);
            const int i0 = (blk << (lh + 1)) + jj, i1 = i0 + h;
            uint64_t *p0 = s + a * sa + i0 * si, *p1 = s + a * sa + i1 * si;
            const uint64_t x = *p0, y = *p1;
            *p0 = add_mod(x, y, q);
            const u64x2 w = psi[jj * tstep];
            *p1 = mul_shoup(sub_mod(x, y, q), w.w, w.ws, q);
        }
        __syncthreads();
    }
}

template <bool COLT>
__device__ __forceinline__ void smem_dit_inv(uint64_t *s, int lcnt, int llen, int sa, int si,
                                             const u64x2 *__restrict__ psi, uint32_t M, uint64_t q) {
    const int cnt = 1 << lcnt, halfn = 1 << (llen - 1);
    const int nb = cnt * halfn;
    for (int lh = 0; lh < llen; ++lh) {
        const int h = 1 << lh;
        const uint32_t tstep = M >> (lh + 1);
        for (int t = threadIdx.x; t < nb; t += blockDim.x) {
            int a, b;
            if (COLT) { a = t & (cnt - 1); b = t >> lcnt; }
            else { a = t >> (llen - 1); b = t & (halfn - 1); }
            const int blk = b >> lh, jj = b & (h - 1);
            const int i0 = (blk << (lh + 1)) + jj, i1 = i0 + h;
            uint64_t *p0 = s + a * sa + i0 * si, *p1 = s + a * sa + i1 * si;
            const uint64_t x = *p0;
            const u64x2 w = psi[(M - jj * tstep) & (M - 1)];
            const uint64_t y = mul_shoup(*p1, w.w, w.ws, q);
            *p0 = add_mod(x, y, q);
            *p1 = sub_mod(x, y, q);
        }
        __syncthreads();
    }
}

__device__ __forceinline__ uint32_t brev(uint32_t x, uint32_t bits) {
    return bits ? (__brev(x) >> (32 - bits)) : 0;
}

struct JobInfo {
    uint32_t poly, lb, pr;
};
__device__ __forceinline__ JobInfo job_info(const LimbMap &lm, uint32_t job) {
    JobInfo j;
    const uint32_t jl = job / lm.npoly;          // limb-major: polys sharing a prime are adjacent
    j.poly = job - jl * lm.npoly;
    j.lb = lm.limb(jl);
    j.pr = lm.prime(j.lb);
    return j;
}

// ---- pass A: chirp-multiply input, column DIF (length R), twiddle psi^(c*k1), store ----
template <int INV>
__global__ void __launch_bounds__(256) k_passA(NttTables T, const uint64_t *__restrict__ in,
                                               uint64_t in_pstride, LimbMap lm, uint64_t job0,
                                               uint64_t *__restrict__ scratch, int lTC) {
    extern __shared__ uint64_t sm[];
    const uint32_t job = (uint32_t)(job0 + blockIdx.y);
    const JobInfo J = job_info(lm, job);
    const uint64_t q = T.mods[J.pr].q;
    const uint64_t *src = in + (uint64_t)J.poly * in_pstride + (uint64_t)J.lb * T.n;
    const int TC = 1 << lTC;
    const uint32_t c0 = blockIdx.x << lTC;
    const u64x2 *tf = (INV ? T.tf1i : T.tf1) + (uint64_t)J.pr * T.m;
    const u64x2 *psi = T.psi + (uint64_t)J.pr * T.M;
    const int tot = T.R << lTC;
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
        const int r = e >> lTC, c = e & (TC - 1);
        const uint32_t t = r * T.C + c0 + c;
        uint64_t v = 0;
        if (!INV) {
            if (t < T.n) { const u64x2 w = tf[t]; v = mul_shoup(src[t], w.w, w.ws, q); }
        } else {
            if (t < T.m) {
                const int ps = T.pos[t];
                if (ps >= 0) { const u64x2 w = tf[t]; v = mul_shoup(src[ps], w.w, w.ws, q); }
            }
        }
        sm[e] = v;
    }
    __syncthreads();
    smem_dif<true>(sm, lTC, T.logR, 1, TC, psi, T.M, q);
    uint64_t *dst = scratch + (uint64_t)blockIdx.y * T.M;
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
        const int rp = e >> lTC, c = e & (TC - 1);
        const uint32_t k1 = brev(rp, T.logR);
        const u64x2 w = psi[((c0 + c) * k1) & (T.M - 1)];
        dst[rp * T.C + c0 + c] = mul_shoup(sm[e], w.w, w.ws, q);
    }
}

// ---- pass B: row DIF (length C), x D^, row inverse DIT, twiddle psi^(-c*k1) ----
template <int INV>
__global__ void __launch_bounds__(256) k_passB(NttTables T, LimbMap lm, uint64_t job0,
                                               uint64_t *__restrict__ scratch, int lTR) {
    extern __shared__ uint64_t sm[];
    const uint32_t job = (uint32_t)(job0 + blockIdx.y);
    const JobInfo J = job_info(lm, job);
    const uint64_t q = T.mods[J.pr].q;
    const u64x2 *psi = T.psi + (uint64_t)J.pr * T.M;
    const u64x2 *dh = (INV ? T.dhi : T.dhf) + (uint64_t)J.pr * T.M;
    const int TR = 1 << lTR;
    const uint32_t r0 = blockIdx.x << lTR;
    uint64_t *row = scratch + (uint64_t)blockIdx.y * T.M + (uint64_t)r0 * T.C;
    const int tot = TR << T.logC;
    for (int e = threadIdx.x; e < tot; e += blockDim.x) sm[e] = row[e];
    __syncthreads();
    smem_dif<false>(sm, lTR, T.logC, T.C, 1, psi, T.M, q);
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
        const u64x2 w = dh[(uint64_t)r0 * T.C + e];
        sm[e] = mul_shoup(sm[e], w.w, w.ws, q);
    }
    __syncthreads();
    smem_dit_inv<false>(sm, lTR, T.logC, T.C, 1, psi, T.M, q);
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
        const int a = e >> T.logC, c = e & (T.C - 1);
        const uint32_t k1 = brev(r0 + a, T.logR);
        const u64x2 w = psi[(T.M - c * k1) & (T.M - 1)];
        row[e] = mul_shoup(sm[e], w.w, w.ws, q);
    }
}

// ---- pass C: column inverse DIT (length R) -> natural t, output chirp, filter / store ----
template <int INV>
__global__ void __launch_bounds__(256) k_passC(NttTables T, uint64_t *__restrict__ out,
                                               uint64_t out_pstride, LimbMap lm, uint64_t job0,
                                               uint64_t *__restrict__ scratch, int lTC) {
    extern __shared__ uint64_t sm[];
    const uint32_t job = (uint32_t)(job0 + blockIdx.y);
    const JobInfo J = job_info(lm, job);
    const uint64_t q = T.mods[J.pr].q;
    const u64x2 *psi = T.psi + (uint64_t)J.pr * T.M;
    const int TC = 1 << lTC;
    const uint32_t c0 = blockIdx.x << lTC;
    uint64_t *scr = scratch + (uint64_t)blockIdx.y * T.M;
    const int tot = T.R << lTC;
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
        const int rp = e >> lTC, c = e & (TC - 1);
        sm[e] = scr[rp * T.C + c0 + c];
    }
    __syncthreads();
    smem_dit_inv<true>(sm, lTC, T.logR, 1, TC, psi, T.M, q);
    const u64x2 *tfo = (INV ? T.tfoi : T.tfo) + (uint64_t)J.pr * T.m;
    uint64_t *dst = out + (uint64_t)J.poly * out_pstride + (uint64_t)J.lb * T.n;
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
        const int r = e >> lTC, c = e & (TC - 1);
        const uint32_t t = r * T.C + c0 + c;
        if (t >= T.m) continue;
        const u64x2 w = tfo[t];
        const uint64_t v = mul_shoup(sm[e], w.w, w.ws, q);
        if (!INV) {
            const int ps = T.pos[t];
            if (ps >= 0) dst[ps] = v;
        } else {
            scr[t] = v;    // A_t, t < m (reduced mod Phi_m by k_reduce_phi)
        }
    }
}

// ---- inverse epilogue: reduce A (length m) modulo Phi_m ----
__global__ void k_reduce_prime(NttTables T, uint64_t *__restrict__ out, uint64_t out_pstride,
                               LimbMap lm, uint64_t job0, uint32_t njobs,
                               const uint64_t *__restrict__ scratch) {
    ROW_LOOP(jr, x, njobs, T.n) {
        const JobInfo J = job_info(lm, (uint32_t)(job0 + jr));
        const uint64_t q = T.mods[J.pr].q;
        const uint64_t *A = scratch + (uint64_t)jr * T.M;
        out[(uint64_t)J.poly * out_pstride + (uint64_t)J.lb * T.n + x] = sub_mod(A[x], A[T.m - 1], q);
    }
}

// composite m: long division by Phi_m (one CTA per job, m - n sequential steps)
__global__ void k_reduce_composite(NttTables T, uint64_t *__restrict__ out, uint64_t out_pstride,
                                   LimbMap lm, uint64_t job0, uint64_t *__restrict__ scratch) {
    const JobInfo J = job_info(lm, (uint32_t)(job0 + blockIdx.x));
    const uint64_t q = T.mods[J.pr].q;
    uint64_t *A = scratch + (uint64_t)blockIdx.x * T.M;
    for (int k = (int)T.m - 1; k >= (int)T.n; --k) {
        const uint64_t c = A[k];
        __syncthreads();
        for (int j = threadIdx.x; j < (int)T.n; j += blockDim.x) {
            const int f = T.phi[j];
            uint64_t *d = &A[k - T.n + j];
            if (f == 1) *d = sub_mod(*d, c, q);
            else if (f == -1) *d = add_mod(*d, c, q);
            else if (f != 0) {
                const uint64_t fm = from_signed(f, q);
                *d = sub_mod(*d, mul_mod(c, fm, T.mods[J.pr]), q);
            }
        }
        __syncthreads();
    }
    uint64_t *dst = out + (uint64_t)J.poly * out_pstride + (uint64_t)J.lb * T.n;
    for (int j = threadIdx.x; j < (int)T.n; j += blockDim.x) dst[j] = A[j];
}

// jobs per launch group: scratch of one group stays within g_ntt_group_bytes (Barrett: two slots per job)
uint64_t ntt_group_jobs(const NttTables &T, uint64_t jobs, bool barrett) {
    const uint64_t g = std::max<uint64_t>(1, std::min<uint64_t>(65535, (uint64_t)g_ntt_group_bytes / ((uint64_t)T.M * 8 * (barrett ? 2 : 1))));
    return std::max<uint64_t>(1, std::min(jobs, g));
}
bool ntt_inverse_barrett(const NttTables &T) {
    return (g_ntt_impl == 0 || g_ntt_impl >= 10) && nttf_supported(T) && !T.prime_m && T.tb != nullptr;
}

static void ntt_common(const NttTables &T, const uint64_t *in, uint64_t *out, uint32_t npoly, LimbMap lm,
                       uint64_t in_pstride, uint64_t out_pstride, uint64_t *scratch, cudaStream_t st,
                       int inv) {
    const uint64_t jobs = (uint64_t)npoly * lm.njl;
    if (!jobs) return;
    const int lTC = T.logC < 4 ? (int)T.logC : 4;
    const int lTR = T.logR < 3 ? (int)T.logR : 3;
    const size_t smA = ((size_t)T.R << lTC) * 8, smB = ((size_t)T.C << lTR) * 8;
    static std::atomic<uint64_t> attr_set_dev{0};
    if (attr_pending(attr_set_dev)) {
        cudaFuncSetAttribute(k_passA<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        cudaFuncSetAttribute(k_passA<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        cudaFuncSetAttribute(k_passB<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        cudaFuncSetAttribute(k_passB<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        cudaFuncSetAttribute(k_passC<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        cudaFuncSetAttribute(k_passC<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        attr_done(attr_set_dev);
    }
    lm.npoly = npoly;
    if (T.rad > 1 && !((g_ntt_impl == 0 || g_ntt_impl >= 10) && nttf_supported(T)))
        throw std::runtime_error("mixed-radix Bluestein lengths (R25) run on the binary64 passes only");
    // L2-sized job groups: the scratch of one group (A -> B -> C) stays resident in the 126 MB L2
    const bool vf = (g_ntt_impl == 0 || g_ntt_impl >= 10) && nttf_supported(T);   // 20: fused cluster kernel (below)
    // composite m on the binary64 path: Barrett reduction mod Phi_m (needs a second M-word slot per job)
    const bool barrett = inv && vf && !T.prime_m && T.tb != nullptr;
    const uint64_t chunk = ntt_group_jobs(T, jobs, barrett);
    const bool v2 = g_ntt_impl != 1 && (ntt2_supported(T) || (T.rad > 1 && vf));   // R25 rows: binary64 only
    for (uint64_t j0 = 0; j0 < jobs; j0 += chunk) {
        const uint32_t nj = (uint32_t)((jobs - j0) < chunk ? (jobs - j0) : chunk);
        dim3 gA(T.C >> lTC, nj), gB(T.R >> lTR, nj);
        if (g_ntt_impl == 20 && nttf_supported(T) && nttc_supported(T)) {
            nttc_run(T, in, out, lm, in_pstride, out_pstride, j0, nj, inv, st);
        } else if (v2) {
            const bool direct = vf && inv && T.prime_m;      // pass C writes A_t - A_{m-1} itself
            if (vf) {
                nttf_run(T, in, out, lm, in_pstride, out_pstride, scratch, j0, nj, inv, st,
                         direct ? scratch + chunk * T.M : nullptr);
                if (barrett) nttf_barrett(*T.tb, out, lm, out_pstride, scratch, scratch + chunk * T.M, j0, nj, st);
            } else
                ntt2_run(T, in, out, lm, in_pstride, out_pstride, scratch, j0, nj, inv, st);
            if (inv && !barrett && !direct) {
                if (T.prime_m)
                    k_reduce_prime<<<grid_rows(T.n, nj), 256, 0, st>>>(T, out, out_pstride, lm, j0, nj,
                                                                                     scratch);
                else
                    k_reduce_composite<<<nj, 256, 0, st>>>(T, out, out_pstride, lm, j0, scratch);
                launch_counter() += 1;
            }
        } else if (!inv) {
            k_passA<0><<<gA, 256, smA, st>>>(T, in, in_pstride, lm, j0, scratch, lTC);
            k_passB<0><<<gB, 256, smB, st>>>(T, lm, j0, scratch, lTR);
            k_passC<0><<<gA, 256, smA, st>>>(T, out, out_pstride, lm, j0, scratch, lTC);
            launch_counter() += 3;
        } else {
            k_passA<1><<<gA, 256, smA, st>>>(T, in, in_pstride, lm, j0, scratch, lTC);
            k_passB<1><<<gB, 256, smB, st>>>(T, lm, j0, scratch, lTR);
            k_passC<1><<<gA, 256, smA, st>>>(T, out, out_pstride, lm, j0, scratch, lTC);
            if (T.prime_m)
                k_reduce_prime<<<grid_rows(T.n, nj), 256, 0, st>>>(T, out, out_pstride, lm, j0,
                                                                                 nj, scratch);
            else
                k_reduce_composite<<<nj, 256, 0, st>>>(T, out, out_pstride, lm, j0, scratch);
            launch_counter() += 4;
        }
    }
}

// two-stream split (bc_tune "ntt_split"): the polys of a call in two halves on the caller's stream and a
// side stream (fork / join by events, capturable), with the persistent column passes capped at one CTA
// per SM so that one half's row pass can share the SMs with the other half's column passes.  Disjoint
// scratch regions; the words are identical (every job is independent).
int g_ntt_split = 0;
int g_ntt_persist_occ = 0;
int g_ntt_lean = 4;
int g_ptsum = 1;
int g_lift_blocks = 16;
int g_axpy = 1;
int g_ntt_epi = 0;      // measured: C2 compare 3.53 -> 3.55 ms with the fused epilogue (pass C's scattered
                        // u / d loads cost more than the separate 128-bit streaming kernel), so off
static cudaStream_t side_stream_for_device() {
    static std::mutex mu;
    static cudaStream_t s[64] = {nullptr};
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    if (!s[dev & 63]) cudaStreamCreateWithFlags(&s[dev & 63], cudaStreamNonBlocking);
    return s[dev & 63];
}
static void ntt_split_or_common(const NttTables &T, const uint64_t *in, uint64_t *out, uint32_t npoly, LimbMap lm,
                                uint64_t in_pstride, uint64_t out_pstride, uint64_t *scratch, cudaStream_t st, int inv) {
    const uint64_t jobs = (uint64_t)npoly * lm.njl;
    const bool barrett = inv && nttf_supported(T) && !T.prime_m && T.tb != nullptr;
    if (!g_ntt_split || npoly < 2 || jobs < 2 * 296 || ntt_group_jobs(T, jobs, barrett) < jobs) {
        ntt_common(T, in, out, npoly, lm, in_pstride, out_pstride, scratch, st, inv);
        return;
    }
    const uint32_t p1 = npoly / 2, p2 = npoly - p1;
    const uint64_t j1 = (uint64_t)p1 * lm.njl;
    uint64_t *scr2 = scratch + j1 * T.M * (barrett ? 2 : 1) + (inv ? j1 : 0);
    cudaStream_t side = side_stream_for_device();
    cudaEvent_t fork = ev_get(), join = ev_get();
    cudaEventRecord(fork, st);
    cudaStreamWaitEvent(side, fork, 0);
    const int occ = g_ntt_persist_occ;
    g_ntt_persist_occ = 1;
    ntt_common(T, in, out, p1, lm, in_pstride, out_pstride, scratch, st, inv);
    ntt_common(T, in + (uint64_t)p1 * in_pstride, out + (uint64_t)p1 * out_pstride, p2, lm, in_pstride, out_pstride,
               scr2, side, inv);
    g_ntt_persist_occ = occ;
    cudaEventRecord(join, side);
    cudaStreamWaitEvent(st, join, 0);
    ev_pool().push_back(fork);          // reusable once recorded work completes: re-recording is ordered
    ev_pool().push_back(join);
}

static void ntt_timed(const NttTables &T, const uint64_t *in, uint64_t *out, uint32_t npoly, LimbMap lm,
                      uint64_t in_pstride, uint64_t out_pstride, uint64_t *scratch, cudaStream_t st, int inv) {
    if (!g_ntt_timing) {
        ntt_split_or_common(T, in, out, npoly, lm, in_pstride, out_pstride, scratch, st, inv);
        return;
    }
    NttRec r{ev_get(), ev_get(), (uint64_t)npoly * lm.njl, inv};
    cudaEventRecord(r.a, st);
    ntt_split_or_common(T, in, out, npoly, lm, in_pstride, out_pstride, scratch, st, inv);
    cudaEventRecord(r.b, st);
    ntt_recs().push_back(r);
}
void ntt_forward(const NttTables &T, const uint64_t *in, uint64_t *out, uint32_t npoly, LimbMap lm,
                 uint64_t in_pstride, uint64_t out_pstride, uint64_t *scratch, cudaStream_t st) {
    ntt_timed(T, in, out, npoly, lm, in_pstride, out_pstride, scratch, st, 0);
}
void ntt_inverse(const NttTables &T, const uint64_t *in, uint64_t *out, uint32_t npoly, LimbMap lm,
                 uint64_t in_pstride, uint64_t out_pstride, uint64_t *scratch, cudaStream_t st) {
    ntt_timed(T, in, out, npoly, lm, in_pstride, out_pstride, scratch, st, 1);
}
bool ntt_epi_supported(const NttTables &T) {
    return (g_ntt_impl == 0 || (g_ntt_impl >= 10 && g_ntt_impl != 20)) && nttf_supported(T) && !g_ntt_split;
}
void ntt_forward_epi(const NttTables &T, const NttEpi &e, const uint64_t *in, uint64_t *out, uint32_t npoly, LimbMap lm,
                     uint64_t in_pstride, uint64_t out_pstride, uint64_t *scratch, cudaStream_t st) {
    if (!ntt_epi_supported(T)) throw std::runtime_error("ntt_forward_epi: fused epilogue needs the binary64 passes");
    NttTables Te = T;
    Te.epi = e;
    ntt_timed(Te, in, out, npoly, lm, in_pstride, out_pstride, scratch, st, 0);
}

// =====================================================================================
// element-wise kernels, layout [B][parts][lvl][n]; limb i -> prime i
// =====================================================================================
#define GRID_LOOP(i, total) \
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (total); i += (uint64_t)gridDim.x * blockDim.x)

// residue of a small signed constant (|c| < q: the engine's constants are in F_p or small)
__device__ __forceinline__ uint64_t small_res(int64_t c, uint64_t q) {
    if (c >= 0) return (uint64_t)c < q ? (uint64_t)c : (uint64_t)c % q;
    const uint64_t a = (uint64_t)(-c);
    return a < q ? (a ? q - a : 0) : from_signed(c, q);
}

__global__ void k_add(const Mod *__restrict__ mods, const uint64_t *__restrict__ a, const uint64_t *__restrict__ b,
                      uint64_t *__restrict__ o, uint32_t rows, uint32_t lvl, uint32_t n, int sub) {
    ROW_LOOP2(r, x, rows, n) {
        const uint64_t q = mods[r % lvl].q, i = (uint64_t)r * n + x;
        const ulonglong2 av = LD2(a + i), bv = LD2(b + i);
        if (sub) ST2(o + i, sub_mod(av.x, bv.x, q), sub_mod(av.y, bv.y, q));
        else ST2(o + i, add_mod(av.x, bv.x, q), add_mod(av.y, bv.y, q));
    }
}
void ew_add(const Mod *mods, const uint64_t *a, const uint64_t *b, uint64_t *o, uint32_t B, uint32_t parts,
            uint32_t lvl, uint32_t n, int sub, cudaStream_t st) {
    const uint64_t rows = (uint64_t)B * parts * lvl;
    k_add<<<grid_rows(n / 2, rows), 256, 0, st>>>(mods, a, b, o, (uint32_t)rows, lvl, n, sub);
    LAUNCHED();
}

__global__ void k_neg(const Mod *__restrict__ mods, const uint64_t *__restrict__ a, uint64_t *__restrict__ o,
                      uint32_t rows, uint32_t lvl, uint32_t n) {
    ROW_LOOP(r, x, rows, n) {
        const uint64_t i = (uint64_t)r * n + x;
        o[i] = neg_mod(a[i], mods[r % lvl].q);
    }
}
void ew_neg(const Mod *mods, const uint64_t *a, uint64_t *o, uint32_t B, uint32_t parts, uint32_t lvl,
            uint32_t n, cudaStream_t st) {
    const uint64_t rows = (uint64_t)B * parts * lvl;
    k_neg<<<grid_rows(n, rows), 256, 0, st>>>(mods, a, o, (uint32_t)rows, lvl, n);
    LAUNCHED();
}

__global__ void k_scalar(const Mod *__restrict__ mods, const uint64_t *__restrict__ a, int64_t c,
                         uint64_t *__restrict__ o, uint32_t rows, uint32_t lvl, uint32_t n) {
    ROW_LOOP(r, x, rows, n) {
        const Mod M = mods[r % lvl];
        const uint64_t i = (uint64_t)r * n + x;
        o[i] = mul_mod(a[i], small_res(c, M.q), M);
    }
}
// binary64: c (|c| < p) times a canonical residue, |r| <= 0.75 q (wq = fl(c fl(1/q)), |c| << q)
__global__ void k_scalar_f(const double2 *__restrict__ fm, const uint64_t *__restrict__ a, int64_t c,
                           uint64_t *__restrict__ o, uint32_t rows, uint32_t lvl, uint32_t n) {
    using namespace f64;
    const double cd = (double)c;
    ROW_LOOP2(r, x, rows, n) {
        const double q = fm[r % lvl].x, qi = fm[r % lvl].y;
        const uint64_t i = (uint64_t)r * n + x;
        const ulonglong2 av = LD2(a + i);
        ST2(o + i, to_u64(fmulv(from_u64(av.x), cd, q, qi), q), to_u64(fmulv(from_u64(av.y), cd, q, qi), q));
    }
}
void ew_scalar(const Mod *mods, const uint64_t *a, int64_t c, uint64_t *o, uint32_t B, uint32_t parts,
               uint32_t lvl, uint32_t n, cudaStream_t st, const double2 *fm) {
    const uint64_t rows = (uint64_t)B * parts * lvl;
    if (fm && c > -(1 << 20) && c < (1 << 20))
        k_scalar_f<<<grid_rows(n / 2, rows), 256, 0, st>>>(fm, a, c, o, (uint32_t)rows, lvl, n);
    else
        k_scalar<<<grid_rows(n, rows), 256, 0, st>>>(mods, a, c, o, (uint32_t)rows, lvl, n);
    LAUNCHED();
}

// R27: W[b][k][r] (+)= u[b][k][r] + (r < lv ? (P mod q_r) d_k[b][r] : 0) over the lv cipher rows and the K
// special rows (prime L1 + r - lv) of the extended basis -- R15's w_k of one product, summed (first: W = w)
__global__ void k_ext_acc(const Mod *__restrict__ mods, uint64_t *__restrict__ W, const uint64_t *__restrict__ u,
                          const uint64_t *__restrict__ d, uint64_t d_bstride, uint64_t d_kstride,
                          const u64x2 *__restrict__ pm, uint32_t rows, uint32_t lv, uint32_t nl, uint32_t L1,
                          uint32_t n, int first) {
    ROW_LOOP(rw, x, rows, n) {   // rows = 2B * nl
        const uint64_t poly = rw / nl;
        const uint32_t r = rw - (uint32_t)poly * nl;
        const uint64_t q = mods[r < lv ? r : L1 + (r - lv)].q, i = (uint64_t)rw * n + x;
        uint64_t w = u[i];
        if (r < lv) {
            const u64x2 c = pm[r];
            w = add_mod(w, mul_shoup(d[(poly >> 1) * d_bstride + (poly & 1) * d_kstride + (uint64_t)r * n + x], c.w, c.ws, q), q);
        }
        W[i] = first ? w : add_mod(W[i], w, q);
    }
}
void ew_ext_acc(const Mod *mods, uint64_t *W, const uint64_t *u, const uint64_t *d, uint64_t d_bstride,
                uint64_t d_kstride, const u64x2 *pm, uint32_t B, uint32_t lv, uint32_t K, uint32_t L1, uint32_t n,
                int first, cudaStream_t st) {
    const uint64_t rows = (uint64_t)2 * B * (lv + K);
    k_ext_acc<<<grid_rows(n, rows), 256, 0, st>>>(mods, W, u, d, d_bstride, d_kstride, pm, (uint32_t)rows, lv, lv + K,
                                                  L1, n, first);
    LAUNCHED();
}

// o = a + c x (the linear-combination step of the digit circuits: one pass instead of ew_scalar + ew_add)
__global__ void k_axpy(const Mod *__restrict__ mods, const uint64_t *__restrict__ a, const uint64_t *__restrict__ xs,
                       int64_t c, uint64_t *__restrict__ o, uint32_t rows, uint32_t lvl, uint32_t n) {
    ROW_LOOP(r, x, rows, n) {
        const Mod M = mods[r % lvl];
        const uint64_t i = (uint64_t)r * n + x;
        o[i] = add_mod(a[i], mul_mod(xs[i], small_res(c, M.q), M), M.q);
    }
}
__global__ void k_axpy_f(const double2 *__restrict__ fm, const uint64_t *__restrict__ a, const uint64_t *__restrict__ xs,
                         int64_t c, uint64_t *__restrict__ o, uint32_t rows, uint32_t lvl, uint32_t n) {
    using namespace f64;
    const double cd = (double)c;
    ROW_LOOP2(r, x, rows, n) {
        const double q = fm[r % lvl].x, qi = fm[r % lvl].y;
        const uint64_t qq = (uint64_t)q, i = (uint64_t)r * n + x;
        const ulonglong2 av = LD2(a + i), xv = LD2(xs + i);
        ST2(o + i, add_mod(av.x, to_u64(fmulv(from_u64(xv.x), cd, q, qi), q), qq),
            add_mod(av.y, to_u64(fmulv(from_u64(xv.y), cd, q, qi), q), qq));
    }
}
void ew_axpy(const Mod *mods, const uint64_t *a, const uint64_t *x, int64_t c, uint64_t *o, uint32_t B, uint32_t parts,
             uint32_t lvl, uint32_t n, cudaStream_t st, const double2 *fm) {
    const uint64_t rows = (uint64_t)B * parts * lvl;
    if (fm && c > -(1 << 20) && c < (1 << 20))
        k_axpy_f<<<grid_rows(n / 2, rows), 256, 0, st>>>(fm, a, x, c, o, (uint32_t)rows, lvl, n);
    else
        k_axpy<<<grid_rows(n, rows), 256, 0, st>>>(mods, a, x, c, o, (uint32_t)rows, lvl, n);
    LAUNCHED();
}

__global__ void k_add_const(const Mod *__restrict__ mods, const uint64_t *__restrict__ a, int64_t c,
                            uint64_t *__restrict__ o, uint32_t rows, uint32_t parts, uint32_t lvl, uint32_t n) {
    ROW_LOOP2(r, x, rows, n) {
        const uint32_t limb = r % lvl, part = (r / lvl) % parts;
        const uint64_t q = mods[limb].q, i = (uint64_t)r * n + x;
        const ulonglong2 av = LD2(a + i);
        if (part == 0) {
            const uint64_t cr = small_res(c, q);
            ST2(o + i, add_mod(av.x, cr, q), add_mod(av.y, cr, q));
        } else {
            ST2(o + i, av.x, av.y);
        }
    }
}
void ew_add_const(const Mod *mods, const uint64_t *a, int64_t c, uint64_t *o, uint32_t B, uint32_t parts,
                  uint32_t lvl, uint32_t n, cudaStream_t st) {
    const uint64_t rows = (uint64_t)B * parts * lvl;
    k_add_const<<<grid_rows(n / 2, rows), 256, 0, st>>>(mods, a, c, o, (uint32_t)rows, parts, lvl, n);
    LAUNCHED();
}

__global__ void k_ptmul(const Mod *__restrict__ mods, const uint64_t *__restrict__ a,
                        const uint64_t *__restrict__ pt, uint64_t *__restrict__ o, uint32_t rows,
                        uint32_t lvl, uint32_t n) {
    ROW_LOOP(r, x, rows, n) {
        const uint32_t limb = r % lvl;
        const uint64_t i = (uint64_t)r * n + x;
        o[i] = mul_mod(a[i], pt[(uint64_t)limb * n + x], mods[limb]);
    }
}
__global__ void k_ptmul_f(const double2 *__restrict__ fm, const uint64_t *__restrict__ a,
                          const uint64_t *__restrict__ pt, uint64_t *__restrict__ o, uint32_t rows,
                          uint32_t lvl, uint32_t n) {
    using namespace f64;
    ROW_LOOP2(r, x, rows, n) {
        const uint32_t limb = r % lvl;
        const double q = fm[limb].x, qi = fm[limb].y;
        const uint64_t i = (uint64_t)r * n + x;
        const ulonglong2 av = LD2(a + i), pv = LD2(pt + (uint64_t)limb * n + x);
        ST2(o + i, to_u64(fmulv(from_u64(av.x), from_u64(pv.x), q, qi), q),
            to_u64(fmulv(from_u64(av.y), from_u64(pv.y), q, qi), q));
    }
}
void ew_ptmul(const Mod *mods, const uint64_t *a, const uint64_t *pt, uint64_t *o, uint32_t B, uint32_t parts,
              uint32_t lvl, uint32_t n, cudaStream_t st, const double2 *fm) {
    const uint64_t rows = (uint64_t)B * parts * lvl;
    if (fm)
        k_ptmul_f<<<grid_rows(n / 2, rows), 256, 0, st>>>(fm, a, pt, o, (uint32_t)rows, lvl, n);
    else
        k_ptmul<<<grid_rows(n, rows), 256, 0, st>>>(mods, a, pt, o, (uint32_t)rows, lvl, n);
    LAUNCHED();
}

// a8 digit extraction: o = sum_k pt_k (.) F_k (the kappa-weighted sum of the Frobenius images) in one
// pass instead of D plaintext products and D - 1 additions (modular sums are exact: the same words)
__global__ void k_ptsum(const Mod *__restrict__ mods, PtSumArgs A, uint64_t *__restrict__ o, uint32_t rows, uint32_t lvl,
                        uint32_t n) {
    ROW_LOOP(r, x, rows, n) {
        const uint32_t limb = r % lvl;
        const Mod M = mods[limb];
        const uint64_t i = (uint64_t)r * n + x, j = (uint64_t)limb * n + x;
        uint64_t acc = 0;
        for (uint32_t k = 0; k < A.D; ++k) acc = add_mod(acc, mul_mod(A.F[k][i], A.pt[k][j], M), M.q);
        o[i] = acc;
    }
}
__global__ void k_ptsum_f(const double2 *__restrict__ fm, PtSumArgs A, uint64_t *__restrict__ o, uint32_t rows,
                          uint32_t lvl, uint32_t n) {
    using namespace f64;
    ROW_LOOP2(r, x, rows, n) {
        const uint32_t limb = r % lvl;
        const double q = fm[limb].x, qi = fm[limb].y;
        const uint64_t i = (uint64_t)r * n + x, j = (uint64_t)limb * n + x;
        double a0 = 0.0, a1 = 0.0;      // |a| <= q/2 + 2 after each fred, + a product |r| <= 0.75 q
        for (uint32_t k = 0; k < A.D; ++k) {
            const ulonglong2 fv = LD2(A.F[k] + i), pv = LD2(A.pt[k] + j);
            a0 = fred(__dadd_rn(a0, fmulv(from_u64(fv.x), from_u64(pv.x), q, qi)), q, qi);
            a1 = fred(__dadd_rn(a1, fmulv(from_u64(fv.y), from_u64(pv.y), q, qi)), q, qi);
        }
        ST2(o + i, to_u64(a0, q), to_u64(a1, q));
    }
}
void ew_ptsum(const Mod *mods, const PtSumArgs &A, uint64_t *o, uint32_t B, uint32_t parts, uint32_t lvl, uint32_t n,
              cudaStream_t st, const double2 *fm) {
    const uint64_t rows = (uint64_t)B * parts * lvl;
    if (fm)
        k_ptsum_f<<<grid_rows(n / 2, rows), 256, 0, st>>>(fm, A, o, (uint32_t)rows, lvl, n);
    else
        k_ptsum<<<grid_rows(n, rows), 256, 0, st>>>(mods, A, o, (uint32_t)rows, lvl, n);
    LAUNCHED();
}

// o = a (.) pm, + pa on part 0 (ShiftMul's masked rotation plus 1 - mask, a9: one pass for ptmul + add_pt)
__global__ void k_ptmul_addpt_f(const double2 *__restrict__ fm, const uint64_t *__restrict__ a,
                                const uint64_t *__restrict__ pm, const uint64_t *__restrict__ pa, uint64_t *__restrict__ o,
                                uint32_t rows, uint32_t parts, uint32_t lvl, uint32_t n) {
    using namespace f64;
    ROW_LOOP2(r, x, rows, n) {
        const uint32_t limb = r % lvl, part = (r / lvl) % parts;
        const double q = fm[limb].x, qi = fm[limb].y;
        const uint64_t qq = (uint64_t)q, i = (uint64_t)r * n + x, j = (uint64_t)limb * n + x;
        const ulonglong2 av = LD2(a + i), mv = LD2(pm + j);
        uint64_t r0 = to_u64(fmulv(from_u64(av.x), from_u64(mv.x), q, qi), q);
        uint64_t r1 = to_u64(fmulv(from_u64(av.y), from_u64(mv.y), q, qi), q);
        if (part == 0) {
            const ulonglong2 cv = LD2(pa + j);
            r0 = add_mod(r0, cv.x, qq);
            r1 = add_mod(r1, cv.y, qq);
        }
        ST2(o + i, r0, r1);
    }
}
void ew_ptmul_addpt(const double2 *fm, const uint64_t *a, const uint64_t *pm, const uint64_t *pa, uint64_t *o,
                    uint32_t B, uint32_t parts, uint32_t lvl, uint32_t n, cudaStream_t st) {
    const uint64_t rows = (uint64_t)B * parts * lvl;
    k_ptmul_addpt_f<<<grid_rows(n / 2, rows), 256, 0, st>>>(fm, a, pm, pa, o, (uint32_t)rows, parts, lvl, n);
    LAUNCHED();
}

__global__ void k_add_pt(const Mod *__restrict__ mods, const uint64_t *__restrict__ a,
                         const uint64_t *__restrict__ pt, uint64_t *__restrict__ o, uint32_t rows,
                         uint32_t parts, uint32_t lvl, uint32_t n) {
    ROW_LOOP(r, x, rows, n) {
        const uint32_t limb = r % lvl, part = (r / lvl) % parts;
        const uint64_t i = (uint64_t)r * n + x;
        o[i] = part == 0 ? add_mod(a[i], pt[(uint64_t)limb * n + x], mods[limb].q) : a[i];
    }
}
void ew_add_pt(const Mod *mods, const uint64_t *a, const uint64_t *pt, uint64_t *o, uint32_t B, uint32_t parts,
               uint32_t lvl, uint32_t n, cudaStream_t st) {
    const uint64_t rows = (uint64_t)B * parts * lvl;
    k_add_pt<<<grid_rows(n, rows), 256, 0, st>>>(mods, a, pt, o, (uint32_t)rows, parts, lvl, n);
    LAUNCHED();
}

// tensor: (a0 b0, a0 b1 + a1 b0, a1 b1)
__global__ void k_tensor(const Mod *__restrict__ mods, const uint64_t *__restrict__ a,
                         const uint64_t *__restrict__ b, uint64_t *__restrict__ o, uint32_t rows,
                         uint32_t lvl, uint32_t n) {
    const uint64_t ln = (uint64_t)lvl * n;
    ROW_LOOP(rw, x, rows, n) {   // rows = B * lvl
        const uint32_t bi = rw / lvl, limb = rw - bi * lvl;
        const uint64_t r = (uint64_t)limb * n + x;
        const Mod M = mods[limb];
        const uint64_t a0 = a[bi * 2 * ln + r], a1 = a[bi * 2 * ln + ln + r];
        const uint64_t b0 = b[bi * 2 * ln + r], b1 = b[bi * 2 * ln + ln + r];
        uint64_t *ob = o + bi * 3 * ln + r;
        ob[0] = mul_mod(a0, b0, M);
        ob[ln] = add_mod(mul_mod(a0, b1, M), mul_mod(a1, b0, M), M.q);
        ob[2 * ln] = mul_mod(a1, b1, M);
    }
}
// binary64 variant (all primes in [2^49, 2^50)): four fmulv per coefficient
__global__ void k_tensor_f(const double2 *__restrict__ fm, const uint64_t *__restrict__ a,
                           const uint64_t *__restrict__ b, uint64_t *__restrict__ o, uint32_t rows,
                           uint32_t lvl, uint32_t n) {
    using namespace f64;
    const uint64_t ln = (uint64_t)lvl * n;
    ROW_LOOP2(rw, x, rows, n) {   // rows = B * lvl; two coefficients per thread
        const uint32_t bi = rw / lvl, limb = rw - bi * lvl;
        const uint64_t r = (uint64_t)limb * n + x;
        const double q = fm[limb].x, qi = fm[limb].y;
        const ulonglong2 A0 = LD2(a + bi * 2 * ln + r), A1 = LD2(a + bi * 2 * ln + ln + r);
        const ulonglong2 B0 = LD2(b + bi * 2 * ln + r), B1 = LD2(b + bi * 2 * ln + ln + r);
        uint64_t *ob = o + bi * 3 * ln + r;
        uint64_t d0[2], d1[2], d2[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const double a0 = from_u64(e ? A0.y : A0.x), a1 = from_u64(e ? A1.y : A1.x);
            const double b0 = from_u64(e ? B0.y : B0.x), b1 = from_u64(e ? B1.y : B1.x);
            d0[e] = to_u64(fmulv(a0, b0, q, qi), q);
            d1[e] = to_u64(fred(__dadd_rn(fmulv(a0, b1, q, qi), fmulv(a1, b0, q, qi)), q, qi), q);
            d2[e] = to_u64(fmulv(a1, b1, q, qi), q);
        }
        ST2(ob, d0[0], d0[1]);
        ST2(ob + ln, d1[0], d1[1]);
        ST2(ob + 2 * ln, d2[0], d2[1]);
    }
}
void ew_tensor(const Mod *mods, const uint64_t *a, const uint64_t *b, uint64_t *o, uint32_t B, uint32_t lvl,
               uint32_t n, cudaStream_t st, const double2 *fm) {
    const uint64_t rows = (uint64_t)B * lvl;
    if (fm)
        k_tensor_f<<<grid_rows(n / 2, rows), 256, 0, st>>>(fm, a, b, o, (uint32_t)rows, lvl, n);
    else
        k_tensor<<<grid_rows(n, rows), 256, 0, st>>>(mods, a, b, o, (uint32_t)rows, lvl, n);
    LAUNCHED();
}

// automorphism sigma_t in evaluation form: E'[k] = E[pos[t z_k mod m]]
__global__ void k_automorph(NttTables T, const uint64_t *__restrict__ a, uint64_t *__restrict__ o,
                            uint32_t rows, uint32_t t) {
    const uint32_t xx = blockIdx.x * blockDim.x + threadIdx.x;
    if (xx >= T.n) return;
    const uint32_t src = (uint32_t)T.pos[(uint32_t)(((uint64_t)t * (uint32_t)T.z[xx]) % T.m)];
    ROW_LOOP(r, x, rows, T.n) o[(uint64_t)r * T.n + x] = a[(uint64_t)r * T.n + src];
}
// part 0 of each ciphertext of a (batch stride abs) -> o [B][1][lvl][n], permuted by sigma_t
__global__ void k_automorph_part(NttTables T, const uint64_t *__restrict__ a, uint64_t abs, uint64_t *__restrict__ o,
                                 uint32_t rows, uint32_t lvl, uint32_t t) {
    const uint32_t xx = blockIdx.x * blockDim.x + threadIdx.x;
    if (xx >= T.n) return;
    const uint32_t src = (uint32_t)T.pos[(uint32_t)(((uint64_t)t * (uint32_t)T.z[xx]) % T.m)];
    ROW_LOOP(rw, x, rows, T.n) {   // rows = B * lvl
        const uint32_t b = rw / lvl, r = rw - b * lvl;
        o[(uint64_t)rw * T.n + x] = a[(uint64_t)b * abs + (uint64_t)r * T.n + src];
    }
}
void ew_automorph_part(const NttTables &T, const uint64_t *a, uint64_t abs, uint64_t *o, uint32_t B, uint32_t lvl,
                       uint32_t t, cudaStream_t st) {
    const uint64_t rows = (uint64_t)B * lvl;
    k_automorph_part<<<grid_rows(T.n, rows), 256, 0, st>>>(T, a, abs, o, (uint32_t)rows, lvl, t);
    LAUNCHED();
}
void ew_automorph(const NttTables &T, const uint64_t *a, uint64_t *o, uint32_t B, uint32_t parts, uint32_t lvl,
                  uint32_t t, cudaStream_t st) {
    const uint64_t rows = (uint64_t)B * parts * lvl;
    k_automorph<<<grid_rows(T.n, rows), 256, 0, st>>>(T, a, o, (uint32_t)rows, t);
    LAUNCHED();
}

// copy parts [part0, part0+nparts) of a [B][parts_in][lvl_in][n] (first lvl_out limbs) into
// o [B][parts_out][lvl_out][n] at part opart0
__global__ void k_copy_parts(const uint64_t *__restrict__ a, uint64_t *__restrict__ o, uint32_t rows,
                             uint32_t parts_in, uint32_t part0, uint32_t nparts, uint32_t lvl_in,
                             uint32_t lvl_out, uint32_t n, uint32_t parts_out, uint32_t opart0) {
    ROW_LOOP(rw, x, rows, n) {   // rows = B * nparts * lvl_out
        const uint32_t limb = rw % lvl_out, r = rw / lvl_out;
        const uint32_t k = r % nparts;
        const uint64_t b = r / nparts;
        o[((b * parts_out + opart0 + k) * lvl_out + limb) * n + x] =
            a[((b * parts_in + part0 + k) * lvl_in + limb) * n + x];
    }
}
void ew_copy_parts(const uint64_t *a, uint64_t *o, uint32_t B, uint32_t parts_in, uint32_t part0, uint32_t nparts,
                   uint32_t lvl_in, uint32_t lvl_out, uint32_t n, uint32_t parts_out, uint32_t opart0,
                   cudaStream_t st) {
    const uint64_t rows = (uint64_t)B * nparts * lvl_out;
    k_copy_parts<<<grid_rows(n, rows), 256, 0, st>>>(a, o, (uint32_t)rows, parts_in, part0, nparts, lvl_in, lvl_out, n,
                                                      parts_out, opart0);
    LAUNCHED();
}

// =====================================================================================
// key switching: KIP and ModDown scaling
// =====================================================================================
// x < 2^(2b+4) (sums of up to 16 products of residues): Barrett estimate + correction loop
__device__ __forceinline__ uint64_t reduce128(uint64_t hi, uint64_t lo, const Mod &M) {
    const uint32_t s = M.b - 1, t = M.b + 1;
    const uint64_t x1 = (lo >> s) | (hi << (64 - s));
    const uint64_t plo = x1 * M.mu, phi = __umul64hi(x1, M.mu);
    const uint64_t qhat = (plo >> t) | (phi << (64 - t));
    uint64_t r = lo - qhat * M.q;
    while (r >= M.q) r -= M.q;
    return r;
}

__device__ __forceinline__ void mac128(uint64_t &hi, uint64_t &lo, uint64_t a, uint64_t b) {
    const uint64_t pl = a * b, ph = __umul64hi(a, b);
    lo += pl;
    hi += ph + (lo < pl ? 1 : 0);
}

__global__ void k_kip(const Mod *__restrict__ mods, const uint64_t *__restrict__ d, uint64_t dps,
                      const uint64_t *__restrict__ ext, const uint64_t *__restrict__ key,
                      uint64_t *__restrict__ u, uint32_t rows, uint32_t lvl, uint32_t K, uint32_t L1,
                      uint32_t alpha, uint32_t ndig, uint32_t n, const int32_t *__restrict__ pos,
                      const int32_t *__restrict__ zt, uint32_t m, uint32_t perm_t) {
    const uint32_t nl = lvl + K;
    const uint64_t ln = (uint64_t)nl * n;
    const uint32_t x0 = blockIdx.x * blockDim.x + threadIdx.x;
    if (x0 >= n) return;
    // R22: digits read through sigma_t's evaluation-index permutation
    const uint32_t x = perm_t ? (uint32_t)pos[(uint32_t)(((uint64_t)perm_t * (uint32_t)zt[x0]) % m)] : x0;
    ROW_LOOP(rw, xo, rows, n) {   // rows = B * nl
        const uint64_t b = rw / nl;
        const uint32_t r = rw - (uint32_t)b * nl;
        const uint64_t rr = (uint64_t)r * n + xo;
        const uint32_t kl = r < lvl ? r : L1 + (r - lvl);
        const Mod M = mods[kl];
        const uint32_t jr = r < lvl ? r / alpha : 0xffffffffu;
        uint64_t h0 = 0, l0 = 0, h1 = 0, l1 = 0;
        for (uint32_t j = 0; j < ndig; ++j) {
            const uint64_t dig = (j == jr) ? d[b * dps + (uint64_t)r * n + x] : ext[((b * ndig + j) * nl + r) * n + x];
            const uint64_t *kj = key + (uint64_t)j * 2 * (L1 + K) * n;
            mac128(h0, l0, dig, kj[(uint64_t)kl * n + xo]);
            mac128(h1, l1, dig, kj[(uint64_t)(L1 + K + kl) * n + xo]);
        }
        u[(b * 2 + 0) * ln + rr] = reduce128(h0, l0, M);
        u[(b * 2 + 1) * ln + rr] = reduce128(h1, l1, M);
    }
}
// binary64 variant: sum of 2 * ndig fmulv per output coefficient pair, one reduction each.
// NDIG > 0: the digit count is a compile-time constant (loop unrolled, all loads issued up front)
template <int NDIG>
__global__ void k_kip_f(const double2 *__restrict__ fm, const uint64_t *__restrict__ d, uint64_t dps,
                        const uint64_t *__restrict__ ext, const uint64_t *__restrict__ key,
                        uint64_t *__restrict__ u, uint32_t rows, uint32_t lvl, uint32_t K, uint32_t L1,
                        uint32_t alpha, uint32_t ndig, uint32_t n, const int32_t *__restrict__ pos,
                        const int32_t *__restrict__ zt, uint32_t m, uint32_t perm_t) {
    using namespace f64;
    const uint32_t nl = lvl + K;
    const uint64_t ln = (uint64_t)nl * n;
    const uint32_t x0 = blockIdx.x * blockDim.x + threadIdx.x;
    if (x0 >= n) return;
    const uint32_t x = perm_t ? (uint32_t)pos[(uint32_t)(((uint64_t)perm_t * (uint32_t)zt[x0]) % m)] : x0;
    ROW_LOOP(rw, xo, rows, n) {   // rows = B * nl
        const uint64_t b = rw / nl;
        const uint32_t r = rw - (uint32_t)b * nl;
        const uint64_t rr = (uint64_t)r * n + xo;
        const uint32_t kl = r < lvl ? r : L1 + (r - lvl);
        const double q = fm[kl].x, qi = fm[kl].y;
        const uint32_t jr = r < lvl ? r / alpha : 0xffffffffu;
        double s0 = 0.0, s1 = 0.0;      // |s| <= 0.75 q ndig (ndig <= 10: < 8q)
        const uint32_t nd = NDIG > 0 ? (uint32_t)NDIG : ndig;
#pragma unroll
        for (uint32_t j = 0; j < nd; ++j) {
            const uint64_t dig = (j == jr) ? d[b * dps + (uint64_t)r * n + x] : ext[((b * ndig + j) * nl + r) * n + x];
            const uint64_t *kj = key + (uint64_t)j * 2 * (L1 + K) * n;
            const double dg = from_u64(dig);
            s0 = __dadd_rn(s0, fmulv(dg, from_u64(kj[(uint64_t)kl * n + xo]), q, qi));
            s1 = __dadd_rn(s1, fmulv(dg, from_u64(kj[(uint64_t)(L1 + K + kl) * n + xo]), q, qi));
        }
        u[(b * 2 + 0) * ln + rr] = to_u64(fred(s0, q, qi), q);
        u[(b * 2 + 1) * ln + rr] = to_u64(fred(s1, q, qi), q);
    }
}
// batch-blocked variant: a thread keeps the 2 NDIG key words of its (limb, coefficient) in registers and
// applies them to BB ciphertexts of the batch (the key stream is read once per BB ciphertexts instead of
// once per ciphertext); sums in the same digit order, so the words are identical to k_kip_f's
template <int NDIG, int BB>
__global__ void __launch_bounds__(256) k_kip_fb(const double2 *__restrict__ fm, const uint64_t *__restrict__ d, uint64_t dps,
                                                const uint64_t *__restrict__ ext, const uint64_t *__restrict__ key,
                                                uint64_t *__restrict__ u, uint32_t B, uint32_t lvl, uint32_t K,
                                                uint32_t L1, uint32_t alpha, uint32_t n, const int32_t *__restrict__ pos,
                                                const int32_t *__restrict__ zt, uint32_t m, uint32_t perm_t) {
    using namespace f64;
    const uint32_t nl = lvl + K;
    const uint64_t ln = (uint64_t)nl * n;
    const uint32_t xo = blockIdx.x * blockDim.x + threadIdx.x;
    if (xo >= n) return;
    const uint32_t x = perm_t ? (uint32_t)pos[(uint32_t)(((uint64_t)perm_t * (uint32_t)zt[xo]) % m)] : xo;
    const uint32_t nbc = (B + BB - 1) / BB, rows = nl * nbc;
    for (uint32_t rw = blockIdx.y; rw < rows; rw += gridDim.y) {
        const uint32_t r = rw / nbc, b0 = (rw - r * nbc) * BB;
        const uint32_t kl = r < lvl ? r : L1 + (r - lvl);
        const double q = fm[kl].x, qi = fm[kl].y;
        const uint32_t jr = r < lvl ? r / alpha : 0xffffffffu;
        double k0[NDIG], k1[NDIG];
#pragma unroll
        for (int j = 0; j < NDIG; ++j) {
            const uint64_t *kj = key + (uint64_t)j * 2 * (L1 + K) * n;
            k0[j] = from_u64(__ldg(kj + (uint64_t)kl * n + xo));
            k1[j] = from_u64(__ldg(kj + (uint64_t)(L1 + K + kl) * n + xo));
        }
#pragma unroll
        for (int bb = 0; bb < BB; ++bb) {
            const uint64_t b = b0 + bb;
            if (b >= B) break;
            double s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int j = 0; j < NDIG; ++j) {
                const uint64_t dig = ((uint32_t)j == jr) ? __ldcs(d + b * dps + (uint64_t)r * n + x)
                                                         : __ldcs(ext + ((b * NDIG + j) * nl + r) * n + x);
                const double dg = from_u64(dig);
                s0 = __dadd_rn(s0, fmulv(dg, k0[j], q, qi));
                s1 = __dadd_rn(s1, fmulv(dg, k1[j], q, qi));
            }
            const uint64_t rr = (uint64_t)r * n + xo;
            __stcs(u + (b * 2 + 0) * ln + rr, to_u64(fred(s0, q, qi), q));
            __stcs(u + (b * 2 + 1) * ln + rr, to_u64(fred(s1, q, qi), q));
        }
    }
}

// the same with two coefficients per thread and 128-bit accesses (no automorphism on the digit reads:
// perm_t == 0, rows 16-byte aligned since n is even)
template <int NDIG, int BB>
__global__ void __launch_bounds__(256) k_kip_fb2(const double2 *__restrict__ fm, const uint64_t *__restrict__ d, uint64_t dps,
                                                 const uint64_t *__restrict__ ext, const uint64_t *__restrict__ key,
                                                 uint64_t *__restrict__ u, uint32_t B, uint32_t lvl, uint32_t K,
                                                 uint32_t L1, uint32_t alpha, uint32_t n) {
    using namespace f64;
    const uint32_t nl = lvl + K;
    const uint64_t ln = (uint64_t)nl * n;
    const uint32_t x = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (x >= n) return;
    const uint32_t nbc = (B + BB - 1) / BB, rows = nl * nbc;
    for (uint32_t rw = blockIdx.y; rw < rows; rw += gridDim.y) {
        const uint32_t r = rw / nbc, b0 = (rw - r * nbc) * BB;
        const uint32_t kl = r < lvl ? r : L1 + (r - lvl);
        const double q = fm[kl].x, qi = fm[kl].y;
        const uint32_t jr = r < lvl ? r / alpha : 0xffffffffu;
        double k0a[NDIG], k0b[NDIG], k1a[NDIG], k1b[NDIG];
#pragma unroll
        for (int j = 0; j < NDIG; ++j) {
            const uint64_t *kj = key + (uint64_t)j * 2 * (L1 + K) * n;
            const ulonglong2 w0 = __ldg((const ulonglong2 *)(kj + (uint64_t)kl * n + x));
            const ulonglong2 w1 = __ldg((const ulonglong2 *)(kj + (uint64_t)(L1 + K + kl) * n + x));
            k0a[j] = from_u64(w0.x); k0b[j] = from_u64(w0.y);
            k1a[j] = from_u64(w1.x); k1b[j] = from_u64(w1.y);
        }
#pragma unroll
        for (int bb = 0; bb < BB; ++bb) {
            const uint64_t b = b0 + bb;
            if (b >= B) break;
            double s0a = 0.0, s0b = 0.0, s1a = 0.0, s1b = 0.0;
#pragma unroll
            for (int j = 0; j < NDIG; ++j) {
                const uint64_t *src = ((uint32_t)j == jr) ? d + b * dps + (uint64_t)r * n
                                                          : ext + ((b * NDIG + j) * nl + r) * n;
                const ulonglong2 dg = __ldcs((const ulonglong2 *)(src + x));
                const double ga = from_u64(dg.x), gb = from_u64(dg.y);
                s0a = __dadd_rn(s0a, fmulv(ga, k0a[j], q, qi));
                s0b = __dadd_rn(s0b, fmulv(gb, k0b[j], q, qi));
                s1a = __dadd_rn(s1a, fmulv(ga, k1a[j], q, qi));
                s1b = __dadd_rn(s1b, fmulv(gb, k1b[j], q, qi));
            }
            const uint64_t rr = (uint64_t)r * n + x;
            __stcs((ulonglong2 *)(u + (b * 2 + 0) * ln + rr),
                   make_ulonglong2(to_u64(fred(s0a, q, qi), q), to_u64(fred(s0b, q, qi), q)));
            __stcs((ulonglong2 *)(u + (b * 2 + 1) * ln + rr),
                   make_ulonglong2(to_u64(fred(s1a, q, qi), q), to_u64(fred(s1b, q, qi), q)));
        }
    }
}

static void kip_f_dispatch(dim3 g, cudaStream_t st, const double2 *fm, const uint64_t *d, uint64_t dps,
                           const uint64_t *ext, const uint64_t *key, uint64_t *u, uint32_t rows, uint32_t lvl,
                           uint32_t K, uint32_t L1, uint32_t alpha, uint32_t ndig, uint32_t n, const int32_t *pos,
                           const int32_t *zt, uint32_t m, uint32_t perm_t) {
#define KIPF(N) k_kip_f<N><<<g, 256, 0, st>>>(fm, d, dps, ext, key, u, rows, lvl, K, L1, alpha, ndig, n, pos, zt, m, perm_t)
#define KIPB(N) k_kip_fb<N, 4><<<dim3(g.x, (unsigned)std::min<uint64_t>(65535, (uint64_t)(lvl + K) * ((B + 3) / 4))), 256, 0, st>>>( \
        fm, d, dps, ext, key, u, B, lvl, K, L1, alpha, n, pos, zt, m, perm_t)
    const uint32_t B = rows / (lvl + K);
#define KIPB2(N) k_kip_fb2<N, 4><<<dim3((n / 2 + 255) / 256, (unsigned)std::min<uint64_t>(65535, (uint64_t)(lvl + K) * ((B + 3) / 4))), 256, 0, st>>>( \
        fm, d, dps, ext, key, u, B, lvl, K, L1, alpha, n)
    if (g_kip_blocked == 1 && B >= 4 && perm_t == 0 && (n % 2) == 0 && (dps % 2) == 0) {
        switch (ndig) {
            case 1: KIPB2(1); return;
            case 2: KIPB2(2); return;
            case 3: KIPB2(3); return;
            case 4: KIPB2(4); return;
            default: break;
        }
    }
#undef KIPB2
    if (g_kip_blocked && B >= 4) {
        switch (ndig) {
            case 1: KIPB(1); return;
            case 2: KIPB(2); return;
            case 3: KIPB(3); return;
            case 4: KIPB(4); return;
            default: break;
        }
    }
#undef KIPB
    switch (ndig) {
        case 1: KIPF(1); break;
        case 2: KIPF(2); break;
        case 3: KIPF(3); break;
        case 4: KIPF(4); break;
        default: KIPF(0); break;
    }
#undef KIPF
}
void ks_kip(const Mod *mods, const uint64_t *d, uint64_t dps, const uint64_t *ext, const uint64_t *key, uint64_t *u,
            uint32_t B, uint32_t lvl, uint32_t K, uint32_t L1, uint32_t alpha, uint32_t ndig, uint32_t n, cudaStream_t st,
            const double2 *fm) {
    const uint64_t rows = (uint64_t)B * (lvl + K);
    if (fm && ndig <= 10)
        kip_f_dispatch(grid_rows(n, rows), st, fm, d, dps, ext, key, u, (uint32_t)rows, lvl, K, L1, alpha, ndig, n,
                       nullptr, nullptr, 1, 0);
    else
        k_kip<<<grid_rows(n, rows), 256, 0, st>>>(mods, d, dps, ext, key, u, (uint32_t)rows, lvl, K, L1, alpha, ndig, n,
                                                  nullptr, nullptr, 1, 0);
    LAUNCHED();
}
void ks_kip_perm(const Mod *mods, const NttTables &T, uint32_t perm_t, const uint64_t *d, uint64_t dps,
                 const uint64_t *ext, const uint64_t *key, uint64_t *u, uint32_t B, uint32_t lvl, uint32_t K, uint32_t L1,
                 uint32_t alpha, uint32_t ndig, uint32_t n, cudaStream_t st, const double2 *fm) {
    const uint64_t rows = (uint64_t)B * (lvl + K);
    if (fm && ndig <= 10)
        kip_f_dispatch(grid_rows(n, rows), st, fm, d, dps, ext, key, u, (uint32_t)rows, lvl, K, L1, alpha, ndig, n,
                       T.pos, T.z, T.m, perm_t);
    else
        k_kip<<<grid_rows(n, rows), 256, 0, st>>>(mods, d, dps, ext, key, u, (uint32_t)rows, lvl, K, L1, alpha, ndig, n,
                                                  T.pos, T.z, T.m, perm_t);
    LAUNCHED();
}

// o[b] = a[b] + b[b] over parts x lvl x n words per ciphertext, with per-operand batch strides
__global__ void k_add_bs(const Mod *__restrict__ mods, const uint64_t *__restrict__ a, uint64_t abs,
                         const uint64_t *__restrict__ b, uint64_t bbs, uint64_t *__restrict__ o, uint64_t obs,
                         uint32_t rows, uint32_t per_rows, uint32_t lvl, uint32_t n) {
    ROW_LOOP(rw, x, rows, n) {   // rows = B * parts * lvl
        const uint32_t bi = rw / per_rows, rr = rw - bi * per_rows;
        const uint64_t r = (uint64_t)rr * n + x;
        o[bi * obs + r] = add_mod(a[bi * abs + r], b[bi * bbs + r], mods[rr % lvl].q);
    }
}
void ew_add_bs(const Mod *mods, const uint64_t *a, uint64_t abs, const uint64_t *b, uint64_t bbs, uint64_t *o,
               uint64_t obs, uint32_t B, uint32_t parts, uint32_t lvl, uint32_t n, cudaStream_t st) {
    const uint64_t rows = (uint64_t)B * parts * lvl;
    k_add_bs<<<grid_rows(n, rows), 256, 0, st>>>(mods, a, abs, b, bbs, o, obs, (uint32_t)rows, parts * lvl, lvl, n);
    LAUNCHED();
}

__global__ void k_scale_sub(const Mod *__restrict__ mods, const uint64_t *__restrict__ u, uint64_t u_pstride,
                            const uint64_t *__restrict__ delta, const u64x2 *__restrict__ inv,
                            uint64_t *__restrict__ o, uint32_t rows, uint32_t lvl, uint32_t n) {
    ROW_LOOP2(rw, x, rows, n) {   // rows = npoly * lvl
        const uint32_t pidx = rw / lvl, limb = rw - pidx * lvl;
        const uint64_t rr = (uint64_t)limb * n + x, i = (uint64_t)rw * n + x;
        const uint64_t q = mods[limb].q;
        const ulonglong2 uv = LD2(u + (uint64_t)pidx * u_pstride + rr), dv = LD2(delta + i);
        const u64x2 w = inv[limb];
        ST2(o + i, mul_shoup(sub_mod(uv.x, dv.x, q), w.w, w.ws, q), mul_shoup(sub_mod(uv.y, dv.y, q), w.w, w.ws, q));
    }
}
void ew_scale_sub(const Mod *mods, const uint64_t *u, uint64_t u_pstride, const uint64_t *delta, const u64x2 *inv,
                  uint64_t *o, uint32_t npoly, uint32_t lvl, uint32_t n, cudaStream_t st) {
    const uint64_t rows = (uint64_t)npoly * lvl;
    k_scale_sub<<<grid_rows(n / 2, rows), 256, 0, st>>>(mods, u, u_pstride, delta, inv, o, (uint32_t)rows, lvl, n);
    LAUNCHED();
}

// fused ModDown + modulus switch (R15): u[b][k][i] += Pm_i d_k[i] on limb `limb` only (before its INTT)
__global__ void k_axpy_limb(const Mod *__restrict__ mods, uint64_t *__restrict__ u, uint64_t u_pstride,
                            const uint64_t *__restrict__ d, uint64_t d_bstride, uint64_t d_kstride,
                            const u64x2 *__restrict__ pm, uint32_t limb, uint32_t rows, uint32_t n) {
    const uint64_t q = mods[limb].q;
    const u64x2 w = pm[limb];
    ROW_LOOP(poly, x, rows, n) {      // poly = b * 2 + k
        const uint64_t b = poly >> 1, k = poly & 1;
        uint64_t *pu = u + poly * u_pstride + (uint64_t)limb * n + x;
        const uint64_t dv = d[b * d_bstride + k * d_kstride + (uint64_t)limb * n + x];
        *pu = add_mod(*pu, mul_shoup(dv, w.w, w.ws, q), q);
    }
}
// out[b][k][i] = (u[b][k][i] + Pm_i d_k[i] - delta[b][k][i]) Dinv_i, i < lvl (= level - 1)
__global__ void k_fused_down(const Mod *__restrict__ mods, const uint64_t *__restrict__ u, uint64_t u_pstride,
                             const uint64_t *__restrict__ d, uint64_t d_bstride, uint64_t d_kstride,
                             const uint64_t *__restrict__ delta, const u64x2 *__restrict__ pm,
                             const u64x2 *__restrict__ dinv, uint64_t *__restrict__ o, uint32_t rows, uint32_t lvl,
                             uint32_t n) {
    ROW_LOOP2(rw, x, rows, n) {   // rows = 2B * lvl
        const uint64_t poly = rw / lvl;
        const uint32_t limb = rw - (uint32_t)poly * lvl;
        const uint64_t rr = (uint64_t)limb * n + x, i = (uint64_t)rw * n + x;
        const uint64_t b = poly >> 1, k = poly & 1;
        const uint64_t q = mods[limb].q;
        const u64x2 w = pm[limb], v = dinv[limb];
        const ulonglong2 dv = LD2(d + b * d_bstride + k * d_kstride + rr), uv = LD2(u + poly * u_pstride + rr);
        const ulonglong2 de = LD2(delta + i);
        const uint64_t x0 = sub_mod(add_mod(uv.x, mul_shoup(dv.x, w.w, w.ws, q), q), de.x, q);
        const uint64_t x1 = sub_mod(add_mod(uv.y, mul_shoup(dv.y, w.w, w.ws, q), q), de.y, q);
        ST2(o + i, mul_shoup(x0, v.w, v.ws, q), mul_shoup(x1, v.w, v.ws, q));
    }
}
void ew_fused_down(const Mod *mods, uint64_t *u, uint64_t u_pstride, const uint64_t *d, uint64_t d_bstride,
                   uint64_t d_kstride, const uint64_t *delta, const u64x2 *pm, const u64x2 *dinv, uint64_t *o,
                   uint32_t B, uint32_t level, uint32_t n, cudaStream_t st) {
    k_axpy_limb<<<grid_rows(n, 2ull * B), 256, 0, st>>>(mods, u, u_pstride, d, d_bstride, d_kstride, pm, level - 1, 2 * B, n);
    LAUNCHED();
    (void)delta; (void)dinv; (void)o;
}
void ew_fused_down_out(const Mod *mods, const uint64_t *u, uint64_t u_pstride, const uint64_t *d, uint64_t d_bstride,
                       uint64_t d_kstride, const uint64_t *delta, const u64x2 *pm, const u64x2 *dinv, uint64_t *o,
                       uint32_t B, uint32_t lvl_out, uint32_t n, cudaStream_t st) {
    const uint64_t rows = (uint64_t)2 * B * lvl_out;
    k_fused_down<<<grid_rows(n / 2, rows), 256, 0, st>>>(mods, u, u_pstride, d, d_bstride, d_kstride, delta, pm, dinv,
                                                     o, (uint32_t)rows, lvl_out, n);
    LAUNCHED();
}

// =====================================================================================
// exact centered CRT lift (Garner mixed radix + lexicographic sign test)
// plan blob (u64 words): [0]=ns [1]=nt, then
//   src[ns] inv[ns] invs[ns] qm[ns*ns] qms[ns*ns] half[ns] tgt[nt] B[nt*ns] Bs[nt*ns] Qm[nt] Qms[nt] pmu
// tgt[t] = prime index, or ~0 for the plaintext modulus p.  All constant products use Shoup
// companions (lazy outputs < 2T), one Barrett reduction per target.
// =====================================================================================
__device__ __forceinline__ uint64_t mod_small(uint64_t v, uint32_t p, uint64_t pmu) {
    uint64_t r = v - __umul64hi(v, pmu) * p;
    return r >= p ? r - p : r;
}

template <int MAXS>
__global__ void k_lift(const uint64_t *__restrict__ plan, const Mod *__restrict__ mods, uint32_t p,
                       const uint64_t *__restrict__ src, uint64_t src_pstride, uint64_t *__restrict__ out,
                       uint64_t out_pstride, int16_t *__restrict__ out16, uint64_t total, uint32_t n,
                       uint32_t skip0, uint32_t skipn, int mode) {
    const uint32_t ns = (uint32_t)plan[0], nt = (uint32_t)plan[1];
    const uint64_t *P_src = plan + 2, *P_inv = P_src + ns, *P_invs = P_inv + ns, *P_qm = P_invs + ns;
    const uint64_t *P_qms = P_qm + ns * ns, *P_half = P_qms + ns * ns, *P_tgt = P_half + ns;
    const uint64_t *P_B = P_tgt + nt, *P_Bs = P_B + (uint64_t)nt * ns, *P_Q = P_Bs + (uint64_t)nt * ns;
    const uint64_t *P_Qs = P_Q + nt;
    const uint64_t pmu = P_Qs[nt];
    GRID_LOOP(i, total) {
        const uint64_t poly = i / n;
        const uint32_t x = (uint32_t)(i - poly * n);
        const uint64_t *s = src + poly * src_pstride + x;
        uint64_t v[MAXS];
        for (uint32_t k = 0; k < ns; ++k) {
            const uint64_t xk = s[(uint64_t)k * n];
            if (k == 0) { v[0] = xk; continue; }
            const Mod Mk = mods[P_src[k]];
            uint64_t acc = v[k - 1];
            for (int j = (int)k - 2; j >= 0; --j)
                acc = mul_shoup_lazy(acc, P_qm[k * ns + j], P_qms[k * ns + j], Mk.q) + v[j];
            acc = reduce64(acc, Mk);
            v[k] = mul_shoup(sub_mod(xk, acc, Mk.q), P_inv[k], P_invs[k], Mk.q);
        }
        bool neg = false;
        for (int k = (int)ns - 1; k >= 0; --k) {
            if (v[k] != P_half[k]) { neg = v[k] > P_half[k]; break; }
        }
        if (mode == 0) {
            for (uint32_t t = 0; t < nt; ++t) {
                const Mod Mt = mods[P_tgt[t]];
                const uint64_t *B = P_B + (uint64_t)t * ns, *Bs = P_Bs + (uint64_t)t * ns;
                uint64_t acc = 0;
                for (uint32_t k = 0; k < ns; ++k) acc += mul_shoup_lazy(v[k], B[k], Bs[k], Mt.q);
                acc = reduce64(acc, Mt);
                if (neg) acc = sub_mod(acc, P_Q[t], Mt.q);
                const uint32_t lb = t < skip0 ? t : t + skipn;
                out[poly * out_pstride + (uint64_t)lb * n + x] = acc;
            }
        } else {
            // value mod p (last target in mode 1, only target in mode 2)
            const uint32_t tp = nt - 1;
            uint64_t rp = 0;
            for (uint32_t k = 0; k < ns; ++k) rp += mod_small(v[k], p, pmu) * P_B[(uint64_t)tp * ns + k];
            rp %= p;
            if (neg) rp = (rp + p - P_Q[tp]) % p;
            if (mode == 2) {
                int32_t c = (int32_t)rp;
                if (c > (int32_t)(p / 2)) c -= (int32_t)p;
                out16[poly * n + x] = (int16_t)c;
                continue;
            }
            // delta = r + Q * [-r]_p
            int64_t tc = (int64_t)((p - rp) % p);
            if (tc > (int64_t)(p / 2)) tc -= p;
            const uint64_t atc = (uint64_t)(tc < 0 ? -tc : tc);
            for (uint32_t t = 0; t + 1 < nt; ++t) {
                const Mod Mt = mods[P_tgt[t]];
                const uint64_t *B = P_B + (uint64_t)t * ns, *Bs = P_Bs + (uint64_t)t * ns;
                uint64_t acc = 0;
                for (uint32_t k = 0; k < ns; ++k) acc += mul_shoup_lazy(v[k], B[k], Bs[k], Mt.q);
                acc = reduce64(acc, Mt);
                if (neg) acc = sub_mod(acc, P_Q[t], Mt.q);
                const uint64_t qc = mul_shoup(atc, P_Q[t], P_Qs[t], Mt.q);     // (Q mod T) |c|
                acc = tc < 0 ? sub_mod(acc, qc, Mt.q) : add_mod(acc, qc, Mt.q);
                out[poly * out_pstride + (uint64_t)t * n + x] = acc;
            }
        }
    }
}
// Specialised lift for a compile-time source count NS (digits in registers, fully unrolled Garner)
// with the plan staged in shared memory once per block.  Same arithmetic as k_lift (modes 0, 1).
template <int NS>
__global__ void __launch_bounds__(256) k_lift_ns(const uint64_t *__restrict__ plan, const Mod *__restrict__ mods,
                                                 uint32_t p, const uint64_t *__restrict__ src, uint64_t src_pstride,
                                                 uint64_t *__restrict__ out, uint64_t out_pstride, uint64_t total,
                                                 uint32_t n, uint32_t skip0, uint32_t skipn, int mode) {
    __shared__ uint64_t sp[1024];
    __shared__ Mod smod[64];
    const uint32_t nt = (uint32_t)plan[1];
    const uint32_t words = 2 + 3 * NS + 2 * NS * NS + NS + nt + 2 * nt * NS + 2 * nt + 1;
    for (uint32_t i = threadIdx.x; i < words && i < 1024; i += blockDim.x) sp[i] = plan[i];
    __syncthreads();
    const uint64_t *P_src = sp + 2, *P_inv = P_src + NS, *P_invs = P_inv + NS, *P_qm = P_invs + NS;
    const uint64_t *P_qms = P_qm + NS * NS, *P_half = P_qms + NS * NS, *P_tgt = P_half + NS;
    const uint64_t *P_B = P_tgt + nt, *P_Bs = P_B + (uint64_t)nt * NS, *P_Q = P_Bs + (uint64_t)nt * NS;
    const uint64_t *P_Qs = P_Q + nt;
    const uint64_t pmu = P_Qs[nt];
    for (uint32_t t = threadIdx.x; t < nt && t < 64; t += blockDim.x)
        smod[t] = P_tgt[t] == ~0ull ? Mod{p, 0, 0, 0} : mods[P_tgt[t]];
    __shared__ Mod ssrc[NS];
    if (threadIdx.x < NS) ssrc[threadIdx.x] = mods[P_src[threadIdx.x]];
    __syncthreads();
    const uint32_t npoly = (uint32_t)(total / n);
    ROW_LOOP(poly, x, npoly, n) {
        const uint64_t *s = src + (uint64_t)poly * src_pstride + x;
        uint64_t v[NS];
#pragma unroll
        for (int k = 0; k < NS; ++k) v[k] = __ldcs(s + (uint64_t)k * n);
#pragma unroll
        for (int k = 1; k < NS; ++k) {
            const uint64_t qk = ssrc[k].q;
            uint64_t acc = v[k - 1];
#pragma unroll
            for (int j = k - 2; j >= 0; --j) acc = mul_shoup_lazy(acc, P_qm[k * NS + j], P_qms[k * NS + j], qk) + v[j];
            acc = reduce64(acc, ssrc[k]);
            v[k] = mul_shoup(sub_mod(v[k], acc, qk), P_inv[k], P_invs[k], qk);
        }
        bool neg = false;
#pragma unroll
        for (int k = NS - 1; k >= 0; --k) {
            if (v[k] != P_half[k]) { neg = v[k] > P_half[k]; break; }
        }
        int64_t tc = 0;
        if (mode == 1) {
            const uint32_t tp = nt - 1;
            uint64_t rp = 0;
#pragma unroll
            for (int k = 0; k < NS; ++k) rp += mod_small(v[k], p, pmu) * P_B[(uint64_t)tp * NS + k];
            rp %= p;
            if (neg) rp = (rp + p - P_Q[tp]) % p;
            tc = (int64_t)((p - rp) % p);
            if (tc > (int64_t)(p / 2)) tc -= p;
        }
        const uint64_t atc = (uint64_t)(tc < 0 ? -tc : tc);
        const uint32_t ntw = mode == 1 ? nt - 1 : nt;
        for (uint32_t t = 0; t < ntw; ++t) {
            const Mod Mt = smod[t];
            const uint64_t *B = P_B + (uint64_t)t * NS, *Bs = P_Bs + (uint64_t)t * NS;
            uint64_t acc = 0;
#pragma unroll
            for (int k = 0; k < NS; ++k) acc += mul_shoup_lazy(v[k], B[k], Bs[k], Mt.q);
            acc = reduce64(acc, Mt);
            if (neg) acc = sub_mod(acc, P_Q[t], Mt.q);
            if (mode == 1) {
                const uint64_t qc = mul_shoup(atc, P_Q[t], P_Qs[t], Mt.q);
                acc = tc < 0 ? sub_mod(acc, qc, Mt.q) : add_mod(acc, qc, Mt.q);
                out[(uint64_t)poly * out_pstride + (uint64_t)t * n + x] = acc;
            } else {
                const uint32_t lb = t < skip0 ? t : t + skipn;
                out[(uint64_t)poly * out_pstride + (uint64_t)lb * n + x] = acc;
            }
        }
    }
}

// Binary64 lift (all primes in [2^49, 2^50), so every source digit is < 2 q_t of any target):
// same plan and the same exact result as k_lift_ns (modes 0, 1).  Garner digits are made canonical
// (they decide the sign test), the target sums use one fmm per digit (B[t][0] = 1 needs none).
template <int NS>
__global__ void __launch_bounds__(256) k_lift_f(const uint64_t *__restrict__ plan, const double2 *__restrict__ fm,
                                                uint32_t p, const uint64_t *__restrict__ src, uint64_t src_pstride,
                                                uint64_t *__restrict__ out, uint64_t out_pstride, uint32_t npoly,
                                                uint32_t n, uint32_t skip0, uint32_t skipn, int mode) {
    using namespace f64;
    __shared__ double2 sB[64 * NS], sQ[64], sT[64], sqm[NS * NS], sinv[NS], ssrc[NS];
    __shared__ double shalf[NS];
    __shared__ uint64_t sBp[NS];
    const uint32_t nt = (uint32_t)plan[1];
    const uint64_t *P_src = plan + 2, *P_inv = P_src + NS, *P_invs = P_inv + NS, *P_qm = P_invs + NS;
    const uint64_t *P_qms = P_qm + NS * NS, *P_half = P_qms + NS * NS, *P_tgt = P_half + NS;
    const uint64_t *P_B = P_tgt + nt, *P_Bs = P_B + (uint64_t)nt * NS, *P_Q = P_Bs + (uint64_t)nt * NS;
    const uint64_t *P_Qs = P_Q + nt;
    const uint64_t pmu = P_Qs[nt];
    const uint32_t ntq = mode == 1 ? nt - 1 : nt;       // prime targets (mode 1: the last target is p)
    for (uint32_t i = threadIdx.x; i < ntq * NS; i += blockDim.x) {
        const uint32_t t = i / NS;
        const uint64_t qt = (uint64_t)fm[P_tgt[t]].x;
        sB[i] = centred_entry(P_B[i], qt);
    }
    for (uint32_t t = threadIdx.x; t < ntq; t += blockDim.x) {
        sT[t] = fm[P_tgt[t]];
        const uint64_t qt = (uint64_t)sT[t].x;
        sQ[t] = centred_entry(P_Q[t], qt);
    }
    if (threadIdx.x < NS) {
        const uint32_t k = threadIdx.x;
        ssrc[k] = fm[P_src[k]];
        const uint64_t qk = (uint64_t)ssrc[k].x;
        sinv[k] = centred_entry(P_inv[k], qk);
        shalf[k] = (double)P_half[k];
        for (uint32_t j = 0; j < NS; ++j) sqm[k * NS + j] = centred_entry(P_qm[k * NS + j], qk);
        if (mode == 1) sBp[k] = P_B[(uint64_t)(nt - 1) * NS + k];
    }
    __syncthreads();
    ROW_LOOP(poly, x, npoly, n) {
        const uint64_t *s = src + (uint64_t)poly * src_pstride + x;
        double v[NS];
#pragma unroll
        for (int k = 0; k < NS; ++k) v[k] = from_u64(__ldcs(s + (uint64_t)k * n));
#pragma unroll
        for (int k = 1; k < NS; ++k) {
            const double qk = ssrc[k].x;
            double acc = v[k - 1];                               // < 2 q_k
#pragma unroll
            for (int j = k - 2; j >= 0; --j) acc = __dadd_rn(fmm(acc, sqm[k * NS + j], qk), v[j]);   // < 2.625 q_k
            v[k] = canon(fmm(__dsub_rn(v[k], acc), sinv[k], qk), qk);
        }
        bool neg = false;
#pragma unroll
        for (int k = NS - 1; k >= 0; --k) {
            if (v[k] != shalf[k]) { neg = v[k] > shalf[k]; break; }
        }
        double tcd = 0.0;
        if (mode == 1) {
            uint64_t rp = 0;
#pragma unroll
            for (int k = 0; k < NS; ++k) {
                const uint64_t vk = (uint64_t)v[k];
                rp += mod_small(vk, p, pmu) * sBp[k];
            }
            rp %= p;
            if (neg) rp = (rp + p - P_Q[nt - 1]) % p;
            int64_t tc = (int64_t)((p - rp) % p);
            if (tc > (int64_t)(p / 2)) tc -= p;
            tcd = (double)tc;
        }
        for (uint32_t t = 0; t < ntq; ++t) {
            const double qt = sT[t].x, qit = sT[t].y;
            const double2 *B = sB + t * NS;
            double acc = v[0];                                   // B[t][0] = 1
#pragma unroll
            for (int k = 1; k < NS; ++k) {
                // < (2 + 0.625 (k-1)) q_t before term k; one reduction after 8 terms keeps the sum
                // exact for NS <= 16: |fred| <= q/2 + 2, then < (0.5 + 0.625 (NS-9)) q_t + ...
                if (k == 8) acc = fred(acc, qt, qit);
                acc = __dadd_rn(acc, fmm(v[k], B[k], qt));
            }
            if (neg) acc = __dsub_rn(acc, sQ[t].x);
            if (mode == 1) acc = __dadd_rn(acc, fmm(tcd, sQ[t], qt));   // |tc| <= p/2 <= 4q; sum < 7.5 q_t
            const uint64_t r = to_u64(fred(acc, qt, qit), qt);
            const uint32_t lb = (mode == 1 || t < skip0) ? t : t + skipn;
            out[(uint64_t)poly * out_pstride + (uint64_t)lb * n + x] = r;
        }
    }
}

// the same lift for two adjacent coefficients per thread (128-bit loads / stores; the two Garner chains
// interleave, which the one-coefficient kernel's dependent chain cannot): identical words
template <int NS>
__global__ void __launch_bounds__(256) k_lift_f2(const uint64_t *__restrict__ plan, const double2 *__restrict__ fm,
                                                 uint32_t p, const uint64_t *__restrict__ src, uint64_t src_pstride,
                                                 uint64_t *__restrict__ out, uint64_t out_pstride, uint32_t npoly,
                                                 uint32_t n, uint32_t skip0, uint32_t skipn, int mode) {
    using namespace f64;
    __shared__ double2 sB[64 * NS], sQ[64], sT[64], sqm[NS * NS], sinv[NS], ssrc[NS];
    __shared__ double shalf[NS];
    __shared__ uint64_t sBp[NS];
    const uint32_t nt = (uint32_t)plan[1];
    const uint64_t *P_src = plan + 2, *P_inv = P_src + NS, *P_invs = P_inv + NS, *P_qm = P_invs + NS;
    const uint64_t *P_qms = P_qm + NS * NS, *P_half = P_qms + NS * NS, *P_tgt = P_half + NS;
    const uint64_t *P_B = P_tgt + nt, *P_Bs = P_B + (uint64_t)nt * NS, *P_Q = P_Bs + (uint64_t)nt * NS;
    const uint64_t *P_Qs = P_Q + nt;
    const uint64_t pmu = P_Qs[nt];
    const uint32_t ntq = mode == 1 ? nt - 1 : nt;
    for (uint32_t i = threadIdx.x; i < ntq * NS; i += blockDim.x) {
        const uint32_t t = i / NS;
        sB[i] = centred_entry(P_B[i], (uint64_t)fm[P_tgt[t]].x);
    }
    for (uint32_t t = threadIdx.x; t < ntq; t += blockDim.x) {
        sT[t] = fm[P_tgt[t]];
        sQ[t] = centred_entry(P_Q[t], (uint64_t)sT[t].x);
    }
    if (threadIdx.x < NS) {
        const uint32_t kk = threadIdx.x;
        ssrc[kk] = fm[P_src[kk]];
        const uint64_t qk = (uint64_t)ssrc[kk].x;
        sinv[kk] = centred_entry(P_inv[kk], qk);
        shalf[kk] = (double)P_half[kk];
        for (uint32_t j = 0; j < NS; ++j) sqm[kk * NS + j] = centred_entry(P_qm[kk * NS + j], qk);
        if (mode == 1) sBp[kk] = P_B[(uint64_t)(nt - 1) * NS + kk];
    }
    __syncthreads();
    ROW_LOOP2(poly, x, npoly, n) {
        const uint64_t *s = src + (uint64_t)poly * src_pstride + x;
        double v[2][NS];
#pragma unroll
        for (int kk = 0; kk < NS; ++kk) {
            const ulonglong2 w = __ldcs((const ulonglong2 *)(s + (uint64_t)kk * n));
            v[0][kk] = from_u64(w.x);
            v[1][kk] = from_u64(w.y);
        }
#pragma unroll
        for (int kk = 1; kk < NS; ++kk) {
            const double qk = ssrc[kk].x;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                double acc = v[h][kk - 1];
#pragma unroll
                for (int j = kk - 2; j >= 0; --j) acc = __dadd_rn(fmm(acc, sqm[kk * NS + j], qk), v[h][j]);
                v[h][kk] = canon(fmm(__dsub_rn(v[h][kk], acc), sinv[kk], qk), qk);
            }
        }
        bool neg[2];
        double tcd[2] = {0.0, 0.0};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            neg[h] = false;
#pragma unroll
            for (int kk = NS - 1; kk >= 0; --kk) {
                if (v[h][kk] != shalf[kk]) { neg[h] = v[h][kk] > shalf[kk]; break; }
            }
            if (mode == 1) {
                uint64_t rp = 0;
#pragma unroll
                for (int kk = 0; kk < NS; ++kk) rp += mod_small((uint64_t)v[h][kk], p, pmu) * sBp[kk];
                rp %= p;
                if (neg[h]) rp = (rp + p - P_Q[nt - 1]) % p;
                int64_t tc = (int64_t)((p - rp) % p);
                if (tc > (int64_t)(p / 2)) tc -= p;
                tcd[h] = (double)tc;
            }
        }
        for (uint32_t t = 0; t < ntq; ++t) {
            const double qt = sT[t].x, qit = sT[t].y;
            const double2 *B = sB + t * NS;
            uint64_t r[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                double acc = v[h][0];
#pragma unroll
                for (int kk = 1; kk < NS; ++kk) {
                    if (kk == 8) acc = fred(acc, qt, qit);
                    acc = __dadd_rn(acc, fmm(v[h][kk], B[kk], qt));
                }
                if (neg[h]) acc = __dsub_rn(acc, sQ[t].x);
                if (mode == 1) acc = __dadd_rn(acc, fmm(tcd[h], sQ[t], qt));
                r[h] = to_u64(fred(acc, qt, qit), qt);
            }
            const uint32_t lb = (mode == 1 || t < skip0) ? t : t + skipn;
            ST2(out + (uint64_t)poly * out_pstride + (uint64_t)lb * n + x, r[0], r[1]);
        }
    }
}

void lift(const uint64_t *plan, const Mod *mods, uint32_t p, const uint64_t *src, uint64_t src_pstride, uint64_t *out,
          uint64_t out_pstride, int16_t *out16, uint32_t npoly, uint32_t n, uint32_t skip0, uint32_t skipn, int mode,
          cudaStream_t st, uint32_t ns_hint, uint32_t nt_hint, const double2 *fm) {
    const bool two = g_lift2 && (n % 2) == 0 && (src_pstride % 2) == 0 && (out_pstride % 2) == 0 &&
                     (((uintptr_t)src | (uintptr_t)out) & 15) == 0;
    if (fm && mode != 2 && ns_hint >= 1 && ns_hint <= 16 && nt_hint <= 64 && two) {
        dim3 g = grid_rows(n / 2, npoly);
        // each block sets up its constant tables (a barrier) before its rows: cap the row blocks so a block
        // loops over several polys (ROW_LOOP2 strides by gridDim.y) and the setup is amortised
        if (g_lift_blocks > 0) g.y = std::max<unsigned>(1, std::min<unsigned>(g.y, (unsigned)(148u * g_lift_blocks / g.x)));
#define LIFT_F2(K) case K: k_lift_f2<K><<<g, 256, 0, st>>>(plan, fm, p, src, src_pstride, out, out_pstride, npoly, n, skip0, skipn, mode); break;
        switch (ns_hint) { LIFT_F2(1) LIFT_F2(2) LIFT_F2(3) LIFT_F2(4) LIFT_F2(5) LIFT_F2(6) LIFT_F2(7) LIFT_F2(8)
                           LIFT_F2(9) LIFT_F2(10) LIFT_F2(11) LIFT_F2(12) LIFT_F2(13) LIFT_F2(14) LIFT_F2(15) LIFT_F2(16) }
#undef LIFT_F2
        LAUNCHED();
        return;
    }
    if (fm && mode != 2 && ns_hint >= 1 && ns_hint <= 16 && nt_hint <= 64) {
        dim3 g = grid_rows(n, npoly);
        if (g_lift_blocks > 0) g.y = std::max<unsigned>(1, std::min<unsigned>(g.y, (unsigned)(148u * g_lift_blocks / g.x)));
#define LIFT_F(K) case K: k_lift_f<K><<<g, 256, 0, st>>>(plan, fm, p, src, src_pstride, out, out_pstride, npoly, n, skip0, skipn, mode); break;
        switch (ns_hint) { LIFT_F(1) LIFT_F(2) LIFT_F(3) LIFT_F(4) LIFT_F(5) LIFT_F(6) LIFT_F(7) LIFT_F(8)
                           LIFT_F(9) LIFT_F(10) LIFT_F(11) LIFT_F(12) LIFT_F(13) LIFT_F(14) LIFT_F(15) LIFT_F(16) }
#undef LIFT_F
        LAUNCHED();
        return;
    }
    const uint64_t total = (uint64_t)npoly * n;
    const uint32_t words = 2 + 3 * ns_hint + 2 * ns_hint * ns_hint + ns_hint + nt_hint + 2 * nt_hint * ns_hint + 2 * nt_hint + 1;
    if (mode != 2 && ns_hint >= 1 && ns_hint <= 8 && nt_hint <= 64 && words <= 1024) {
        const dim3 g = grid_rows(n, npoly);
#define LIFT_NS(K) case K: k_lift_ns<K><<<g, 256, 0, st>>>(plan, mods, p, src, src_pstride, out, out_pstride, total, n, skip0, skipn, mode); break;
        switch (ns_hint) { LIFT_NS(1) LIFT_NS(2) LIFT_NS(3) LIFT_NS(4) LIFT_NS(5) LIFT_NS(6) LIFT_NS(7) LIFT_NS(8) }
#undef LIFT_NS
        LAUNCHED();
        return;
    }
    if (mode == 2)
        k_lift<64><<<grid_for(total, 128), 128, 0, st>>>(plan, mods, p, src, src_pstride, out, out_pstride, out16,
                                                         total, n, skip0, skipn, mode);
    else
        k_lift<32><<<grid_for(total, 256), 256, 0, st>>>(plan, mods, p, src, src_pstride, out, out_pstride, out16,
                                                         total, n, skip0, skipn, mode);   // ns <= 32 (lift_p checks)
    LAUNCHED();
}

// =====================================================================================
// counter-based sampler (R7)
// =====================================================================================
#define C_TAG 0xD1B54A32D192ED03ull
#define C_STREAM 0x8CB92BA72F3D8DD7ull
#define C_GOLD 0x9E3779B97F4A7C15ull
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27; z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}
__device__ __forceinline__ uint64_t draw(uint64_t seed, uint32_t tag, uint64_t stream, uint64_t j) {
    return mix64(seed + (uint64_t)tag * C_TAG + stream * C_STREAM + (j + 1) * C_GOLD);
}

__global__ void k_sample_small(const Mod *__restrict__ mods, uint64_t seed, uint32_t tag, uint64_t stream0,
                               uint64_t stream_step, int kind, int64_t mult, const int16_t *__restrict__ add16,
                               uint64_t *__restrict__ out, uint64_t total, uint32_t nl, uint32_t prime0,
                               uint32_t n, uint64_t pstride) {
    GRID_LOOP(i, total) {   // over npoly * n
        const uint64_t poly = i / n;
        const uint32_t x = (uint32_t)(i - poly * n);
        int64_t v = 0;
        if (kind >= 0) {
            const uint64_t r = draw(seed, tag, stream0 + poly * stream_step, x);
            if (kind == 0) v = (int64_t)(r % 3) - 1;
            else v = (int64_t)__popcll(r & 0x1FFFFFull) - (int64_t)__popcll((r >> 21) & 0x1FFFFFull);
            v *= mult;
        }
        if (add16) v += add16[i];
        for (uint32_t l = 0; l < nl; ++l)
            out[poly * pstride + (uint64_t)l * n + x] = from_signed(v, mods[prime0 + l].q);
    }
}
void sample_small(const Mod *mods, uint64_t seed, uint32_t tag, uint64_t stream0, uint64_t stream_step, int kind,
                  int64_t mult, const int16_t *add16, uint64_t *out, uint32_t npoly, uint32_t nl, uint32_t prime0,
                  uint32_t n, uint64_t pstride, cudaStream_t st) {
    const uint64_t total = (uint64_t)npoly * n;
    k_sample_small<<<grid_for(total, 256), 256, 0, st>>>(mods, seed, tag, stream0, stream_step, kind, mult, add16,
                                                         out, total, nl, prime0, n, pstride);
    LAUNCHED();
}

__global__ void k_sample_uniform(const Mod *__restrict__ mods, uint64_t seed, uint32_t tag, uint64_t stream0,
                                 uint64_t stream_step, uint64_t *__restrict__ out, uint64_t total, LimbMap lm,
                                 uint32_t n, uint64_t pstride) {
    GRID_LOOP(i, total) {   // over npoly * njl * n
        const uint64_t r0 = i / n;
        const uint32_t x = (uint32_t)(i - r0 * n);
        const uint64_t poly = r0 / lm.njl;
        const uint32_t jl = (uint32_t)(r0 - poly * lm.njl);
        const uint32_t lb = lm.limb(jl), pr = lm.prime(lb);
        const uint64_t q = mods[pr].q;
        const uint64_t ci = (uint64_t)pr * n + x;
        const uint64_t stream = stream0 + poly * stream_step;
        const uint64_t r1 = draw(seed, tag, stream, 2 * ci), r2 = draw(seed, tag, stream, 2 * ci + 1);
        // floor((r1*2^64 + r2) * q / 2^128) = floor((r1*q + floor(r2*q / 2^64)) / 2^64)
        const uint64_t lo1 = r1 * q, hi1 = __umul64hi(r1, q);
        const uint64_t hi2 = __umul64hi(r2, q);
        const uint64_t s = lo1 + hi2;
        const uint64_t carry = s < lo1 ? 1 : 0;
        out[poly * pstride + (uint64_t)lb * n + x] = hi1 + carry;
    }
}
void sample_uniform(const Mod *mods, uint64_t seed, uint32_t tag, uint64_t stream0, uint64_t stream_step,
                    uint64_t *out, uint32_t npoly, LimbMap lm, uint32_t n, uint64_t pstride, cudaStream_t st) {
    const uint64_t total = (uint64_t)npoly * lm.njl * n;
    k_sample_uniform<<<grid_for(total, 256), 256, 0, st>>>(mods, seed, tag, stream0, stream_step, out, total, lm, n,
                                                           pstride);
    LAUNCHED();
}

// =====================================================================================
// encode / decode: exact int8 x int8 -> int32 GEMM (entries centered mod p, |sum| < 2^31)
// =====================================================================================
#define GT 64
#define GK 32
__global__ void __launch_bounds__(256) k_gemm_s8(const int8_t *__restrict__ A, const int8_t *__restrict__ W,
                                                 int32_t *__restrict__ C, uint32_t B, uint32_t N, uint32_t K) {
    __shared__ int32_t sa[GK][GT + 1];
    __shared__ int32_t sw[GK][GT + 1];
    const uint32_t b0 = blockIdx.y * GT, j0 = blockIdx.x * GT;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    int32_t acc[4][4] = {};
    for (uint32_t k0 = 0; k0 < K; k0 += GK) {
        for (int e = threadIdx.x; e < GT * GK; e += 256) {
            const int r = e / GK, k = e % GK;
            const uint32_t kk = k0 + k;
            sa[k][r] = (b0 + r < B && kk < K) ? (int32_t)A[(uint64_t)(b0 + r) * K + kk] : 0;
            sw[k][r] = (j0 + r < N && kk < K) ? (int32_t)W[(uint64_t)(j0 + r) * K + kk] : 0;
        }
        __syncthreads();
#pragma unroll 8
        for (int k = 0; k < GK; ++k) {
            int32_t av[4], wv[4];
            for (int u = 0; u < 4; ++u) { av[u] = sa[k][ty * 4 + u]; wv[u] = sw[k][tx * 4 + u]; }
            for (int u = 0; u < 4; ++u)
                for (int v = 0; v < 4; ++v) acc[u][v] += av[u] * wv[v];
        }
        __syncthreads();
    }
    for (int u = 0; u < 4; ++u)
        for (int v = 0; v < 4; ++v) {
            const uint32_t b = b0 + ty * 4 + u, j = j0 + tx * 4 + v;
            if (b < B && j < N) C[(uint64_t)b * N + j] = acc[u][v];
        }
}
void gemm_s8(const int8_t *A, const int8_t *W, int32_t *C, uint32_t B, uint32_t N, uint32_t K, cudaStream_t st) {
    dim3 g((N + GT - 1) / GT, (B + GT - 1) / GT);
    k_gemm_s8<<<g, 256, 0, st>>>(A, W, C, B, N, K);
    LAUNCHED();
}

__device__ __forceinline__ int32_t center_p(int64_t v, int32_t p) {
    int64_t r = v % p;
    if (r < 0) r += p;
    if (r > p / 2) r -= p;
    return (int32_t)r;
}

__global__ void k_mod_p_center(const int32_t *__restrict__ in, int16_t *__restrict__ out, uint64_t total, int32_t p) {
    GRID_LOOP(i, total) out[i] = (int16_t)center_p(in[i], p);
}
void mod_p_center(const int32_t *in, int16_t *out, uint64_t count, int32_t p, cudaStream_t st) {
    k_mod_p_center<<<grid_for(count, 256), 256, 0, st>>>(in, out, count, p);
    LAUNCHED();
}
__global__ void k_s16_to_s8(const int16_t *__restrict__ in, int8_t *__restrict__ out, uint64_t total, int32_t p) {
    GRID_LOOP(i, total) out[i] = (int8_t)center_p(in[i], p);
}
void s16_to_s8(const int16_t *in, int8_t *out, uint64_t count, int32_t p, cudaStream_t st) {
    k_s16_to_s8<<<grid_for(count, 256), 256, 0, st>>>(in, out, count, p);
    LAUNCHED();
}

// Em[j][s*D+i] = V(j) + sum_{k>=n} V(k) red[k-n][j], V(e) = E0_i[(e t_s) mod m]  (sigma_{t_s^-1} of the
// slot-0 idempotent basis, P:271 CRT);  prime m: red = x^{m-1} -> -1 everywhere.
__global__ void k_build_enc(const int16_t *__restrict__ E0, const uint32_t *__restrict__ ts,
                            const int8_t *__restrict__ red, int8_t *__restrict__ Em, uint32_t n, uint32_t m,
                            uint32_t D, uint32_t S, int32_t p) {
    const uint64_t total = (uint64_t)n * n;
    GRID_LOOP(i, total) {
        const uint32_t j = (uint32_t)(i / n), col = (uint32_t)(i - (uint64_t)j * n);
        const uint32_t s = col / D, ii = col - s * D;
        const uint64_t t = ts[s];
        const int16_t *E = E0 + (uint64_t)ii * m;
        int64_t v = E[(j * t) % m];
        if (!red) {
            v -= E[((uint64_t)(m - 1) * t) % m];
        } else {
            for (uint32_t k = n; k < m; ++k) {
                const int8_t f = red[(uint64_t)(k - n) * n + j];
                if (f) v += (int64_t)f * E[((uint64_t)k * t) % m];
            }
        }
        Em[i] = (int8_t)center_p(v, p);
    }
}
void build_encode_matrix(const int16_t *E0, const uint32_t *ts, const int8_t *red, int8_t *Em, uint32_t n,
                         uint32_t m, uint32_t D, uint32_t S, int32_t p, cudaStream_t st) {
    k_build_enc<<<grid_for((uint64_t)n * n, 256), 256, 0, st>>>(E0, ts, red, Em, n, m, D, S, p);
    LAUNCHED();
}

// Dm[s*D+i][j] = coeff_i(zeta^{t_s j mod m})  (decode: beta_s = a(zeta^{t_s}))
__global__ void k_build_dec(const int16_t *__restrict__ zpow, const uint32_t *__restrict__ ts,
                            int8_t *__restrict__ Dm, uint32_t n, uint32_t m, uint32_t D, int32_t p) {
    const uint64_t total = (uint64_t)n * n;
    GRID_LOOP(i, total) {
        const uint32_t row = (uint32_t)(i / n), j = (uint32_t)(i - (uint64_t)row * n);
        const uint32_t s = row / D, ii = row - s * D;
        Dm[i] = (int8_t)center_p(zpow[((uint64_t)ts[s] * j % m) * D + ii], p);
    }
}
void build_decode_matrix(const int16_t *zpow, const uint32_t *ts, int8_t *Dm, uint32_t n, uint32_t m, uint32_t D,
                         uint32_t S, int32_t p, cudaStream_t st) {
    k_build_dec<<<grid_for((uint64_t)n * n, 256), 256, 0, st>>>(zpow, ts, Dm, n, m, D, p);
    LAUNCHED();
}

__global__ void k_s16_to_rns(const Mod *__restrict__ mods, const int16_t *__restrict__ in, uint64_t *__restrict__ out,
                             uint64_t total, uint32_t nl, uint32_t n) {
    GRID_LOOP(i, total) {   // over npoly * n
        const uint64_t poly = i / n;
        const uint32_t x = (uint32_t)(i - poly * n);
        const int64_t v = in[i];
        for (uint32_t l = 0; l < nl; ++l) out[(poly * nl + l) * n + x] = from_signed(v, mods[l].q);
    }
}
void s16_to_rns(const Mod *mods, const int16_t *in, uint64_t *out, uint32_t npoly, uint32_t nl, uint32_t n,
                cudaStream_t st) {
    const uint64_t total = (uint64_t)npoly * n;
    k_s16_to_rns<<<grid_for(total, 256), 256, 0, st>>>(mods, in, out, total, nl, n);
    LAUNCHED();
}

__global__ void k_dec_dot(const Mod *__restrict__ mods, const uint64_t *__restrict__ ct,
                          const uint64_t *__restrict__ s, uint64_t *__restrict__ o, uint64_t total, uint32_t lvl,
                          uint32_t n) {
    const uint64_t ln = (uint64_t)lvl * n;
    GRID_LOOP(i, total) {
        const uint64_t b = i / ln, r = i - b * ln;
        const uint32_t limb = (uint32_t)(r / n);
        const Mod M = mods[limb];
        o[i] = add_mod(ct[b * 2 * ln + r], mul_mod(ct[b * 2 * ln + ln + r], s[r], M), M.q);
    }
}
void dec_dot(const Mod *mods, const uint64_t *ct, const uint64_t *s, uint64_t *o, uint32_t B, uint32_t lvl,
             uint32_t n, cudaStream_t st) {
    const uint64_t total = (uint64_t)B * lvl * n;
    k_dec_dot<<<grid_for(total, 256), 256, 0, st>>>(mods, ct, s, o, total, lvl, n);
    LAUNCHED();
}

}  // namespace bc
