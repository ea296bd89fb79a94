// capi.cu -- extern "C" boundary of libboostcom.so (include/boostcom.h).
#include <algorithm>
#include <cstring>
#include <mutex>

#include "engine.h"

using namespace bc;

#define API_BEGIN try {
#define API_END                                   \
    }                                             \
    catch (BcError & e) {                         \
        last_error() = e.msg;                     \
        return e.st;                              \
    }                                             \
    catch (std::exception & e) {                  \
        last_error() = e.what();                  \
        return BC_E_INTERNAL;                     \
    }                                             \
    return BC_OK;

static cudaStream_t S(void *s) { return (cudaStream_t)s; }

static void check_launch() {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) BC_THROW(BC_E_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
}

extern "C" {

const char *bc_last_error(void) { return last_error().c_str(); }
void bc_set_ntt_impl(int impl) { g_ntt_impl = impl; }
int bc_tune(const char *key, int64_t value) {
    if (!key) return -1;
    if (!strcmp(key, "vec_chunk")) { g_vec_chunk = (uint64_t)std::max<int64_t>(value, 0); return 0; }
    if (!strcmp(key, "ntt_timing")) { g_ntt_timing = value ? 1 : 0; return 0; }
    if (!strcmp(key, "phase_timing")) { g_phase_timing = value ? 1 : 0; return 0; }
    if (!strcmp(key, "ntt_split")) { g_ntt_split = (int)value; return 0; }
    if (!strcmp(key, "ntt_persist_occ")) { g_ntt_persist_occ = (int)value; return 0; }
    if (!strcmp(key, "ntt_lean")) { g_ntt_lean = (int)value; return 0; }
    if (!strcmp(key, "axpy")) { g_axpy = (int)value; return 0; }
    if (!strcmp(key, "lift_blocks")) { g_lift_blocks = (int)value; return 0; }
    if (!strcmp(key, "ptsum")) { g_ptsum = (int)value; return 0; }
    if (!strcmp(key, "ntt_epi")) { g_ntt_epi = (int)value; return 0; }
    if (!strcmp(key, "lift2")) { g_lift2 = (int)value; return 0; }
    if (!strcmp(key, "kip_blocked")) { g_kip_blocked = (int)value; return 0; }
    if (!strcmp(key, "f64_elem")) { g_f64_elem = (int)value; return 0; }
    if (!strcmp(key, "phi_conv")) { g_phi_conv = (int)value; return 0; }
    if (!strcmp(key, "ntt_dbg")) { g_ntt_dbg = (int)value; return 0; }
    if (!strcmp(key, "nttc_variant")) { g_nttc_variant = (int)value; return 0; }
    if (!strcmp(key, "nttc_clusters")) { g_nttc_clusters = (int)value; return g_nttc_active; }
    if (!strcmp(key, "ntt_group_bytes")) { g_ntt_group_bytes = (uint64_t)std::max<int64_t>(value, 1 << 20); return 0; }
    return -1;
}
int bc_phase_timing(double *ms, uint64_t *calls) { return phase_timing_collect(ms, calls); }
int bc_ntt_timing(double *ms, uint64_t *limb_transforms, uint64_t *calls) {
    return ntt_timing_collect(ms, limb_transforms, calls);
}
int bc_ntt_timing_split(double *ms, uint64_t *limb_transforms, uint64_t *inverse_limb_transforms, uint64_t *calls) {
    return ntt_timing_collect(ms, limb_transforms, calls, inverse_limb_transforms);
}
uint64_t bc_launch_count(int reset) {
    uint64_t c = launch_counter();
    if (reset) launch_counter() = 0;
    return c;
}

bc_status bc_ctx_create(const bc_params *prm, int device, bc_ctx **out) {
    API_BEGIN
    if (!prm || !out) BC_THROW(BC_E_ARG, "null argument");
    bc_ctx *X = new bc_ctx();
    X->prm = *prm;
    X->device = device;
    try {
        ctx_build(X);
        ctx_precompute_pt(X);
    } catch (...) {
        ctx_free(X);
        delete X;
        throw;
    }
    *out = X;
    API_END
}

void bc_ctx_destroy(bc_ctx *ctx) {
    if (!ctx) return;
    compact_plans_release(ctx);
    ctx_free(ctx);
    delete ctx;
}

bc_status bc_ctx_info(const bc_ctx *X, bc_info *o) {
    API_BEGIN
    if (!X || !o) BC_THROW(BC_E_ARG, "null argument");
    o->n = X->n; o->m = X->m; o->M = X->M; o->D = X->alg.D; o->S = X->alg.S;
    o->ints_per_ct = X->ints; o->n_cipher = X->L1; o->n_special = X->K; o->dnum = X->dnum;
    o->g = X->alg.g; o->base = X->base; o->n_galois = (uint32_t)X->galois.size();
    API_END
}

bc_status bc_circuit_plan(uint32_t p, char circuit, uint32_t schedule, uint32_t *k, uint32_t *products,
                          uint32_t *depth) {
    API_BEGIN
    if (!k || !products || !depth) BC_THROW(BC_E_ARG, "null argument");
    if (p < 3 || p > 257 || !is_prime_u64(p)) BC_THROW(BC_E_PARAM, "p must be an odd prime <= 257");
    if (circuit != 'U' && circuit != 'B') BC_THROW(BC_E_PARAM, "circuit must be 'U' or 'B'");
    if (schedule != 0 && schedule != 16 && schedule != 23 && schedule != 26 && schedule != 27)
        BC_THROW(BC_E_PARAM, "schedule must be 16, 23, 26 or 27");
    int kk, mu, de;
    circuit_plan(p, circuit, (int)schedule, &kk, &mu, &de);
    *k = (uint32_t)kk;
    *products = (uint32_t)mu;
    *depth = (uint32_t)de;
    API_END
}

bc_status bc_ctx_moduli(const bc_ctx *X, uint64_t *h_out, uint64_t *h_omega) {
    API_BEGIN
    if (!X) BC_THROW(BC_E_ARG, "null ctx");
    if (h_out) std::copy(X->moduli.begin(), X->moduli.end(), h_out);
    if (h_omega) std::copy(X->omega.begin(), X->omega.end(), h_omega);
    API_END
}

bc_status bc_ctx_slots(const bc_ctx *X, int64_t *h_G, int64_t *h_zeta, int64_t *h_t) {
    API_BEGIN
    if (!X) BC_THROW(BC_E_ARG, "null ctx");
    if (h_G) std::copy(X->alg.gf.G.begin(), X->alg.gf.G.end(), h_G);
    if (h_zeta) std::copy(X->alg.zeta.begin(), X->alg.zeta.end(), h_zeta);
    if (h_t) for (size_t s = 0; s < X->alg.t.size(); ++s) h_t[s] = X->alg.t[s];
    API_END
}

bc_status bc_ctx_galois(const bc_ctx *X, uint32_t *h_out) {
    API_BEGIN
    if (!X || !h_out) BC_THROW(BC_E_ARG, "null argument");
    std::copy(X->galois.begin(), X->galois.end(), h_out);
    API_END
}

size_t bc_ct_bytes(const bc_ctx *X, uint32_t batch, uint32_t level) {
    return X ? (size_t)batch * 2 * level * X->n * 8 : 0;
}

}  // extern "C"

// ------------------------------------------------------------------ dry-run sizing
template <class F>
static size_t dry_peak(bc_ctx *X, const bc_keys *keys, F fn) {
    Arena A;
    A.init(nullptr, (size_t)1 << 62, true);
    Eng E{X, keys, &A, 0};
    fn(E);
    return A.hwm;      // includes fragmentation (same best-fit sequence as the real run)
}

static size_t compare_peak(bc_ctx *X, const bc_keys *keys, uint32_t B, uint32_t lvl, int which) {
    return dry_peak(X, keys, [&](Eng &E) {
        CT a = E.view((uint64_t *)(uintptr_t)256, B, lvl), b = E.view((uint64_t *)(uintptr_t)256, B, lvl);
        CT lt, eq;
        if (which == 2) {
            compare_batch(E, a, b, &lt, nullptr);
            CT o = select_batch(E, lt, a, b);
        } else {
            compare_batch(E, a, b, &lt, which == 1 ? &eq : nullptr);
        }
    });
}

extern "C" size_t bc_workspace_bytes(bc_ctx *X, uint32_t batch) {
    // max over compare (lt + eq) and min/max/select where the chain allows them
    size_t best = 0;
    for (int which : {1, 2}) {
        try {
            best = std::max(best, compare_peak(X, nullptr, batch, X->L1, which));
        } catch (...) {
        }
    }
    return best + best / 4 + (64u << 20);   // slack for fragmentation of the first-fit arena
}

extern "C" uint32_t bc_compare_out_level(bc_ctx *X, uint32_t level, int which) {
    try {
        uint32_t out = 0;
        Arena A;
        A.init(nullptr, (size_t)1 << 62, true);
        Eng E{X, nullptr, &A, 0};
        CT a = E.view((uint64_t *)(uintptr_t)256, 1, level), b = a;
        CT lt, eq;
        if (which == 2) {
            compare_batch(E, a, b, &lt, nullptr);
            out = select_batch(E, lt, a, b).lvl;
        } else {
            compare_batch(E, a, b, &lt, which == 1 ? &eq : nullptr);
            out = which == 1 ? eq.lvl : lt.lvl;
        }
        return out;
    } catch (...) {
        return 0;
    }
}

// choose the largest chunk whose dry-run peak fits the workspace
static uint32_t choose_chunk(bc_ctx *X, const bc_keys *keys, uint32_t B, uint32_t lvl, int which, size_t ws) {
    auto need = [&](uint32_t b) { size_t pk = compare_peak(X, keys, b, lvl, which); return pk + pk / 4 + (32u << 20); };
    size_t p1 = need(1);
    if (p1 > ws) BC_THROW(BC_E_OOM, "workspace smaller than one pair needs (" + std::to_string(p1) + " bytes)");
    if (B == 1) return 1;
    size_t p2 = need(2);
    size_t per = p2 > p1 ? p2 - p1 : p1;
    uint64_t c = 1 + (ws - p1) / per;
    uint32_t chunk = (uint32_t)std::min<uint64_t>(B, c);
    while (chunk > 1 && need(chunk) > ws) chunk = chunk * 7 / 8;
    return std::max<uint32_t>(chunk, 1);
}

static void out_copy(Eng &E, const CT &src, const bc_ct &dst, uint32_t b0) {
    if (src.lvl != dst.level) BC_THROW(BC_E_LEVEL, "output level " + std::to_string(dst.level) + " != computed " + std::to_string(src.lvl));
    if (!dst.data || (uint64_t)b0 + src.B > dst.batch) BC_THROW(BC_E_ARG, "output view too small");
    uint64_t *d = (uint64_t *)dst.data + (uint64_t)b0 * 2 * dst.level * E.X->n;
    CK(cudaMemcpyAsync(d, src.d, (size_t)src.B * src.bstride * 8, cudaMemcpyDeviceToDevice, E.st));
}

static void check_ct(const bc_ctx *X, const bc_ct &c, const char *nm) {
    if (!c.data || c.batch == 0) BC_THROW(BC_E_ARG, std::string(nm) + ": empty ciphertext view");
    if (c.level < 1 || c.level > X->L1) BC_THROW(BC_E_LEVEL, std::string(nm) + ": bad level");
}

// output views are validated BEFORE anything is enqueued (no partial outputs on error): the
// level an operation produces is found by a host-only dry run of the same schedule
template <class F>
static uint32_t dry_level(bc_ctx *X, F fn) {
    Arena A;
    A.init(nullptr, (size_t)1 << 62, true);
    Eng E{X, nullptr, &A, 0};
    return fn(E).lvl;
}
static CT dry_view(Eng &E, const bc_ct &c) { return E.view((uint64_t *)(uintptr_t)256, 1, c.level); }
static void check_out(const bc_ctx *X, const bc_ct &o, uint32_t batch, uint32_t level, const char *nm) {
    check_ct(X, o, nm);
    if (o.batch < batch) BC_THROW(BC_E_ARG, std::string(nm) + ": output batch " + std::to_string(o.batch) + " < " + std::to_string(batch));
    if (o.level != level)
        BC_THROW(BC_E_LEVEL, std::string(nm) + ": output level " + std::to_string(o.level) + " != " + std::to_string(level));
}

// which: 0 lt, 1 lt+eq, 3 eq only, 2 min, 4 max
static bc_status run_compare(bc_ctx *X, const bc_keys *keys, bc_ct a, bc_ct b, bc_ct o1, bc_ct o2, void *ws,
                             size_t wsb, void *st, int which) {
    API_BEGIN
    if (!X || !keys) BC_THROW(BC_E_ARG, "null ctx/keys");
    check_ct(X, a, "a");
    check_ct(X, b, "b");
    if (a.batch != b.batch) BC_THROW(BC_E_ARG, "batch mismatch");
    const uint32_t lvl = std::min(a.level, b.level);
    const int pk = (which == 2 || which == 4) ? 2 : (which == 0 ? 0 : 1);
    {
        const uint32_t want = dry_level(X, [&](Eng &E) {
            CT av = dry_view(E, a), bv = dry_view(E, b), lt, eq;
            if (which == 2 || which == 4) {
                compare_batch(E, av, bv, &lt, nullptr);
                return select_batch(E, lt, av, bv);
            }
            compare_batch(E, av, bv, which == 3 ? nullptr : &lt, which ? &eq : nullptr);
            return which == 3 ? eq : lt;
        });
        check_out(X, o1, a.batch, want, "out");
        if (which == 1 && o2.data) {
            const uint32_t weq = dry_level(X, [&](Eng &E) {
                CT av = dry_view(E, a), bv = dry_view(E, b), lt, eq;
                compare_batch(E, av, bv, &lt, &eq);
                return eq;
            });
            check_out(X, o2, a.batch, weq, "eq_out");
        }
    }
    const uint32_t chunk = choose_chunk(X, keys, a.batch, lvl, pk, wsb);
    for (uint32_t b0 = 0; b0 < a.batch; b0 += chunk) {
        const uint32_t nb = std::min(chunk, a.batch - b0);
        Arena A;
        A.init(ws, wsb, false);
        Eng E{X, keys, &A, S(st)};
        CT av = E.view((uint64_t *)a.data + (uint64_t)b0 * 2 * a.level * X->n, nb, a.level);
        CT bv = E.view((uint64_t *)b.data + (uint64_t)b0 * 2 * b.level * X->n, nb, b.level);
        CT lt, eq;
        if (which == 2 || which == 4) {
            compare_batch(E, av, bv, &lt, nullptr);
            CT r = which == 2 ? select_batch(E, lt, av, bv) : select_batch(E, lt, bv, av);
            out_copy(E, r, o1, b0);
        } else {
            compare_batch(E, av, bv, which == 3 ? nullptr : &lt, which ? &eq : nullptr);   // 3: EQ only
            if (which == 0 || which == 1) out_copy(E, lt, o1, b0);
            if (which == 1 && o2.data) out_copy(E, eq, o2, b0);
            if (which == 3) out_copy(E, eq, o1, b0);
        }
        check_launch();
        // the next chunk reuses the arena: its kernels are ordered after this chunk's on the same stream,
        // so no host synchronisation is needed (the compare never blocks the host: a11)
    }
    API_END
}

extern "C" {

bc_status bc_compare(bc_ctx *X, const bc_keys *k, bc_ct a, bc_ct b, bc_ct lt, bc_ct eq, void *ws, size_t wsb, void *st) {
    return run_compare(X, k, a, b, lt, eq, ws, wsb, st, 1);
}
bc_status bc_compare_lt(bc_ctx *X, const bc_keys *k, bc_ct a, bc_ct b, bc_ct out, void *ws, size_t wsb, void *st) {
    bc_ct none{nullptr, 0, 0};
    return run_compare(X, k, a, b, out, none, ws, wsb, st, 0);
}
bc_status bc_compare_eq(bc_ctx *X, const bc_keys *k, bc_ct a, bc_ct b, bc_ct out, void *ws, size_t wsb, void *st) {
    bc_ct none{nullptr, 0, 0};
    return run_compare(X, k, a, b, out, none, ws, wsb, st, 3);
}
bc_status bc_min(bc_ctx *X, const bc_keys *k, bc_ct a, bc_ct b, bc_ct out, void *ws, size_t wsb, void *st) {
    bc_ct none{nullptr, 0, 0};
    return run_compare(X, k, a, b, out, none, ws, wsb, st, 2);
}
bc_status bc_max(bc_ctx *X, const bc_keys *k, bc_ct a, bc_ct b, bc_ct out, void *ws, size_t wsb, void *st) {
    bc_ct none{nullptr, 0, 0};
    return run_compare(X, k, a, b, out, none, ws, wsb, st, 4);
}

bc_status bc_select(bc_ctx *X, const bc_keys *k, bc_ct cond, bc_ct x1, bc_ct x2, bc_ct out, void *ws, size_t wsb,
                    void *st) {
    API_BEGIN
    if (!X || !k) BC_THROW(BC_E_ARG, "null ctx/keys");
    check_ct(X, cond, "cond"); check_ct(X, x1, "x1"); check_ct(X, x2, "x2");
    if (x1.batch != cond.batch || x2.batch != cond.batch) BC_THROW(BC_E_ARG, "batch mismatch");
    check_out(X, out, cond.batch, dry_level(X, [&](Eng &E) {
        return select_batch(E, dry_view(E, cond), dry_view(E, x1), dry_view(E, x2)); }), "out");
    Arena A;
    A.init(ws, wsb, false);
    Eng E{X, k, &A, S(st)};
    CT r = select_batch(E, E.view((uint64_t *)cond.data, cond.batch, cond.level),
                        E.view((uint64_t *)x1.data, x1.batch, x1.level), E.view((uint64_t *)x2.data, x2.batch, x2.level));
    out_copy(E, r, out, 0);
    check_launch();
    API_END
}

// ------------------------------------------------------------------ non-blocking (a11)
bc_status bc_compare_lt_async(bc_ctx *X, const bc_keys *k, bc_ct a, bc_ct b, bc_ct out, void *ws, size_t wsb,
                              void *side, bc_handle *h) {
    if (!h) { last_error() = "null handle"; return BC_E_ARG; }
    bc_status s = bc_compare_lt(X, k, a, b, out, ws, wsb, side);
    if (s != BC_OK) return s;
    API_BEGIN
    cudaEvent_t ev;
    CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CK(cudaEventRecord(ev, S(side)));
    h->event = ev;
    h->stream = side;
    h->consumed = 0;
    API_END
}

// ------------------------------------------------------------------ host buffers, pipelined (e2e)
}  // extern "C"
static cudaStream_t copy_stream_for_device() {
    static std::mutex mu;
    static cudaStream_t s[64] = {nullptr};
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    if (!s[dev & 63]) CK(cudaStreamCreateWithFlags(&s[dev & 63], cudaStreamNonBlocking));
    return s[dev & 63];
}
extern "C" {

size_t bc_host_stage_bytes(bc_ctx *X, uint32_t chunk, uint32_t level) {
    if (!X || !chunk || level < 1 || level > X->L1) return 0;
    const uint32_t lo = bc_compare_out_level(X, level, 0);
    return (size_t)2 * chunk * (2ull * 2 * level + 2ull * lo) * X->n * 8;
}

bc_status bc_compare_lt_host(bc_ctx *X, const bc_keys *keys, const uint64_t *h_a, const uint64_t *h_b, uint32_t batch,
                             uint32_t level, uint64_t *h_out, uint32_t chunk, void *d_stage, size_t stage_bytes,
                             void *ws, size_t wsb, void *st) {
    API_BEGIN
    if (!X || !keys || !h_a || !h_b || !h_out || !d_stage) BC_THROW(BC_E_ARG, "null argument");
    if (!batch) return BC_OK;
    if (level < 1 || level > X->L1) BC_THROW(BC_E_LEVEL, "bad level");
    if (!chunk) chunk = std::max<uint32_t>(1, (batch + 3) / 4);
    chunk = std::min(chunk, batch);
    if (bc_host_stage_bytes(X, chunk, level) > stage_bytes) BC_THROW(BC_E_ARG, "staging buffer smaller than bc_host_stage_bytes");
    const uint32_t lo = bc_compare_out_level(X, level, 0);
    const uint64_t cw = 2ull * level * X->n, ow = 2ull * lo * X->n;     // words per input / output ciphertext
    const uint64_t slot = (uint64_t)chunk * (2 * cw + ow);
    cudaStream_t cs = copy_stream_for_device(), ms = S(st);
    struct Events {                     // destroyed on every exit (pending ones are released once complete)
        cudaEvent_t e[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
        ~Events() {
            for (cudaEvent_t x : e)
                if (x) cudaEventDestroy(x);
        }
    } evs;
    for (int i = 0; i < 5; ++i) CK(cudaEventCreateWithFlags(&evs.e[i], cudaEventDisableTiming));
    cudaEvent_t *h2d = evs.e, *done = evs.e + 2, d2h = evs.e[4];
    // the copy stream starts after the work already queued on the caller's stream (e.g. a previous call's reads)
    CK(cudaEventRecord(d2h, ms));
    CK(cudaStreamWaitEvent(cs, d2h, 0));
    bc_status rc = BC_OK;
    const uint32_t nch = (batch + chunk - 1) / chunk;
    auto slot_ptr = [&](uint32_t i) { return (uint64_t *)d_stage + (i & 1) * slot; };
    // host->device copy of chunk i into slot i & 1 (copy stream).  Queue order on the copy stream:
    // H2D(0), H2D(1), D2H(0), H2D(2), D2H(1), ... -- H2D(i+1) follows D2H(i-1), which waits for compare(i-1), so
    // it overlaps compare(i) and never overwrites a slot that compare(i-1) or D2H(i-1) still reads
    auto h2d_chunk = [&](uint32_t i) {
        const uint32_t b0 = i * chunk, nb = std::min(chunk, batch - b0);
        uint64_t *da = slot_ptr(i), *db = da + (uint64_t)chunk * cw;
        CK(cudaMemcpyAsync(da, h_a + (uint64_t)b0 * cw, (size_t)nb * cw * 8, cudaMemcpyHostToDevice, cs));
        CK(cudaMemcpyAsync(db, h_b + (uint64_t)b0 * cw, (size_t)nb * cw * 8, cudaMemcpyHostToDevice, cs));
        CK(cudaEventRecord(h2d[i & 1], cs));
    };
    h2d_chunk(0);
    for (uint32_t i = 0; i < nch; ++i) {
        const uint32_t b0 = i * chunk, nb = std::min(chunk, batch - b0);
        if (i + 1 < nch) h2d_chunk(i + 1);
        uint64_t *da = slot_ptr(i), *db = da + (uint64_t)chunk * cw, *dout = db + (uint64_t)chunk * cw;
        CK(cudaStreamWaitEvent(ms, h2d[i & 1], 0));
        bc_ct av{da, nb, level}, bv{db, nb, level}, ov{dout, nb, lo}, none{nullptr, 0, 0};
        rc = run_compare(X, keys, av, bv, ov, none, ws, wsb, st, 0);
        if (rc != BC_OK) break;
        CK(cudaEventRecord(done[i & 1], ms));
        CK(cudaStreamWaitEvent(cs, done[i & 1], 0));
        CK(cudaMemcpyAsync(h_out + (uint64_t)b0 * ow, dout, (size_t)nb * ow * 8, cudaMemcpyDeviceToHost, cs));
    }
    // the caller's stream completes only after every output word has reached the host
    CK(cudaEventRecord(d2h, cs));
    CK(cudaStreamWaitEvent(ms, d2h, 0));
    if (rc != BC_OK) return rc;
    API_END
}

// ------------------------------------------------------------------ CUDA graphs
}  // extern "C"
struct bc_graph {
    cudaGraph_t g = nullptr;
    cudaGraphExec_t x = nullptr;
};
extern "C" {
bc_status bc_graph_capture_begin(void *st) {
    API_BEGIN
    if (!st) BC_THROW(BC_E_ARG, "capture needs a non-default stream");
    CK(cudaStreamBeginCapture(S(st), cudaStreamCaptureModeThreadLocal));
    API_END
}
bc_status bc_graph_capture_end(void *st, bc_graph **out) {
    API_BEGIN
    if (!st || !out) BC_THROW(BC_E_ARG, "null argument");
    bc_graph *G = new bc_graph();
    cudaError_t e = cudaStreamEndCapture(S(st), &G->g);
    if (e != cudaSuccess) {
        delete G;
        (void)cudaGetLastError();
        BC_THROW(BC_E_CUDA, std::string("cudaStreamEndCapture: ") + cudaGetErrorString(e));
    }
    e = cudaGraphInstantiateWithFlags(&G->x, G->g, cudaGraphInstantiateFlagUseNodePriority);   // captured stream priorities
    if (e != cudaSuccess) {
        cudaGraphDestroy(G->g);
        delete G;
        (void)cudaGetLastError();
        BC_THROW(BC_E_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e));
    }
    *out = G;
    API_END
}
bc_status bc_graph_launch(bc_graph *g, void *st) {
    API_BEGIN
    if (!g || !g->x) BC_THROW(BC_E_ARG, "null graph");
    CK(cudaGraphLaunch(g->x, S(st)));
    API_END
}
void bc_graph_destroy(bc_graph *g) {
    if (!g) return;
    if (g->x) cudaGraphExecDestroy(g->x);
    if (g->g) cudaGraphDestroy(g->g);
    delete g;
}

// R24 private_q (f4): blocking (side == NULL) or with the branch evaluation on `side` (Listing 5)
static uint32_t pq_level(bc_ctx *X, const bc_keys *k, const bc_ct &data, const bc_ct &q, const bc_ct &codes,
                         const bc_ct &op1, uint32_t e) {
    return dry_level(X, [&](Eng &E) {
        return private_query_batch(E, nullptr, E.view((uint64_t *)(uintptr_t)256, data.batch, data.level),
                                   E.view((uint64_t *)(uintptr_t)256, 1, q.level),
                                   E.view((uint64_t *)(uintptr_t)256, 3, codes.level),
                                   E.view((uint64_t *)(uintptr_t)256, 1, op1.level), e);
    });
}
uint32_t bc_private_query_level(bc_ctx *X, uint32_t n_data, uint32_t data_level, uint32_t q_level,
                                uint32_t op1_level, uint32_t e) {
    try {
        bc_ct d{(void *)256, n_data, data_level}, q{(void *)256, 1, q_level}, c{(void *)256, 3, q_level},
            o{(void *)256, 1, op1_level};
        return pq_level(X, nullptr, d, q, c, o, e);
    } catch (...) {
        return 0;
    }
}
size_t bc_private_query_workspace_bytes(bc_ctx *X, uint32_t n_data, uint32_t data_level, uint32_t q_level,
                                        uint32_t op1_level, uint32_t e, int side) {
    try {
        size_t pk = dry_peak(X, nullptr, [&](Eng &E) {
            CT d = E.view((uint64_t *)(uintptr_t)256, n_data, data_level);
            CT q = E.view((uint64_t *)(uintptr_t)256, 1, q_level), c = E.view((uint64_t *)(uintptr_t)256, 3, q_level);
            CT o = E.view((uint64_t *)(uintptr_t)256, 1, op1_level);
            if (side == 1) {        // the side stream's share: the EQs and broadcasts
                CT qr = concat_batch(E, {q, q, q}), lt, eq;
                compare_batch(E, qr, c, nullptr, &eq);
                CT m = broadcast_batch(E, eq);
            } else {                // the whole query (an upper bound for the main stream's share)
                CT r = private_query_batch(E, nullptr, d, q, c, o, e);
            }
        });
        return pk + pk / 4 + (64u << 20);
    } catch (...) {
        return 0;
    }
}
bc_status bc_private_query(bc_ctx *X, const bc_keys *k, bc_ct data, bc_ct q, bc_ct codes, bc_ct op1, uint32_t e,
                           bc_ct out, void *ws, size_t wsb, void *ws_side, size_t wsb_side, void *st, void *side) {
    API_BEGIN
    if (!X || !k) BC_THROW(BC_E_ARG, "null ctx/keys");
    check_ct(X, data, "data"); check_ct(X, q, "q"); check_ct(X, codes, "codes"); check_ct(X, op1, "op1");
    if (q.batch != 1 || op1.batch != 1 || codes.batch != 3) BC_THROW(BC_E_ARG, "q, op1: batch 1; codes: batch 3");
    if (e < 1) BC_THROW(BC_E_ARG, "exponent must be >= 1");
    if (side && (!ws_side || !wsb_side)) BC_THROW(BC_E_ARG, "non-blocking query needs a side workspace");
    check_out(X, out, data.batch, pq_level(X, k, data, q, codes, op1, e), "out");
    Arena A;
    A.init(ws, wsb, false);
    Eng E{X, k, &A, S(st)};
    Arena A2;
    if (side) A2.init(ws_side, wsb_side, false);
    Eng E2{X, k, &A2, S(side)};
    CT r = private_query_batch(E, side ? &E2 : nullptr, E.view((uint64_t *)data.data, data.batch, data.level),
                               E.view((uint64_t *)q.data, 1, q.level), E.view((uint64_t *)codes.data, 3, codes.level),
                               E.view((uint64_t *)op1.data, 1, op1.level), e);
    out_copy(E, r, out, 0);
    check_launch();
    API_END
}

bc_status bc_wait(bc_handle *h, void *joiner) {
    API_BEGIN
    if (!h || !h->event) BC_THROW(BC_E_ARG, "null handle");
    if (h->consumed) BC_THROW(BC_E_CONSUMED, "handle already waited on");
    CK(cudaStreamWaitEvent(S(joiner), (cudaEvent_t)h->event, 0));
    CK(cudaEventDestroy((cudaEvent_t)h->event));
    h->consumed = 1;
    API_END
}

// ------------------------------------------------------------------ primitives
bc_status bc_ntt_fwd(bc_ctx *X, const void *in, void *out, uint32_t npoly, uint32_t nlimb, uint32_t prime0, void *ws,
                     size_t wsb, void *st) {
    API_BEGIN
    if (!X || !in || !out) BC_THROW(BC_E_ARG, "null argument");
    if (prime0 + nlimb > X->L1 + X->K) BC_THROW(BC_E_ARG, "limbs out of range");
    Arena A;
    A.init(ws, wsb, false);
    Eng E{X, nullptr, &A, S(st)};
    E.ntt_fwd((const uint64_t *)in, (uint64_t *)out, npoly, limbmap_plain(nlimb, prime0), (uint64_t)nlimb * X->n,
              (uint64_t)nlimb * X->n);
    check_launch();
    API_END
}
bc_status bc_ntt_inv(bc_ctx *X, const void *in, void *out, uint32_t npoly, uint32_t nlimb, uint32_t prime0, void *ws,
                     size_t wsb, void *st) {
    API_BEGIN
    if (!X || !in || !out) BC_THROW(BC_E_ARG, "null argument");
    if (prime0 + nlimb > X->L1 + X->K) BC_THROW(BC_E_ARG, "limbs out of range");
    Arena A;
    A.init(ws, wsb, false);
    Eng E{X, nullptr, &A, S(st)};
    E.ntt_inv((const uint64_t *)in, (uint64_t *)out, npoly, limbmap_plain(nlimb, prime0), (uint64_t)nlimb * X->n,
              (uint64_t)nlimb * X->n);
    check_launch();
    API_END
}

bc_status bc_tensor(bc_ctx *X, bc_ct a, bc_ct b, void *out, void *st) {
    API_BEGIN
    if (!X || !out) BC_THROW(BC_E_ARG, "null argument");
    check_ct(X, a, "a"); check_ct(X, b, "b");
    if (a.level != b.level || a.batch != b.batch) BC_THROW(BC_E_LEVEL, "tensor: shape mismatch");
    ew_tensor(X->d_mods, (uint64_t *)a.data, (uint64_t *)b.data, (uint64_t *)out, a.batch, a.level, X->n, S(st));
    check_launch();
    API_END
}

bc_status bc_automorph(bc_ctx *X, bc_ct a, uint32_t t, bc_ct out, void *st) {
    API_BEGIN
    if (!X) BC_THROW(BC_E_ARG, "null ctx");
    check_ct(X, a, "a");
    if (gcd_u64(t, X->m) != 1) BC_THROW(BC_E_ARG, "t not in Z_m^*");
    check_out(X, out, a.batch, a.level, "out");
    ew_automorph(X->T, (uint64_t *)a.data, (uint64_t *)out.data, a.batch, 2, a.level, t % X->m, S(st));
    check_launch();
    API_END
}

bc_status bc_keyswitch(bc_ctx *X, const bc_keys *k, const void *poly, uint32_t batch, uint32_t level, uint32_t t,
                       void *out, void *ws, size_t wsb, void *st) {
    API_BEGIN
    if (!X || !k || !poly || !out) BC_THROW(BC_E_ARG, "null argument");
    Arena A;
    A.init(ws, wsb, false);
    Eng E{X, k, &A, S(st)};
    CT u = E.keyswitch((const uint64_t *)poly, (uint64_t)level * X->n, batch, level, t);
    CK(cudaMemcpyAsync(out, u.d, (size_t)batch * u.bstride * 8, cudaMemcpyDeviceToDevice, S(st)));
    check_launch();
    API_END
}

bc_status bc_modswitch(bc_ctx *X, bc_ct a, bc_ct out, void *ws, size_t wsb, void *st) {
    API_BEGIN
    if (!X) BC_THROW(BC_E_ARG, "null ctx");
    check_ct(X, a, "a");
    if (a.level < 2) BC_THROW(BC_E_LEVEL, "modswitch: out of levels");
    check_out(X, out, a.batch, a.level - 1, "out");
    Arena A;
    A.init(ws, wsb, false);
    Eng E{X, nullptr, &A, S(st)};
    CT r = E.modswitch(E.view((uint64_t *)a.data, a.batch, a.level));
    out_copy(E, r, out, 0);
    check_launch();
    API_END
}

bc_status bc_mul(bc_ctx *X, const bc_keys *k, bc_ct a, bc_ct b, bc_ct out, void *ws, size_t wsb, void *st) {
    API_BEGIN
    if (!X || !k) BC_THROW(BC_E_ARG, "null ctx/keys");
    check_ct(X, a, "a"); check_ct(X, b, "b");
    if (a.batch != b.batch) BC_THROW(BC_E_ARG, "batch mismatch");
    check_out(X, out, a.batch, dry_level(X, [&](Eng &E) { return E.mul(dry_view(E, a), dry_view(E, b)); }), "out");
    Arena A;
    A.init(ws, wsb, false);
    Eng E{X, k, &A, S(st)};
    CT r = E.mul(E.view((uint64_t *)a.data, a.batch, a.level), E.view((uint64_t *)b.data, b.batch, b.level));
    out_copy(E, r, out, 0);
    check_launch();
    API_END
}

bc_status bc_rotate(bc_ctx *X, const bc_keys *k, bc_ct a, int32_t r, bc_ct out, void *ws, size_t wsb, void *st) {
    API_BEGIN
    if (!X || !k) BC_THROW(BC_E_ARG, "null ctx/keys");
    check_ct(X, a, "a");
    check_out(X, out, a.batch, a.level, "out");
    Arena A;
    A.init(ws, wsb, false);
    Eng E{X, k, &A, S(st)};
    CT res = E.rotate(E.view((uint64_t *)a.data, a.batch, a.level), r);
    out_copy(E, res, out, 0);
    check_launch();
    API_END
}

bc_status bc_frobenius(bc_ctx *X, const bc_keys *k, bc_ct a, uint32_t r, bc_ct out, void *ws, size_t wsb, void *st) {
    API_BEGIN
    if (!X || !k) BC_THROW(BC_E_ARG, "null ctx/keys");
    check_ct(X, a, "a");
    check_out(X, out, a.batch, a.level, "out");
    Arena A;
    A.init(ws, wsb, false);
    Eng E{X, k, &A, S(st)};
    CT res = E.frobenius(E.view((uint64_t *)a.data, a.batch, a.level), r);
    out_copy(E, res, out, 0);
    check_launch();
    API_END
}

bc_status bc_extract(bc_ctx *X, const bc_keys *k, bc_ct a, void *out, void *ws, size_t wsb, void *st) {
    API_BEGIN
    if (!X || !k || !out) BC_THROW(BC_E_ARG, "null argument");
    check_ct(X, a, "a");
    Arena A;
    A.init(ws, wsb, false);
    Eng E{X, k, &A, S(st)};
    std::vector<CT> digs = extract_batch(E, E.view((uint64_t *)a.data, a.batch, a.level));
    // digits form one batch [d][B]; the ABI layout is [B][d]
    const uint64_t cw = (uint64_t)2 * a.level * X->n;
    for (uint32_t i = 0; i < digs.size(); ++i)
        for (uint32_t b = 0; b < a.batch; ++b)
            CK(cudaMemcpyAsync((uint64_t *)out + ((uint64_t)b * digs.size() + i) * cw, digs[i].d + (uint64_t)b * cw, cw * 8,
                               cudaMemcpyDeviceToDevice, S(st)));
    check_launch();
    API_END
}

}  // extern "C"

// ------------------------------------------------------------------ vectors: tournament / sort
// which: 0 min tree, 1 max tree, 2 sort.  Returns the output level(s) of a dry run.
static std::vector<CT> vec_run(Eng &E, int which, const std::vector<CT> &v) {
    if (which == 2) return sort_batch(E, v);
    return {tournament_batch(E, v, which == 1)};
}

static std::vector<CT> vec_views(bc_ctx *X, Eng &E, const bc_ct *v, uint32_t T) {
    if (!v || T == 0) BC_THROW(BC_E_ARG, "empty element list");
    std::vector<CT> out;
    for (uint32_t i = 0; i < T; ++i) {
        check_ct(X, v[i], "v[i]");
        if (v[i].batch != v[0].batch) BC_THROW(BC_E_ARG, "element batches differ");
        out.push_back(E.view((uint64_t *)v[i].data, v[i].batch, v[i].level));
    }
    return out;
}

extern "C" uint32_t bc_vec_out_level(bc_ctx *X, int which, const uint32_t *levels, uint32_t T) {
    try {
        if (!X || !levels || T == 0) return 0;
        Arena A;
        A.init(nullptr, (size_t)1 << 62, true);
        Eng E{X, nullptr, &A, 0};
        std::vector<CT> v;
        for (uint32_t i = 0; i < T; ++i) v.push_back(E.view((uint64_t *)(uintptr_t)256, 1, levels[i]));
        return vec_run(E, which, v)[0].lvl;
    } catch (...) {
        return 0;
    }
}

extern "C" size_t bc_vec_workspace_bytes(bc_ctx *X, int which, const uint32_t *levels, uint32_t T, uint32_t batch) {
    try {
        if (!X || !levels || T == 0) return 0;
        size_t pk = dry_peak(X, nullptr, [&](Eng &E) {
            std::vector<CT> v;
            for (uint32_t i = 0; i < T; ++i) v.push_back(E.view((uint64_t *)(uintptr_t)256, batch, levels[i]));
            vec_run(E, which, v);
        });
        return pk + pk / 4 + (64u << 20);
    } catch (...) {
        return 0;
    }
}

static bc_status run_vec(bc_ctx *X, const bc_keys *k, int which, const bc_ct *v, uint32_t T, bc_ct *out, void *ws,
                         size_t wsb, void *st) {
    API_BEGIN
    if (!X || !k || !out) BC_THROW(BC_E_ARG, "null argument");
    Arena A;
    A.init(ws, wsb, false);
    Eng E{X, k, &A, S(st)};
    std::vector<CT> views = vec_views(X, E, v, T);
    {
        std::vector<uint32_t> lv(T);
        for (uint32_t i = 0; i < T; ++i) lv[i] = v[i].level;
        const uint32_t want = bc_vec_out_level(X, which, lv.data(), T);
        const uint32_t nout = which == 2 ? T : 1;
        for (uint32_t i = 0; i < nout; ++i) check_out(X, out[i], v[0].batch, want, "out[i]");
    }
    std::vector<CT> r = vec_run(E, which, views);
    for (size_t i = 0; i < r.size(); ++i) {
        if (out[i].batch != r[i].B) BC_THROW(BC_E_ARG, "output batch mismatch");
        out_copy(E, r[i], out[i], 0);
    }
    check_launch();
    API_END
}

extern "C" {
bc_status bc_min_tree(bc_ctx *X, const bc_keys *k, const bc_ct *v, uint32_t T, bc_ct out, void *ws, size_t wsb,
                      void *st) {
    return run_vec(X, k, 0, v, T, &out, ws, wsb, st);
}
bc_status bc_max_tree(bc_ctx *X, const bc_keys *k, const bc_ct *v, uint32_t T, bc_ct out, void *ws, size_t wsb,
                      void *st) {
    return run_vec(X, k, 1, v, T, &out, ws, wsb, st);
}
bc_status bc_sort(bc_ctx *X, const bc_keys *k, const bc_ct *v, uint32_t T, bc_ct *out, void *ws, size_t wsb,
                  void *st) {
    return run_vec(X, k, 2, v, T, out, ws, wsb, st);
}
}  // extern "C"
