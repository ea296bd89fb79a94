// Butterfly throughput microbenchmark (sm_100a): 64-bit integer Shoup butterflies (IMAD pipe)
// vs FP64 FMA butterflies (fp64 pipe) vs both interleaved. Register-only loops, no memory.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t shoup4(uint64_t x, uint64_t w, uint64_t wp, uint64_t nq) {
    const uint32_t x0 = (uint32_t)x, x1 = (uint32_t)(x >> 32);
    const uint32_t p0 = (uint32_t)wp, p1 = (uint32_t)(wp >> 32);
    const uint64_t hi = (uint64_t)x1 * p1 + __umulhi(x1, p0) + __umulhi(x0, p1);
    return x * w + hi * nq;
}
// fp64 modular product: a*w - rint(a*wq)*q, exact (|a| < 2^52, q < 2^50), result |r| <= 0.75q
__device__ __forceinline__ double fmulmod(double a, double w, double wq, double q) {
    const double C = 6755399441055744.0;  // 1.5 * 2^52
    double h = a * w;
    double l = fma(a, w, -h);
    double t = fma(a, wq, C) - C;
    double r = fma(-t, q, h);
    return r + l;
}
__device__ __forceinline__ double fred(double x, double qi, double q) {
    const double C = 6755399441055744.0;
    double t = fma(x, qi, C) - C;
    return fma(-t, q, x);
}

constexpr int CH = 8;  // independent butterfly pairs per thread

__global__ void k_int(uint64_t *out, int iters, uint64_t q, uint64_t w0, uint64_t wp0) {
    uint64_t x[CH], y[CH];
    for (int i = 0; i < CH; ++i) { x[i] = threadIdx.x * 7 + i; y[i] = blockIdx.x * 13 + i * 3; }
    uint64_t w = w0, wp = wp0; const uint64_t nq = 0 - q, q4 = 4 * q, q2 = 2*q;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            uint64_t t = shoup4(y[i], w, wp, nq);
            uint64_t a = x[i];
            a = a >= q2 ? a - q2 : a;      // keep bounded (one conditional per butterfly as in lazy NTT)
            x[i] = a + t;
            y[i] = a + q4 - t;
        }
        w += 1; wp += 3;
    }
    uint64_t s = 0; for (int i = 0; i < CH; ++i) s += x[i] ^ y[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_f64(double *out, int iters, double q, double w0, double wq0) {
    double x[CH], y[CH];
    for (int i = 0; i < CH; ++i) { x[i] = threadIdx.x * 7 + i; y[i] = blockIdx.x * 13 + i * 3; }
    double w = w0, wq = wq0; const double qi = 1.0 / q;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            double t = fmulmod(y[i], w, wq, q);
            double a = x[i];
            if (it & 1) a = fred(a, qi, q);   // a reduction every other stage (bounded growth)
            x[i] = a + t;
            y[i] = a - t;
        }
        w += 1.0; wq += 1e-15;
    }
    double s = 0; for (int i = 0; i < CH; ++i) s += x[i] + y[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_mix(uint64_t *out, int iters, uint64_t q, uint64_t w0, uint64_t wp0, double qd, double wd0, double wqd0) {
    uint64_t x[CH/2], y[CH/2]; double xd[CH/2], yd[CH/2];
    for (int i = 0; i < CH/2; ++i) { x[i] = threadIdx.x * 7 + i; y[i] = blockIdx.x * 13 + i * 3; xd[i] = x[i]; yd[i] = y[i]; }
    uint64_t w = w0, wp = wp0; const uint64_t nq = 0 - q, q4 = 4 * q, q2 = 2*q;
    double wd = wd0, wqd = wqd0; const double qi = 1.0 / qd;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CH/2; ++i) {
            uint64_t t = shoup4(y[i], w, wp, nq);
            uint64_t a = x[i];
            a = a >= q2 ? a - q2 : a;
            x[i] = a + t; y[i] = a + q4 - t;
            double td = fmulmod(yd[i], wd, wqd, qd);
            double ad = xd[i];
            if (it & 1) ad = fred(ad, qi, qd);
            xd[i] = ad + td; yd[i] = ad - td;
        }
        w += 1; wp += 3; wd += 1.0; wqd += 1e-15;
    }
    uint64_t s = 0; for (int i = 0; i < CH/2; ++i) s += (x[i] ^ y[i]) + (uint64_t)(xd[i] + yd[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dfma(double *out, int iters) {
    double a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(a[i], 1.0000001, 0.5);
    double s = 0; for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_imad(uint32_t *out, int iters) {
    uint32_t a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = a[i] * 2654435761u + (uint32_t)it;
    uint32_t s = 0; for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int blocks = 148 * 8, threads = 256, iters = 4096;
    void *buf; cudaMalloc(&buf, (size_t)blocks * threads * 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const uint64_t q = 1125899906842597ull;  // ~2^50 (primality irrelevant for throughput)
    const double nthreads = (double)blocks * threads;
    auto timeit = [&](const char *name, double ops_per_iter, auto launch) {
        launch(); cudaDeviceSynchronize();
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
        }
        double rate = nthreads * iters * ops_per_iter / (best * 1e-3);
        printf("%-28s %8.3f ms  %8.3f G/s\n", name, best, rate / 1e9);
    };
    timeit("dfma (lane-ops)", 8, [&] { k_dfma<<<blocks, threads>>>((double *)buf, iters); });
    timeit("imad32 (lane-ops)", 8, [&] { k_imad<<<blocks, threads>>>((uint32_t *)buf, iters); });
    timeit("int64 shoup butterflies", CH, [&] { k_int<<<blocks, threads>>>((uint64_t *)buf, iters, q, 123456789ull, 987654321ull); });
    timeit("fp64 butterflies", CH, [&] { k_f64<<<blocks, threads>>>((double *)buf, iters, (double)q, 123456789.0, 123456789.0 / (double)q); });
    timeit("mixed int+fp64 butterflies", CH, [&] { k_mix<<<blocks, threads>>>((uint64_t *)buf, iters, q, 123456789ull, 987654321ull, (double)q, 123456789.0, 123456789.0 / (double)q); });
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("clock attr %d kHz\n", clk);
    return 0;
}
