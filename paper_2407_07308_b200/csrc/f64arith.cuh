// f64arith.cuh -- exact modular arithmetic of residues below 2^50 on the binary64 FMA pipe (sm_100a).
//
// A residue class mod q (2^49 <= q < 2^50 for the element-wise kernels; q < 2^50 for the NTT) is held
// as a signed integer-valued double v with |v| <= 8q < 2^53 (every such integer is exact in binary64).
//   fmm (a, (w, wq)):  h = fl(a w); l = a w - h (one FMA, exact); t = rint(a wq) (FMA with 1.5*2^52,
//                      DADD); r = (h - t q) + l  -- both steps exact (integers below 2^53).
//                      |a| <= 4q, |w| <= q/2, wq = fl(w/q)  =>  |r| <= 0.625 q.
//   fmulv(a, b):       a, b canonical (|a|, |b| < q): t = rint(fl(a b) fl(1/q)), same exact
//                      remainder  =>  |r| <= 0.75 q.
//   fred(x):           x - rint(x fl(1/q)) q, |x| <= 8q  =>  |r| <= q/2 + 2.
// B200 issues 64 DFMA per SM per clock (the IMAD rate), so these cost 6 FP64-pipe operations per
// modular product against ~12-30 integer-pipe instructions for the 64-bit Shoup/Barrett products.
#pragma once
#include <cstdint>

namespace bc {
namespace f64 {

constexpr double RND = 6755399441055744.0;   // 1.5 * 2^52: fl(x + RND) - RND = rint(x) for |x| < 2^51
constexpr double TWO52 = 4503599627370496.0;

__device__ __forceinline__ double fmm(double a, double2 w, double q) {
    const double h = __dmul_rn(a, w.x);
    const double l = __fma_rn(a, w.x, -h);
    const double t = __dsub_rn(__fma_rn(a, w.y, RND), RND);
    const double r = __fma_rn(-t, q, h);
    return __dadd_rn(r, l);
}
__device__ __forceinline__ double fmulv(double a, double b, double q, double qi) {
    const double h = __dmul_rn(a, b);
    const double l = __fma_rn(a, b, -h);
    const double t = __dsub_rn(__fma_rn(h, qi, RND), RND);
    const double r = __fma_rn(-t, q, h);
    return __dadd_rn(r, l);
}
__device__ __forceinline__ double fred(double x, double q, double qi) {
    const double t = __dsub_rn(__fma_rn(x, qi, RND), RND);
    return __fma_rn(-t, q, x);
}
// canonical residue of |x| <= q -> u64
__device__ __forceinline__ uint64_t to_u64(double x, double q) {
    double c = x < 0.0 ? __dadd_rn(x, q) : x;
    c = c >= q ? __dsub_rn(c, q) : c;
    return (uint64_t)__double_as_longlong(__dadd_rn(c, TWO52)) - 0x4330000000000000ull;
}
// canonical double of |x| <= q (for digit comparisons)
__device__ __forceinline__ double canon(double x, double q) {
    double c = x < 0.0 ? __dadd_rn(x, q) : x;
    return c >= q ? __dsub_rn(c, q) : c;
}
__device__ __forceinline__ double from_u64(uint64_t x) {   // x < 2^52
    return __dsub_rn(__longlong_as_double((long long)(x | 0x4330000000000000ull)), TWO52);
}
// host/device: centred table entry (w, fl(w/q)) of a canonical residue w
__host__ __device__ inline double2 centred_entry(uint64_t w, uint64_t q) {
    const double wc = (double)(w > q / 2 ? (int64_t)w - (int64_t)q : (int64_t)w);
    double2 e;
    e.x = wc;
    e.y = wc / (double)q;
    return e;
}

}  // namespace f64
}  // namespace bc
