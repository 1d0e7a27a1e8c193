// dpds.cuh -- exact, instruction-lean restatement of the per-value decimal analysis
// (dp_ds_calculate_counted, reference numeric.hpp:108-140).  Included only by the
// kernel translation unit.  Every function returns exactly what the reference loop
// decides; DESIGN.md "Exact fast analysis" carries the proofs, and
// tests/test_gpu_dpds.py checks them against the CPU oracle on ~1.6 M adversarial f64
// inputs (random bit patterns, decimals, 1-3 ulp perturbations, decade edges) per candidate
// scale (10 scales), ~1.2 M f32 inputs per scale (7 scales); the full-size parity gates
// cover the encoder's use of them on every config's whole archive.
//
// (1) Gap test.  The reference accepts scale a when |s - round(s)| <= |s| * 2^-52 with
//     s = RN(v * 10^a).  Writing s = M * 2^(E-52) (M in [2^52, 2^53)) and G for the
//     distance of s to the nearest integer in ulps, the test is G * 2^(E-52) <=
//     M * 2^(E-104), i.e. G <= M / 2^52 in [1, 2): it holds iff G <= 1.  For |s| < 1
//     it holds only for s = +-(1 - 2^-53) (nearest +-1).  So the test is a mask on the
//     fraction bits of s, and the rounded integer N is read off the same bits.
// (2) Reconstruction check.  The reference rejects v unless RN(N / 10^a) == v.  Within
//     the loop bounds (beta <= max_beta, so |s| < 10^15 for f64), e = N - v * 10^a is a
//     multiple of 2^(ev-52+a) of magnitude < 2^53 of those units, so fma(-v, p, N)
//     yields e exactly, and RN(N/p) == v  <=>  |e| < p * ulp(v)/2 (halved below a power
//     of two), ties resolved to even -- all exact comparisons.  f32 keeps the residual
//     in float: exact whenever |e| < 2^24 u (u its grid), while H < 2^23 u.
// (3) Certification at a candidate scale A (alpha0 <= A <= loop bound).  If the
//     reference test passes at some alpha_v <= A, then v*10^A lies within 3.5 ulp of
//     N_v * 10^(A - alpha_v) and that integer is the N found at A (|s| < 2^50 makes the
//     ulp <= 1/8).  Hence when the test passes at A: alpha_v <= A, and the
//     reconstruction check at A divides the same real number N_v / 10^alpha_v, so it
//     gives the same verdict.  When the test fails at A nothing is concluded.
#pragma once

#include <climits>

#include "falcon_common.cuh"

namespace fb200 {

template <typename T> struct fpx;

template <> struct fpx<double> {
    using B = uint64_t;
    using S = int64_t;
    static constexpr int MB = 52;                 // mantissa bits
    static constexpr B MANT = (B(1) << 52) - 1;
    static constexpr B SIGN = B(1) << 63;
    static constexpr B EXPF = B(0x7ff) << 52;
    static constexpr int BIAS = 1023;
    static constexpr unsigned EMASK = 0x7ffu;
    static constexpr int MAXA = 22, MAXB = 15, MIND = -308;
    __device__ static double pow10(int a) { return g_pow10_f64[a]; }
    __device__ static B dec(int k) { return g_decade_f64[k - MIND]; }
    __device__ static B bits(double v) { return (B)__double_as_longlong(v); }
    __device__ static double val(B b) { return __longlong_as_double((long long)b); }
    __device__ static double rint_(double x) { return rint(x); }
    __device__ static S to_int(double N) { return (S)__double2ll_rz(N); }
    // exact reconstruction verdict RN(N / p) == v from the exact residual (2)
    __device__ static bool recon_ok(double v, double p, double N) {
        const B eb = bits(__fma_rn(-v, p, N));   // exact: N - v*p
        const B ae = eb & ~SIGN;
        const B vb = bits(v);
        const B halve = (((eb ^ vb) & SIGN) != 0 && (vb & MANT) == 0) ? 1 : 0;
        // H = p * 2^(ev - 53) (halved below a power of two) by exponent arithmetic
        const B hb = bits(p) + (((vb >> MB) & EMASK) - (B)(BIAS + MB + 1) - halve << MB);
        return ae == 0 || ae < hb || (ae == hb && (vb & 1) == 0);
    }
};

template <> struct fpx<float> {
    using B = uint32_t;
    using S = int32_t;
    static constexpr int MB = 23;
    static constexpr B MANT = (B(1) << 23) - 1;
    static constexpr B SIGN = B(1) << 31;
    static constexpr B EXPF = B(0xff) << 23;
    static constexpr int BIAS = 127;
    static constexpr unsigned EMASK = 0xffu;
    static constexpr int MAXA = 10, MAXB = 6, MIND = -38;
    __device__ static float pow10(int a) { return g_pow10_f32[a]; }
    __device__ static B dec(int k) { return g_decade_f32[k - MIND]; }
    __device__ static B bits(float v) { return __float_as_uint(v); }
    __device__ static float val(B b) { return __uint_as_float(b); }
    __device__ static float rint_(float x) { return rintf(x); }
    __device__ static S to_int(float N) { return (S)__float2int_rz(N); }
    __device__ static bool recon_ok(float v, float p, float N) {
        // residual in float: a multiple of u = 2^(ev-23+a), exact whenever |e| < 2^24 u,
        // while H = p * ulp(v) / 2 = 5^a u / 2 < 2^23 u (a <= 10): exact verdicts
        const B eb = bits(__fmaf_rn(-v, p, N));
        const B ae = eb & ~SIGN;
        const B vb = bits(v);
        const B halve = (((eb ^ vb) & SIGN) != 0 && (vb & MANT) == 0) ? 1 : 0;
        // H = p * 2^(ev - 24) (halved below a power of two) by exponent arithmetic
        const B hb = bits(p) + (((vb >> MB) & EMASK) - (B)(BIAS + MB + 1) - halve << MB);
        return ae == 0 || ae < hb || (ae == hb && (vb & 1) == 0);
    }
};

// exact floor_log10 of a positive normal magnitude (numeric.hpp:54-66): with
// k0 = (floor_log2 * 78913) >> 18 the decade-table answer is always k0 or k0 + 1
// (checked exhaustively over every binade of both formats).
template <typename T>
__device__ __forceinline__ int mag_of(typename fpx<T>::B m) {
    using X = fpx<T>;
    const int e2 = (int)(m >> X::MB) - X::BIAS;
    const int k0 = (e2 * 78913) >> 18;
    return k0 + (m >= X::dec(k0 + 1) ? 1 : 0);
}

// (1): the reference gap test for s (|s - round(s)| <= |s| * 2^-52, numeric.hpp:127-129)
// holds iff s is within one ulp of an integer; rint() finds that integer (ties cannot
// pass), the difference is exact, and the comparison is on bit patterns.  On success
// *N = round_half_away(s).
template <typename T>
__device__ __forceinline__ bool near_integer(T s, T* N) {
    using X = fpx<T>;
    using B = typename X::B;
    const T r = X::rint_(s);
    const B sb = X::bits(s);
    const B ef = sb & X::EXPF;
    const B ulp = ef - ((B)X::MB << X::MB);        // bits of 2^(E - MB)
    const B ad = X::bits(s - r) & ~X::SIGN;         // exact |s - rint(s)|
    *N = r;
    return ef > ((B)X::MB << X::MB) && ad <= ulp;
}

// Reference loop (numeric.hpp:108-140) with (1) and (2).  alpha_v or -1 (exception).
// K consecutive candidate scales are tested per step (independent multiply/round
// chains: one step costs the latency of one candidate); the first candidate passing
// the gap test decides, exactly as in the sequential loop.  K = 1 keeps the call-site
// footprint small for the encoder's rare per-thread fallback; K = 3 is phase 1's
// sampling (sample_chunks_kernel, encode.cu).
template <typename T, int K>
__device__ __forceinline__ int dp_alpha_k(T v) {
    using X = fpx<T>;
    using B = typename X::B;
    const B b = X::bits(v);
    const B m = b & ~X::SIGN;
    if (m == 0) return (b & X::SIGN) ? -1 : 0;
    const B ef = b & X::EXPF;
    if (ef == 0 || ef == X::EXPF) return -1;
    const int mag = mag_of<T>(m);
    int alpha = mag < 0 ? -mag : 0;
    const int lim0 = X::MAXB - 1 - mag;
    const int limit = lim0 < X::MAXA ? lim0 : X::MAXA;
    for (; alpha <= limit; alpha += K) {
        T p[K], N[K];
        bool near[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int a = alpha + k <= limit ? alpha + k : limit;
            p[k] = X::pow10(a);
            near[k] = alpha + k <= limit && near_integer<T>(mul_rn(v, p[k]), &N[k]);
        }
        // first passing candidate, selected without indexing (keeps p/N in registers)
        int kk = -1;
        T pk = p[0], Nk = N[0];
#pragma unroll
        for (int k = K - 1; k >= 0; --k) {
            kk = near[k] ? k : kk;
            pk = near[k] ? p[k] : pk;
            Nk = near[k] ? N[k] : Nk;
        }
        if (kk >= 0) return X::recon_ok(v, pk, Nk) ? alpha + kk : -1;
    }
    return -1;
}

template <typename T>
__device__ __noinline__ int dp_alpha_full(T v) { return dp_alpha_k<T, 1>(v); }

// ---- inverse scale without a division (decode hot loop) ----
// RN(g / 10^a) (numeric.hpp:159-162) from the correctly rounded reciprocal rp = RN(1/p):
//   q0 = RN(g * rp);  r = g - q0 * p (exact, one FMA);  q = RN(q0 + r * rp)
// is exactly RN(g/p) when 5^a < 2^(P-2) (P = 53 / 24: a <= 21 f64, a <= 9 f32).  Proof
// (DESIGN.md 4): |q0 - x| < 2 ulp(x) for x = g/p, so q0 + r*rp = x + (x - q0) * d with
// |d| = |p*rp - 1| <= 2^-P, an error below 2^(E-2P+2) in x's binade E.  A midpoint m of
// that binade is an odd multiple of 2^(E-P) and g - m*p is a multiple of 2^(E-P+a) that is
// never zero (m*p has an odd part of more than P bits, g is a P-bit float), so
// |x - m| >= 2^(E-P) / 5^a > 2^(E-2P+2): no midpoint separates x from q0 + r*rp.
constexpr int kMarksteinMaxAlpha64 = 21;
constexpr int kMarksteinMaxAlpha32 = 9;
__device__ __forceinline__ double div_pow10_markstein(double g, double p, double rp) {
    const double q0 = __dmul_rn(g, rp);
    const double r = __fma_rn(-q0, p, g);
    return __fma_rn(r, rp, q0);
}
__device__ __forceinline__ float div_pow10_markstein(float g, float p, float rp) {
    const float q0 = __fmul_rn(g, rp);
    const float r = __fmaf_rn(-q0, p, g);
    return __fmaf_rn(r, rp, q0);
}

enum : int { CERT_UNDECIDED = 0, CERT_OK = 1, CERT_EXC = 2 };

// SELF-TEST ONLY (selftest.cu; the encoder uses certify_lean below): branch-free form of
// dp_certify with the same verdicts (the self-test compares the two), written with selects so the unrolled per-thread
// values interleave.  Also returns floor_log10(|v|) of nonzero normal values
// (max over the chunk gives floor_log10(max|v|) for beta_hat, transform.hpp:62-63);
// *mag = INT_MIN for zeros and specials.
__device__ __forceinline__ int certify_fast(double v, int A, double p, int64_t* g, int* mag_out) {
    using X = fpx<double>;
    const uint64_t b = X::bits(v);
    const uint32_t hi = (uint32_t)(b >> 32), lo = (uint32_t)b;
    const uint32_t ahi = hi & 0x7fffffffu;
    const bool zero = (ahi | lo) == 0;
    const uint32_t ef = ahi >> 20;
    const bool special = ef == 0 || ef == 0x7ffu;
    const int e2 = (int)ef - 1023;
    const int k0 = (e2 * 78913) >> 18;
    const int mag = k0 + ((b & ~X::SIGN) >= X::dec(k0 + 1) ? 1 : 0);  // table has a guard entry
    const bool inrange = A + mag >= 0 && A + mag <= X::MAXB - 1;
    // gap test: |s - rint(s)| <= ulp(s)  (valid for |s| >= 1/2, guaranteed when inrange)
    const double s = __dmul_rn(v, p);
    const double r = rint(s);
    const double d = __dsub_rn(s, r);
    const uint32_t uhi = (__double2hiint(s) & 0x7ff00000u) - (52u << 20);
    const double ulp = __hiloint2double((int)uhi, 0);
    const bool near = fabs(d) <= ulp;
    // reconstruction: |N - v*p| against p * ulp(v) / 2, halved below a power of two
    const double e = __fma_rn(-v, p, r);
    const bool toward0 = (__double2hiint(e) ^ (int)hi) < 0;
    const bool pow2 = (hi & 0x000fffffu) == 0 && lo == 0;
    const uint32_t hexp = ef - 53u - ((pow2 && toward0) ? 1u : 0u);
    const double H = __dmul_rn(p, __hiloint2double((int)(hexp << 20), 0));
    const double ae = fabs(e);
    const bool recon = ae < H || (ae == H && (lo & 1u) == 0);
    *g = zero ? 0 : (int64_t)__double2ll_rz(r);
    *mag_out = (zero || special) ? INT_MIN : mag;
    if (zero) return (hi >> 31) ? CERT_EXC : CERT_OK;
    if (special) return CERT_EXC;
    if (!inrange || !near) return CERT_UNDECIDED;
    return recon ? CERT_OK : CERT_EXC;
}

__device__ __forceinline__ int certify_fast(float v, int A, float p, int32_t* g, int* mag_out) {
    using X = fpx<float>;
    const uint32_t b = X::bits(v);
    const uint32_t ab = b & 0x7fffffffu;
    const bool zero = ab == 0;
    const uint32_t ef = ab >> 23;
    const bool special = ef == 0 || ef == 0xffu;
    const int e2 = (int)ef - 127;
    const int k0 = (e2 * 78913) >> 18;
    const int mag = k0 + (ab >= X::dec(k0 + 1) ? 1 : 0);  // table has a guard entry
    const bool inrange = A + mag >= 0 && A + mag <= X::MAXB - 1;
    const float s = __fmul_rn(v, p);
    const float r = rintf(s);
    const float d = __fsub_rn(s, r);
    const float ulp = __uint_as_float((__float_as_uint(s) & 0x7f800000u) - (23u << 23));
    const bool near = fabsf(d) <= ulp;
    const double e = __fma_rn(-(double)v, (double)p, (double)r);
    const bool toward0 = ((uint32_t)__double2hiint(e) >> 31) != (b >> 31);
    const bool pow2 = (b & 0x007fffffu) == 0;
    // 2^(ev - 24) as a double: exponent field ef - 127 - 24 + 1023
    const uint32_t hexp = ef + 872u - ((pow2 && toward0) ? 1u : 0u);
    const double H = __dmul_rn((double)p, __hiloint2double((int)(hexp << 20), 0));
    const double ae = fabs(e);
    const bool recon = ae < H || (ae == H && (b & 1u) == 0);
    *g = zero ? 0 : (int32_t)__float2int_rz(r);
    *mag_out = (zero || special) ? INT_MIN : mag;
    if (zero) return (b >> 31) ? CERT_EXC : CERT_OK;
    if (special) return CERT_EXC;
    if (!inrange || !near) return CERT_UNDECIDED;
    return recon ? CERT_OK : CERT_EXC;
}


// ---- lean certification (the encoder's hot loop) ----
// One-sided form of dp_certify: true only where dp_certify returns CERT_OK, with the
// same lane integer; false means "undecided" (the exact loop decides).  Dropped
// relative to dp_certify, each moving a rare case to the exact loop:
//   * the gap test: with N = rint(s), |N - v*p| < p*ulp(v)/2 already implies
//     |s - N| < ulp(s)/2 + p*2^(ev-53) < 1.5 ulp(s), and s - N is a multiple of ulp(s)
//     (or zero), so the reference gap test (1) holds;
//   * the per-value floor_log10: the range alpha0 <= A, A + mag <= max_beta - 1 is
//     |v| >= dec(-A) and |v| < dec(max_beta - A); f64 compares high words strictly
//     (equal high words -> undecided), f32 compares exactly;
//   * powers of two (halved rounding interval) and exact ties (|e| == H).
// The chunk-uniform parameters come from cert_params_for().
template <typename T> struct cert_params;
template <> struct cert_params<double> {
    double p;         // 10^A
    uint32_t lo1;     // hi(dec(-A)) + 1
    uint32_t span;    // hi(dec(15 - A)) - hi(dec(-A)) - 1
    uint32_t hk;      // hi(p) - (1076 << 20): hi word of H = p * 2^(ev - 53) is (ahi & EXP) + hk
    uint32_t plo;     // lo(p)
};
template <> struct cert_params<float> {
    float p;
    uint32_t lo;      // bits(dec(-A))
    uint32_t span;    // bits(dec(6 - A)) - bits(dec(-A))
    uint32_t hk;      // bits(p) - (151 << 23): bits of H = p * 2^(ev - 24) are (ab & EXP) + hk
};

__device__ __forceinline__ cert_params<double> cert_params_for(double, int A) {
    using X = fpx<double>;
    cert_params<double> c;
    c.p = X::pow10(A);
    const uint32_t L = (uint32_t)(X::dec(-A) >> 32), U = (uint32_t)(X::dec(X::MAXB - A) >> 32);
    c.lo1 = L + 1u;
    c.span = U > L + 1u ? U - L - 1u : 0u;
    c.hk = (uint32_t)__double2hiint(c.p) - (1076u << 20);
    c.plo = (uint32_t)__double2loint(c.p);
    return c;
}
__device__ __forceinline__ cert_params<float> cert_params_for(float, int A) {
    using X = fpx<float>;
    cert_params<float> c;
    c.p = X::pow10(A);
    c.lo = X::dec(-A);
    c.span = X::dec(X::MAXB - A) - c.lo;
    c.hk = __float_as_uint(c.p) - (151u << 23);
    return c;
}

// *g = rint(v * 10^A) (valid when true); *ah = |v|'s high word (f64) / bits (f32)
__device__ __forceinline__ bool certify_lean(double v, const cert_params<double>& c, int64_t* g, uint32_t* ah) {
    const uint32_t hi = (uint32_t)__double2hiint(v), lo = (uint32_t)__double2loint(v);
    const uint32_t ahi = hi & 0x7fffffffu;
    *ah = ahi;
    const bool inr = (ahi - c.lo1) < c.span;
    const bool notpow2 = ((ahi & 0x000fffffu) | lo) != 0u;
    const double s = __dmul_rn(v, c.p);
    const double r = rint(s);
    const double e = __fma_rn(-v, c.p, r);  // exact (dpds (2))
    const double H = __hiloint2double((int)((ahi & 0x7ff00000u) + c.hk), (int)c.plo);
    *g = __double2ll_rz(r);
    return inr && notpow2 && fabs(e) < H;
}
__device__ __forceinline__ bool certify_lean(float v, const cert_params<float>& c, int32_t* g, uint32_t* ah) {
    const uint32_t ab = __float_as_uint(v) & 0x7fffffffu;
    *ah = ab;
    const bool inr = (ab - c.lo) < c.span;
    const bool notpow2 = (ab & 0x007fffffu) != 0u;
    const float s = __fmul_rn(v, c.p);
    const float r = rintf(s);
    // e = r - v*p is a multiple of u = 2^(ev-23+A) (< 1/2 in range); whenever |e| < 2^24 u
    // the FMA is exact, and H = 5^A u / 2 < 2^23 u (A <= 10), so |e| < H is decided exactly
    const float e = __fmaf_rn(-v, c.p, r);
    const float H = __uint_as_float((ab & 0x7f800000u) + c.hk);
    *g = (int32_t)__float2int_rz(r);
    return inr && notpow2 && fabsf(e) < H;
}

// SELF-TEST ONLY (selftest.cu, the specification certify_lean / certify_fast are checked
// against).  (3): decide v against candidate scale A (0 <= A <= max_alpha).  CERT_OK: alpha_v <= A
// and v is not an exception, *g = round_half_away(v*10^A).  CERT_EXC: v is an
// exception.  CERT_UNDECIDED: run dp_alpha_full.
template <typename T>
__device__ __forceinline__ int dp_certify(T v, int A, T p, typename fpx<T>::S* g) {
    using X = fpx<T>;
    using B = typename X::B;
    const B b = X::bits(v);
    const B m = b & ~X::SIGN;
    const B ef = b & X::EXPF;
    *g = 0;
    if (m == 0) return (b & X::SIGN) ? CERT_EXC : CERT_OK;  // -0 -> exception; +0 -> alpha 0
    if (ef == 0 || ef == X::EXPF) return CERT_EXC;           // subnormal, inf, nan
    const int mag = mag_of<T>(m);
    // A must lie inside the reference loop's range: alpha0 = max(0, -mag) <= A and
    // beta = A + mag + 1 <= max_beta
    if (A < -mag || A + mag > X::MAXB - 1) return CERT_UNDECIDED;
    T N;
    if (!near_integer<T>(mul_rn(v, p), &N)) return CERT_UNDECIDED;
    *g = X::to_int(N);
    return X::recon_ok(v, p, N) ? CERT_OK : CERT_EXC;
}

}  // namespace fb200
